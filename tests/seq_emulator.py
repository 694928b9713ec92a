"""Host emulation of the multi-tile kernel's program (test infrastructure).

Replays the exported multi-tile program (``Plan.export("seq_*")``: the tables
``hs_skeleton_create`` uploads for HS_ALGO_TILES) for one character, tile by tile in
the kernel's order, in fp64 on 4x4 homogeneous matrices: import of external parents
from the workspace into Q locations, phase 1 chunk folds publishing anchors, phase 2a
run scans, phase 2 pointer jumping (ping-pong locations as encoded, Q locations
final), phase 3 re-folds with exports to the workspace and the bind epilogue.  On the
exact-arithmetic family every association order gives the same bits, so a bitwise
match with the oracle pins the encoding (tiles, runs, imports, exports, locations).
"""
from __future__ import annotations

import numpy as np

from tests.tile_emulator import SRC_NONE, SRC_PREV, SRC_ROOT, SRC_RUN, _h


def decode(w):
    w = int(w)
    off = w & 0xFFFF
    exp = (w >> 16) & 0xFFFF
    src = (w >> 32) & 0xFFFF
    own = (w >> 48) & 0xFFFF
    src = src - 0x10000 if src >= 0x8000 else src
    own = own - 0x10000 if own >= 0x8000 else own
    return off, exp, src, own


def run(plan, local, inv_bind=None):
    """local: [J,3,4] (one character, user order); returns (G, S) in user order."""
    tiles = plan.export("seq_tiles")
    meta = plan.export("seq_meta")
    p1len = plan.export("seq_p1len")
    round_off = plan.export("seq_round_off")
    rounds = plan.export("seq_rounds")
    imp = plan.export("seq_imp")
    runs = plan.export("seq_runs")
    ib_user = plan.export("seq_ib_user")
    S = plan.query("seq_slots")
    KT, T, K = meta.shape
    J = local.shape[0]
    IB = np.asarray(inv_bind, np.float64) if inv_bind is not None else \
        np.broadcast_to(np.hstack([np.eye(3), np.zeros((3, 1))]), (J, 3, 4))
    G = [None] * J
    SK = [None] * J
    ws = {}
    covered = np.zeros(J, int)
    for k in range(KT):
        first, nj, R2, n_ent, r_off, n_imp, imp_off, n_runs, runs_off, Tk = tiles[k][:10]
        # stage-in through the TMA runs: smem offset -> user label
        Lt = [None] * nj
        user_of = [None] * nj
        for r in range(n_runs):
            u0, o0, ln, _ = runs[runs_off + r]
            for z in range(ln):
                assert Lt[o0 + z] is None, "two runs write one smem slot"
                Lt[o0 + z] = _h(local[u0 + z])
                user_of[o0 + z] = u0 + z
                covered[u0 + z] += 1
        assert all(x is not None for x in Lt), "a smem slot of the tile is not loaded"
        assert list(ib_user[k][:nj]) == user_of
        P = {}
        for z in range(n_imp):
            slot, loc = imp[imp_off + z]
            assert loc >= 2 * S and slot in ws, "import of a value not exported before"
            P[int(loc)] = ws[int(slot)]
        dec = [[decode(meta[k, t, s]) for s in range(K)] for t in range(T)]
        info = [int(x) for x in p1len[k]]
        p1 = [x & 0xFF for x in info]
        run_back = [(x >> 8) & 0xFF for x in info]
        run_anchor = [((x & 0xFFFFFFFF) >> 16) - 1 for x in info]
        accs = [None] * T
        for t in range(T):      # phase 1
            for s in range(p1[t]):
                off, ex, src, own = dec[t][s]
                accs[t] = accs[t] @ Lt[off] if src == SRC_PREV else Lt[off].copy()
                if own >= 0:
                    assert own < 2 * S
                    P[own] = accs[t].copy()
        excl = [None] * T       # phase 2a
        for w0 in range(0, T, 32):
            lanes = list(range(w0, min(T, w0 + 32)))
            v = {t: accs[t] for t in lanes}
            d = 1
            while d < 32:
                nv = dict(v)
                for t in lanes:
                    if run_back[t] >= d:
                        nv[t] = v[t - d] @ v[t]
                v = nv
                d <<= 1
            for t in lanes:
                if run_back[t] > 0:
                    excl[t] = v[t - 1]
                    for s in range(K):
                        own = dec[t][s][3]
                        if own >= 0:
                            P[own] = excl[t] @ P[own]
        for r in range(R2):     # phase 2: ping-pong snapshot semantics
            eb, e1 = round_off[k][r], round_off[k][r + 1]
            writes = []
            for e in range(r_off + eb, r_off + e1):
                w = int(rounds[e])
                slot = w & 0x3FFF
                dst = slot + ((w >> 14) & 1) * S
                self_ = slot + ((w >> 15) & 1) * S
                link = w >> 16
                writes.append((dst, P[link] @ P[self_]))
            for dst, val in writes:
                P[dst] = val
        for t in range(T):      # phase 3
            acc = None
            for s in range(K):
                off, ex, src, own = dec[t][s]
                if src == SRC_NONE:
                    continue
                if src == SRC_PREV:
                    acc = acc @ Lt[off]
                elif src == SRC_ROOT:
                    acc = Lt[off].copy()
                elif src == SRC_RUN:
                    left = P[run_anchor[t]] @ excl[t] if run_anchor[t] >= 0 else excl[t]
                    acc = left @ Lt[off]
                else:
                    acc = P[src] @ Lt[off]
                u = user_of[off]
                G[u] = acc[:3].copy()
                SK[u] = (acc @ _h(IB[u]))[:3]
                if ex:
                    ws[ex - 1] = acc.copy()
    assert (covered == 1).all(), "every joint is loaded exactly once"
    return np.stack(G), np.stack(SK)
