"""Host emulation of the multi-tile kernel's program (test infrastructure).

Replays the exported multi-tile program (``Plan.export("seq_*")``: the tables
``hs_skeleton_create`` uploads for HS_ALGO_TILES) for one character, tile by tile in
the kernel's order, in fp64 on 4x4 homogeneous matrices: phase 1 chunk folds
publishing anchors, phase 2a run scans, phase 2 pointer jumping (ping-pong locations
as encoded, Q locations final), phase 3 re-folds with forwards into the next tile's Q
buffer and the bind epilogue; then the tile's export list fills later tiles' inboxes
and tile k + 2's inbox lands in its Q buffer (each inbox row must have been written).  On the
exact-arithmetic family every association order gives the same bits, so a bitwise
match with the oracle pins the encoding (tiles, runs, imports, exports, locations).
"""
from __future__ import annotations

import numpy as np

from tests.tile_emulator import SRC_NONE, SRC_PREV, SRC_ROOT, SRC_RUN, _h


def decode(w):
    """Slot word: off 10 | src + 8 13 | own + 1 13 | export slot + 1 16 | forward + 1 12."""
    w = int(w)
    return (w & 0x3FF, (w >> 36) & 0xFFFF, ((w >> 10) & 0x1FFF) - 8, ((w >> 23) & 0x1FFF) - 1,
            (w >> 52) & 0xFFF)


def run(plan, local, inv_bind=None):
    """local: [J,3,4] (one character, user order); returns (G, S) in user order."""
    tiles = plan.export("seq_tiles")
    meta = plan.export("seq_meta")
    p1len = plan.export("seq_p1len")
    round_off = plan.export("seq_round_off")
    rounds = plan.export("seq_rounds")
    exl = plan.export("seq_imp")       # export lists: (smem offset, workspace row)
    runs = plan.export("seq_runs")
    ib_user = plan.export("seq_ib_user")
    S = plan.query("seq_slots")
    nQ = plan.query("seq_qslots")
    KT, T, K = meta.shape
    J = local.shape[0]
    IB = np.asarray(inv_bind, np.float64) if inv_bind is not None else \
        np.broadcast_to(np.hstack([np.eye(3), np.zeros((3, 1))]), (J, 3, 4))
    G = [None] * J
    SK = [None] * J
    ws = {}
    P = {}
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
        for loc in [x for x in P if x < 2 * S]:
            del P[loc]                                   # anchors are per tile; Q buffers persist
        dec = [[decode(meta[k, t, s]) for s in range(K)] for t in range(T)]
        info = [int(x) for x in p1len[k]]
        p1 = [x & 0xFF for x in info]
        run_back = [(x >> 8) & 0xFF for x in info]
        run_anchor = [((x & 0xFFFFFFFF) >> 16) - 1 for x in info]
        accs = [None] * T
        for t in range(T):      # phase 1
            for s in range(p1[t]):
                off, ex, src, own, fw = dec[t][s]
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
                off, ex, src, own, fw = dec[t][s]
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
                assert ex == 0                           # exports go through the export list
                if fw:
                    assert k + 1 < KT and fw - 1 < nQ
                    P[2 * S + ((k + 1) & 1) * nQ + fw - 1] = acc.copy()
        # tile k done: its exports into the later inboxes, then tile k + 2's inbox lands
        # in its Q buffer (k + 2) & 1 (the kernel's producer warp, after tile k is done)
        Gt = {o: None for o in range(nj)}
        for t in range(T):
            for s_ in range(K):
                off, ex, src, own, fw = dec[t][s_]
                if src != SRC_NONE:
                    Gt[off] = True
        n_exl, exl_off = tiles[k][10], tiles[k][11]
        for e in range(n_exl):
            off, row = exl[exl_off + e]
            assert Gt[int(off)], "export of a joint the tile did not compute"
            u = user_of[int(off)]
            ws[int(row)] = _h(G[u])
        if k + 2 < KT:
            nb = 2 * S + ((k + 2) & 1) * nQ
            for loc in [x for x in P if nb <= x < nb + nQ]:
                del P[loc]
            n_in, base = tiles[k + 2][5], tiles[k + 2][6]
            for z in range(n_in):
                assert base + z in ws, "inbox row not written before it is read"
                P[nb + z] = ws[base + z]
    assert (covered == 1).all(), "every joint is loaded exactly once"
    return np.stack(G), np.stack(SK)
