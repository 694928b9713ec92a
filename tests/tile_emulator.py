"""Host emulation of the chunked kernel's tile program (test/tool infrastructure).

Replays the exported program (``Plan.export("tile_*")``: the exact tables
``hs_skeleton_create`` uploads for one character) phase by phase in fp64:
phase 1 chunk folds publishing anchors, phase 2 pointer jumping over the anchor
forest with the ping-pong locations as encoded, phase 3 re-folds + bind.  On the
exact-arithmetic family every association order gives the same bits, so a
bitwise match with the oracle pins the encoding (locations, buffers, ordering).

It also counts shared-memory wavefronts per 128-bit warp access the way the
hardware serves them (4 quarter-warp phases; per phase, the max number of
distinct 16-byte units that share a bank group) — the bank-conflict model used
to choose slot colours and list order.
"""
from __future__ import annotations

import collections

import numpy as np

SRC_ROOT, SRC_PREV, SRC_NONE, SRC_RUN = -1, -2, -3, -4


def _h(m):
    h = np.zeros((4, 4))
    h[:3] = m
    h[3, 3] = 1.0
    return h


def decode_meta(w):
    w = int(w)
    off = w & 0xFFFF
    ibu = (w >> 16) & 0xFFFF
    src = ((w >> 32) & 0xFFFF)
    own = ((w >> 48) & 0xFFFF)
    src = src - 0x10000 if src >= 0x8000 else src
    own = own - 0x10000 if own >= 0x8000 else own
    return off, ibu, src, own


class WavefrontCounter:
    """Counts 128-bit shared accesses: list of (lane, byte address) per warp instruction."""

    def __init__(self):
        self.wave = collections.Counter()
        self.ideal = collections.Counter()

    def access(self, name, lane_addrs):
        phases = collections.defaultdict(dict)
        for lane, addr in lane_addrs:
            unit = addr // 16
            phases[lane // 8].setdefault(unit % 8, set()).add(unit)
        for groups in phases.values():
            self.wave[name] += max(len(v) for v in groups.values())
            self.ideal[name] += 1

    def matrix(self, name, lane_addrs):
        """A 48-byte matrix = three 128-bit accesses at +0, +16, +32."""
        for k in range(3):
            self.access(name, [(lane, a + 16 * k) for lane, a in lane_addrs])


def run(plan, local, inv_bind=None, count=False):
    """local: [J,3,4] (one character); returns (G, S) in user order, and the counter."""
    meta = plan.export("tile_meta")
    p1len = plan.export("tile_p1len")
    round_off = plan.export("tile_round_off")
    rounds = plan.export("tile_rounds")
    S = plan.query("tile_slots")
    T, K = meta.shape
    J = local.shape[0]
    L = [_h(m) for m in np.asarray(local, np.float64)]
    IB = [_h(m) for m in (np.asarray(inv_bind, np.float64) if inv_bind is not None
                          else np.broadcast_to(np.hstack([np.eye(3), np.zeros((3, 1))]), (J, 3, 4)))]
    P = [None] * (2 * S)
    G = [None] * J
    SK = [None] * J
    wc = WavefrontCounter() if count else None
    dec = [[decode_meta(meta[t, s]) for s in range(K)] for t in range(T)]
    info = [int(x) for x in p1len]
    p1len = [x & 0xFF for x in info]
    run_back = [(x >> 8) & 0xFF for x in info]
    run_anchor = [((x & 0xFFFFFFFF) >> 16) - 1 for x in info]
    P_BASE = 0          # the P region's base residue is common to all its accesses
    NC = (T + 31) // 32 * 32

    # phase 1
    accs = [None] * T
    for s in range(K):
        lds, sts = collections.defaultdict(list), collections.defaultdict(list)
        for t in range(T):
            if s >= p1len[t]:
                continue
            off, ibu, src, own = dec[t][s]
            accs[t] = accs[t] @ L[off] if src == SRC_PREV else L[off].copy()
            lds[t // 32].append((t % 32, off * 48))
            if own >= 0:
                P[own] = accs[t].copy()
                sts[t // 32].append((t % 32, P_BASE + own * 48))
        if wc:
            for w in lds.values():
                wc.matrix("p1 L load", w)
            for w in sts.values():
                wc.matrix("p1 P store", w)
    # phase 2a: segmented warp scan over runs (Hillis-Steele over lanes, as the kernel)
    excl = [None] * T
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
    # phase 2
    for r in range(len(round_off) - 1):
        e0, e1 = int(round_off[r]), int(round_off[r + 1])
        writes = []
        by_warp = collections.defaultdict(lambda: collections.defaultdict(list))
        for e in range(e0, e1):
            w = int(rounds[e])
            slot, wbuf, sbuf, link = w & 0x3FFF, (w >> 14) & 1, (w >> 15) & 1, w >> 16
            self_loc, dst = slot + sbuf * S, slot + wbuf * S
            writes.append((dst, P[link] @ P[self_loc]))
            t = (e - e0) % NC
            it = (e - e0) // NC
            by_warp[(it, t // 32)]["link"].append((t % 32, P_BASE + link * 48))
            by_warp[(it, t // 32)]["self"].append((t % 32, P_BASE + self_loc * 48))
            by_warp[(it, t // 32)]["dst"].append((t % 32, P_BASE + dst * 48))
        for dst, val in writes:
            P[dst] = val
        if wc:
            for acc in by_warp.values():
                wc.matrix("p2 link load", acc["link"])
                wc.matrix("p2 self load", acc["self"])
                wc.matrix("p2 dst store", acc["dst"])
    # phase 3
    accs = [None] * T
    for s in range(K):
        ll, pl, gs = (collections.defaultdict(list) for _ in range(3))
        for t in range(T):
            off, ibu, src, own = dec[t][s]
            if src == SRC_NONE:
                continue
            if src == SRC_PREV:
                accs[t] = accs[t] @ L[off]
            elif src == SRC_ROOT:
                accs[t] = L[off].copy()
            elif src == SRC_RUN:
                base = P[run_anchor[t]] @ excl[t] if run_anchor[t] >= 0 else excl[t]
                accs[t] = base @ L[off]
            else:
                accs[t] = P[src] @ L[off]
                pl[t // 32].append((t % 32, P_BASE + src * 48))
            G[off] = accs[t]
            SK[off] = accs[t] @ IB[ibu]
            ll[t // 32].append((t % 32, off * 48))
        if wc:
            for w in ll.values():
                wc.matrix("p3 L load", w)
                wc.matrix("p3 G store", w)
                wc.matrix("p3 S store", w)
            for w in pl.values():
                wc.matrix("p3 P load", w)
    Gn = np.stack([g[:3] for g in G])
    Sn = np.stack([s[:3] for s in SK])
    return Gn, Sn, wc
