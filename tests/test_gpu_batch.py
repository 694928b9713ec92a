"""GPU tests of the heterogeneous single launch (hs_scan_batch):
several crowds with different skeletons in one kernel launch.

Bar: bitwise equal to one hs_scan per item (the batch only changes which CTA runs
a tile, never how a character is chunked), and within the north-star 1e-4 of the
fp64 oracle on every item; bitwise to the oracle on the exact family.
"""
from __future__ import annotations

import numpy as np
import pytest

import hsgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2505_06703_b200 as hs  # noqa: E402

TOL = 1e-4


def crowd(name_or_par, n, seed, type_=0, exact=False):
    par = hsgen.skeleton(name_or_par) if isinstance(name_or_par, str) else np.asarray(name_or_par, np.int32)
    J = len(par)
    gen = hsgen.exact_poses if exact else hsgen.local_poses
    loc = gen(seed, J, n, type_=type_)
    ib = (hsgen.exact_inv_bind if exact else hsgen.inv_bind)(seed, J, type_=type_)
    return par, loc, ib


def run_batch(crowds, skin=True, **create):
    sks, items, outs = [], [], []
    for par, loc, ib in crowds:
        sk = hs.Skeleton(par, ib, **create)
        x = torch.from_numpy(loc).cuda()
        g = torch.full_like(x, float("nan"))
        s = torch.full_like(x, float("nan")) if skin else None
        sks.append(sk)
        items.append((sk, x, g, s))
        outs.append((g, s))
    hs.scan_batch(items)
    torch.cuda.synchronize()
    sep = []
    for sk, x, _, _ in items:   # reference: one hs_scan per item
        g2, s2 = sk.scan(x, skin=skin)
        sep.append((g2, s2))
    torch.cuda.synchronize()
    res = [(g.cpu().numpy(), None if s is None else s.cpu().numpy()) for g, s in outs]
    ref = [(g.cpu().numpy(), None if s is None else s.cpu().numpy()) for g, s in sep]
    return sks, res, ref


def test_c5_shaped_batch_bitwise_and_oracle():
    crowds = [crowd("hum64", 3001, 5, 0), crowd("chain256", 777, 5, 1), crowd("tree1024", 301, 5, 2),
              crowd("hum32", 129, 6, 3)]
    sks, res, ref = run_batch(crowds)
    assert len({sk.query("chunk") for sk in sks}) == 1
    for (par, loc, ib), (g, s), (g2, s2) in zip(crowds, res, ref):
        assert np.array_equal(g, g2) and np.array_equal(s, s2)
        idx = np.linspace(0, len(loc) - 1, 9).astype(int)
        G, S = oracle.scan(par, loc[idx], ib)
        assert np.abs(g[idx] - G).max() <= TOL and np.abs(s[idx] - S).max() <= TOL


def test_exact_family_batch_bitwise_to_oracle():
    crowds = [crowd("hum64", 40, 11, exact=True), crowd("tree1024", 7, 12, exact=True),
              crowd(hsgen.random_tree(3, 500, 40), 23, 13, exact=True)]
    _, res, _ = run_batch(crowds)
    for (par, loc, ib), (g, s) in zip(crowds, res):
        G, S = oracle.scan(par, loc, ib)
        assert np.array_equal(g.astype(np.float64), G) and np.array_equal(s.astype(np.float64), S)


def test_max_items_tiny_crowds_and_mixed_skin():
    # 8 segments (HS_MAX_BATCH), one- and two-character crowds, the same skeleton twice,
    # one item without the bind epilogue, one empty item
    sk_a = hs.Skeleton(hsgen.skeleton("hum64"), hsgen.inv_bind(1, 64))
    sk_b = hs.Skeleton(hsgen.skeleton("chain256"), hsgen.inv_bind(2, 256))
    items, want = [], []
    for i in range(hs.MAX_BATCH):
        sk, name = (sk_a, "hum64") if i % 2 == 0 else (sk_b, "chain256")
        n = [1, 2, 0, 1, 5, 1, 3, 2][i]
        loc = hsgen.local_poses(30 + i, sk.n_joints, n)
        x = torch.from_numpy(loc).cuda()
        g = torch.full_like(x, float("nan"))
        s = None if i == 3 else torch.full_like(x, float("nan"))
        items.append((sk, x, g, s))
        want.append((name, loc, g, s))
    hs.scan_batch(items)
    torch.cuda.synchronize()
    for (name, loc, g, s), it in zip(want, items):
        if len(loc) == 0:
            continue
        ref_g, ref_s = it[0].scan(it[1], skin=s is not None)
        assert torch.equal(g, ref_g)
        if s is not None:
            assert torch.equal(s, ref_s)


def test_batch_errors():
    sk5 = hs.Skeleton(hsgen.skeleton("hum64"))
    sk7 = hs.Skeleton(hsgen.skeleton("hum64"), chunk=7)
    x = torch.zeros((4, 64, 3, 4), device="cuda")
    g = torch.empty_like(x)
    with pytest.raises(hs.HSError) as ei:
        hs.scan_batch([(sk5, x, g, None), (sk7, x.clone(), torch.empty_like(x), None)])
    assert ei.value.status == hs.HS_ERR_UNSUPPORTED
    big = hs.Skeleton(hsgen.random_tree(9, 4096, 64))     # multi-CTA (split) path
    xb = torch.zeros((1, 4096, 3, 4), device="cuda")
    with pytest.raises(hs.HSError) as ei:
        hs.scan_batch([(big, xb, torch.empty_like(xb), None)])
    assert ei.value.status == hs.HS_ERR_UNSUPPORTED
    with pytest.raises(hs.HSError) as ei:
        hs.scan_batch([(sk5, x, g, None)] * (hs.MAX_BATCH + 1))
    assert ei.value.status == hs.HS_ERR_INVALID_ARG
    with pytest.raises(hs.HSError) as ei:
        hs.scan_batch([(sk5, x, x, None)])                  # output aliases input
    assert ei.value.status == hs.HS_ERR_INVALID_ARG
    hs.scan_batch([])                                       # nothing to do


def test_mixed_skin_batch_single_s_buffer():
    """items [skin, no skin, skin] with one S buffer, sized so every CTA gets
    exactly one tile of each item.  The consumer must await the S buffer on every tile
    (not only on skin tiles), else the third item's S can overwrite the first item's S
    while its bulk store still reads it.  Every item equals its own hs_scan bit for bit."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    par = hsgen.skeleton("hum64")
    ib = hsgen.inv_bind(71, 64)
    sk = hs.Skeleton(par, ib, stages=3, sbufs=1)
    assert sk.query("sbufs") == 1
    per_tile = sk.query("tile_chars")
    items, want = [], []
    for i, skin in enumerate((True, False, True)):
        n = per_tile * sms
        x = torch.from_numpy(hsgen.local_poses(72 + i, 64, n)).cuda()
        g = torch.full_like(x, float("nan"))
        s = torch.full_like(x, float("nan")) if skin else None
        items.append((sk, x, g, s))
        want.append(sk.scan(x, skin=skin))
    for _ in range(3):   # repeated: the race is timing dependent
        hs.scan_batch(items)
        torch.cuda.synchronize()
        for (_, _, g, s), (g2, s2) in zip(items, want):
            assert torch.equal(g, g2)
            if s is not None:
                assert torch.equal(s, s2)
