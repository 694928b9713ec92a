"""Randomised GPU parity (through the C ABI) over skeleton shapes and plan options the
fixed configs do not reach: random trees and forests of 1..1100 joints with random
depth, shuffled (non-topological) labels, every chunk construction, chunk sizes
3/5/7, stage counts and single/ping-pong anchor buffers, odd crowd sizes (ragged last
tile).  Exact family -> bitwise against the fp64 oracle; rigid family -> 1e-4.
Seeds are fixed, so a failure reproduces."""
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


def random_forest(rng, J):
    """A forest of 1-4 random trees with random depths, labels shuffled."""
    k = min(int(rng.integers(1, 5)), J)
    sizes = 1 + rng.multinomial(J - k, np.ones(k) / k)
    par, base = [], 0
    for n in sizes:
        n = int(n)
        d = int(rng.integers(1, n + 1))
        t = hsgen.random_tree(int(rng.integers(1 << 30)), n, d)
        par += [p + base if p >= 0 else -1 for p in t]
        base += n
    par = np.array(par, np.int32)
    perm = rng.permutation(J).astype(np.int32)
    new_par, _ = hsgen.relabel(par, perm)
    return new_par


CASES = []
_rng = np.random.default_rng(2025)
for i in range(36):
    J = int(_rng.choice([1, 2, 7, 33, 64, 150, 300, 511, 777, 1024, 1100]))
    CASES.append(dict(seed=int(_rng.integers(1 << 30)), J=J, n=int(_rng.integers(1, 70)),
                      chunk=int(_rng.choice([0, 3, 5, 7])), chunking=int(_rng.integers(0, 4)),
                      stages=int(_rng.choice([0, 2, 3])), pbuf=int(_rng.choice([0, 1, 2])),
                      exact=bool(i % 2)))


@pytest.mark.parametrize("case", CASES, ids=[f"J{c['J']}-k{c['chunk']}-c{c['chunking']}-{i}"
                                             for i, c in enumerate(CASES)])
def test_random_skeleton_parity(case):
    rng = np.random.default_rng(case["seed"])
    par = random_forest(rng, case["J"])
    J = len(par)
    gen, gib = (hsgen.exact_poses, hsgen.exact_inv_bind) if case["exact"] else (hsgen.local_poses, hsgen.inv_bind)
    loc = gen(case["seed"] % 1000, J, case["n"])
    ib = gib(case["seed"] % 1000 + 1, J)
    try:
        sk = hs.Skeleton(par, ib, chunk=case["chunk"], chunking=case["chunking"], stages=case["stages"],
                         pbuf=case["pbuf"])
    except hs.HSError as e:   # an option combination that does not fit: must say so, not crash
        assert e.status == hs.HS_ERR_UNSUPPORTED or case["J"] > 1000, e
        sk = hs.Skeleton(par, ib)
    g, s = sk.scan(torch.from_numpy(loc).cuda())
    torch.cuda.synchronize()
    G, S = oracle.scan(par, loc, ib)
    g, s = g.cpu().numpy().astype(np.float64), s.cpu().numpy().astype(np.float64)
    if case["exact"]:
        assert np.array_equal(g, G) and np.array_equal(s, S)
    else:
        assert np.abs(g - G).max() <= 1e-4 and np.abs(s - S).max() <= 1e-4


def test_random_batches_bitwise():
    rng = np.random.default_rng(77)
    for trial in range(4):
        items, ref = [], []
        for _ in range(int(rng.integers(2, hs.MAX_BATCH + 1))):
            J = int(rng.choice([5, 64, 200, 640, 1000]))
            par = random_forest(rng, J)
            sk = hs.Skeleton(par, hsgen.inv_bind(trial, J))
            n = int(rng.integers(0, 400))
            x = torch.from_numpy(hsgen.local_poses(trial, J, n)).cuda()
            g, s = torch.empty_like(x), torch.empty_like(x)
            items.append((sk, x, g, s))
            ref.append(sk.scan(x) if n else (g, s))
        hs.scan_batch(items)
        torch.cuda.synchronize()
        for (_, x, g, s), (rg, rs) in zip(items, ref):
            if x.shape[0]:
                assert torch.equal(g, rg) and torch.equal(s, rs)
