"""GPU parity of the per-character-topology scan (hs_scan_varied; SURVEY.md §8(f)
NEXT-3): every character has its own random forest (shuffled labels, any order) and
its own inverse binds; each is checked against the fp64 oracle on its own skeleton.
Exact family -> bitwise; rigid family -> 1e-4."""
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


def forests(seed, n, J):
    rng = np.random.default_rng(seed)
    out = np.empty((n, J), np.int32)
    for c in range(n):
        par = hsgen.random_tree(int(rng.integers(1 << 30)), J, int(rng.integers(1, J + 1)))
        roots = rng.random(J) < 0.02          # a few extra roots: forests
        par = np.where(roots, -1, par).astype(np.int32)
        perm = rng.permutation(J).astype(np.int32)
        out[c], _ = hsgen.relabel(par, perm)
    return out


@pytest.mark.parametrize("J,n,exact", [(1, 5, False), (33, 70, True), (64, 200, False), (300, 17, True),
                                       (1024, 6, False), (1024, 3, True)])
def test_varied_topology_parity(J, n, exact):
    par = forests(J * 7 + n, n, J)
    gen = hsgen.exact_poses if exact else hsgen.local_poses
    loc = gen(J + 1, J, n)
    ib = np.stack([(hsgen.exact_inv_bind if exact else hsgen.inv_bind)(c, J) for c in range(n)])
    g, s = hs.scan_varied(torch.from_numpy(par).cuda(), torch.from_numpy(loc).cuda(),
                          torch.from_numpy(ib).cuda())
    torch.cuda.synchronize()
    g, s = g.cpu().numpy().astype(np.float64), s.cpu().numpy().astype(np.float64)
    for c in range(n):
        G, S = oracle.scan(par[c], loc[c], ib[c])
        if exact:
            assert np.array_equal(g[c], G) and np.array_equal(s[c], S)
        else:
            assert np.abs(g[c] - G).max() <= 1e-4 and np.abs(s[c] - S).max() <= 1e-4


def test_varied_same_skeleton_matches_hs_scan_family():
    """With one shared skeleton the varied scan agrees with hs_scan on the exact family."""
    par = hsgen.skeleton("tree1024")
    loc = hsgen.exact_poses(5, 1024, 4)
    ib = hsgen.exact_inv_bind(6, 1024)
    sk = hs.Skeleton(par, ib)
    x = torch.from_numpy(loc).cuda()
    g1, s1 = sk.scan(x)
    g2, s2 = hs.scan_varied(torch.from_numpy(np.tile(par, (4, 1))).cuda(), x,
                            torch.from_numpy(np.tile(ib[None], (4, 1, 1, 1))).cuda())
    torch.cuda.synchronize()
    assert torch.equal(g1, g2) and torch.equal(s1, s2)


def test_varied_errors_and_no_skin():
    x = torch.zeros((2, 2000, 3, 4), device="cuda")
    p = torch.full((2, 2000), -1, dtype=torch.int32, device="cuda")
    with pytest.raises(hs.HSError) as e:
        hs.scan_varied(p, x)
    assert e.value.status == hs.HS_ERR_UNSUPPORTED
    # no inverse binds: skin equals global; out-of-range parents act as roots
    par = torch.tensor([[-1, 0, 7, 1]], dtype=torch.int32, device="cuda")
    loc = torch.from_numpy(hsgen.local_poses(3, 4, 1)).cuda()
    g, s = hs.scan_varied(par, loc)
    torch.cuda.synchronize()
    assert torch.equal(g, s)
    G, _ = oracle.scan([-1, 0, -1, 1], loc.cpu().numpy()[0])
    assert np.abs(g.cpu().numpy()[0] - G).max() <= 1e-5


@pytest.mark.parametrize("J,n,deep", [(64, 10_000, False), (1024, 300, True), (300, 1000, False)])
def test_varied_persistent_crowd_sampled(J, n, deep):
    """Crowds of more groups than SMs: the persistent CTA streams group after group
    (double-buffered locals, re-issued inverse binds, prefetched parents); sampled
    characters bitwise against the oracle on the exact family.  deep: 1024-joint chains
    (depth 1024: the longest anchor chains)."""
    rng = np.random.default_rng(J + n)
    base = forests(J + 3, 64, J) if not deep else np.tile(hsgen.chain(J), (64, 1))
    if deep:
        for c in range(64):
            base[c], _ = hsgen.relabel(hsgen.chain(J), rng.permutation(J).astype(np.int32))
    par = base[np.arange(n) % 64]
    loc = hsgen.exact_poses(J + 5, J, n)
    ibs = np.stack([hsgen.exact_inv_bind(c, J) for c in range(64)])
    ib = ibs[np.arange(n) % 64]
    g, s = hs.scan_varied(torch.from_numpy(np.ascontiguousarray(par)).cuda(), torch.from_numpy(loc).cuda(),
                          torch.from_numpy(np.ascontiguousarray(ib)).cuda())
    torch.cuda.synchronize()
    g, s = g.cpu().numpy(), s.cpu().numpy()
    for c in sorted(set([0, 1, n // 2, n - 2, n - 1] + rng.integers(0, n, 12).tolist())):
        G, S = oracle.scan(par[c], loc[c], ib[c])
        assert np.array_equal(g[c], G) and np.array_equal(s[c], S), c


def test_varied_cycle_terminates():
    """A cyclic parent array gives undefined values but the launch terminates."""
    par = torch.tensor([[1, 2, 0, -1, 3] * 100], dtype=torch.int32, device="cuda")[:, :500]
    par = par % 500
    loc = torch.from_numpy(hsgen.local_poses(3, 500, 1)).cuda()
    g, s = hs.scan_varied(par.contiguous(), loc)
    torch.cuda.synchronize()
    assert g.shape == (1, 500, 3, 4)
