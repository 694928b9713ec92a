"""GPU parity of the fused linear-blend-skinning epilogue (hs_scan_skin; SURVEY.md §8(f)
NEXT-4, R24) against the fp64 oracle (oracle.scan -> oracle.skin_vertices).

Tolerance: a skinned vertex is sum_k w_k (S_k (p, 1)) with sum w = 1 and |p_i| <= 1,
so an error e in each skin-matrix element moves it by at most (|p|_1 + 1) e <= 4e with
the north-star e = 1e-4 -> 4e-4, plus the fp32 rounding of the blend itself (~1e-6).
Against the LBS of the GPU's own skin output the bound is that rounding only: a few
fp32 ulps of the vertex magnitude, 2e-6 x (1 + max |v|).
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

TOL_VERTS = 4e-4
TOL_SELF = 2e-6   # x (1 + max |v|)


def run(par, loc, ib, mesh, skin=True, mode="auto", **create):
    sk = hs.Skeleton(par, ib, **create)
    m = hs.Mesh(sk, *mesh)
    x = torch.from_numpy(loc).cuda()
    g, s, v = hs.scan_skin(sk, m, x, skin=skin, mode=mode)
    torch.cuda.synchronize()
    g2, s2 = sk.scan(x)
    torch.cuda.synchronize()
    out = (g.cpu().numpy(), None if s is None else s.cpu().numpy(), v.cpu().numpy(),
           g2.cpu().numpy(), s2.cpu().numpy())
    return out


@pytest.mark.parametrize("mode", ["fused", "two_pass"])
@pytest.mark.parametrize("name,n,V", [("hum32", 100, 700), ("hum64", 300, 1000), ("chain256", 60, 1500),
                                      ("tree1024", 24, 2000)])
def test_lbs_parity(name, n, V, mode):
    par = hsgen.skeleton(name)
    J = len(par)
    loc = hsgen.local_poses(21, J, n)
    ib = hsgen.inv_bind(22, J)
    mesh = hsgen.mesh(23, par, V)
    g, s, v, g2, s2 = run(par, loc, ib, mesh, mode=mode)
    # the scan outputs are the plain hs_scan ones, bit for bit
    assert np.array_equal(g, g2) and np.array_equal(s, s2)
    G, S = oracle.scan(par, loc, ib)
    want = oracle.skin_vertices(S, *mesh)
    err = float(np.abs(v - want).max())
    self_err = float(np.abs(v - oracle.skin_vertices(s.astype(np.float64), *mesh)).max())
    print(f"{name}: verts vs oracle {err:.2e}, vs LBS of the GPU skin {self_err:.2e}")
    assert err <= TOL_VERTS and self_err <= TOL_SELF * (1 + float(np.abs(want).max()))


def test_lbs_without_skin_output_matches():
    par = hsgen.skeleton("hum64")
    loc = hsgen.local_poses(31, 64, 50)
    ib = hsgen.inv_bind(32, 64)
    mesh = hsgen.mesh(33, par, 900)
    _, s_none, v_none, _, _ = run(par, loc, ib, mesh, skin=False)
    _, _, v_skin, _, _ = run(par, loc, ib, mesh, skin=True)
    assert s_none is None and np.array_equal(v_none, v_skin)


def test_lbs_exact_family_bitwise():
    # exact poses (signed permutations, integer translations), positions in {-1, 0, 1}
    # and dyadic weights: every product and sum is exact in fp32
    par = hsgen.skeleton("tree1024")
    J = len(par)
    loc = hsgen.exact_poses(41, J, 5)
    ib = hsgen.exact_inv_bind(42, J)
    pos, jt, _ = hsgen.mesh(43, par, 1200)
    pos = np.sign(np.round(pos * 1.4)).astype(np.float32)
    w = np.tile(np.array([0.5, 0.25, 0.125, 0.125], np.float32), (len(pos), 1))
    _, s, v, _, _ = run(par, loc, ib, (pos, jt, w))
    G, S = oracle.scan(par, loc, ib)
    assert np.array_equal(s.astype(np.float64), S)
    assert np.array_equal(v.astype(np.float64), oracle.skin_vertices(S, pos, jt, w))


def test_lbs_bind_pose_returns_rest_positions():
    # locals = the bind pose's locals -> S = I -> every vertex at its rest position
    par = hsgen.skeleton("hum64")
    bind_local = hsgen.local_poses(51, 64, 1)[0]
    G, _ = oracle.scan(par, bind_local[None])
    ib = np.empty((64, 3, 4), np.float32)
    for j in range(64):
        H = np.eye(4)
        H[:3] = G[0, j]
        ib[j] = np.linalg.inv(H)[:3].astype(np.float32)
    mesh = hsgen.mesh(52, par, 800)
    _, _, v, _, _ = run(par, np.repeat(bind_local[None], 3, 0), ib, mesh)
    assert np.abs(v - mesh[0][None].astype(np.float64)).max() < 1e-4


def test_lbs_errors():
    sk = hs.Skeleton(hsgen.skeleton("hum32"))
    pos, jt, w = hsgen.mesh(61, hsgen.skeleton("hum32"), 10)
    bad = jt.copy()
    bad[3, 2] = 32
    with pytest.raises(hs.HSError) as e:
        hs.Mesh(sk, pos, bad, w)
    assert e.value.status == hs.HS_ERR_OUT_OF_RANGE
    other = hs.Skeleton(hsgen.skeleton("hum64"))
    m_other = hs.Mesh(other, *hsgen.mesh(62, hsgen.skeleton("hum64"), 10))
    x = torch.zeros((2, 32, 3, 4), device="cuda")
    with pytest.raises(hs.HSError) as e:
        hs.scan_skin(sk, m_other, x)
    assert e.value.status == hs.HS_ERR_INVALID_ARG
    big = hs.Skeleton(hsgen.random_tree(9, 4096, 64))
    m_big = hs.Mesh(big, *hsgen.mesh(63, hsgen.random_tree(9, 4096, 64), 10))
    with pytest.raises(hs.HSError) as e:
        hs.scan_skin(big, m_big, torch.zeros((1, 4096, 3, 4), device="cuda"), mode="fused")
    assert e.value.status == hs.HS_ERR_UNSUPPORTED


def test_fused_and_two_pass_bitwise_equal():
    """Both placements run the same per-vertex code on the same skin palette; the
    two-pass path without skin_out batches through a 3-character workspace."""
    for name, n, V in (("hum64", 77, 900), ("tree1024", 9, 1500)):
        par = hsgen.skeleton(name)
        J = len(par)
        sk = hs.Skeleton(par, hsgen.inv_bind(71, J))
        m = hs.Mesh(sk, *hsgen.mesh(72, par, V))
        x = torch.from_numpy(hsgen.local_poses(73, J, n)).cuda()
        g1, s1, v1 = hs.scan_skin(sk, m, x, skin=True, mode="fused")
        g2, s2, v2 = hs.scan_skin(sk, m, x, skin=True, mode="two_pass")
        g3, _, v3 = hs.scan_skin(sk, m, x, skin=False, mode="two_pass", workspace_bytes=3 * J * 48)
        torch.cuda.synchronize()
        assert torch.equal(g1, g2) and torch.equal(s1, s2) and torch.equal(v1, v2)
        assert torch.equal(g1, g3) and torch.equal(v1, v3)


def test_two_pass_lbs_on_multi_cta_skeleton():
    par = hsgen.random_tree(81, 3000, 70)
    J = len(par)
    loc = hsgen.local_poses(82, J, 3)
    ib = hsgen.inv_bind(83, J)
    mesh = hsgen.mesh(84, par, 600)
    sk = hs.Skeleton(par, ib)
    assert sk.query("path") == hs.ALGO["tiles"]   # beyond one CTA (3 characters: the split path)
    _, s, v = hs.scan_skin(sk, hs.Mesh(sk, *mesh), torch.from_numpy(loc).cuda(), skin=True)
    torch.cuda.synchronize()
    G, S = oracle.scan(par, loc, ib)
    assert np.abs(v.cpu().numpy() - oracle.skin_vertices(S, *mesh)).max() <= TOL_VERTS


def test_full_pipeline_animate_then_skin_vertices():
    """The paper's whole GPU pipeline: Stage 1 -> scan -> bind (hs_animate),
    then skinning from the skin poses (hs_skin_vertices), against the fp64 oracles."""
    par = hsgen.skeleton("hum64")
    J = 64
    keys = hsgen.clips(91, J, 4, 13)
    lay = hsgen.layers(92, 40, 2, 4, 1.2)
    ib = hsgen.inv_bind(93, J)
    mesh = hsgen.mesh(94, par, 800)
    sk = hs.Skeleton(par, ib)
    cs = hs.ClipSet(sk, keys, 30.0, 1)
    m = hs.Mesh(sk, *mesh)
    g, s = hs.animate(sk, cs, lay)
    v = hs.skin_vertices(m, s)
    torch.cuda.synchronize()
    G, S = oracle.animate(par, keys, 30.0, 1, lay, ib)
    want = oracle.skin_vertices(S, *mesh)
    assert np.abs(v.cpu().numpy() - want).max() <= TOL_VERTS
    # and bitwise equal to the LBS of the GPU skin poses computed by hs_scan_skin's kernel
    x = torch.from_numpy(np.ascontiguousarray(
        np.stack([oracle.animate(par, keys, 30.0, 1, lay[c:c + 1], None, return_local=True)[2][0]
                  for c in range(2)]).astype(np.float32))).cuda()
    _, s2, v2 = hs.scan_skin(sk, m, x, skin=True, mode="two_pass")
    v3 = hs.skin_vertices(m, s2)
    torch.cuda.synchronize()
    assert torch.equal(v2, v3)


def test_animate_skin_one_call_matches_two_calls():
    """hs_animate_skin (Stage 1 -> scan -> bind -> LBS in one call) equals hs_animate followed
    by the same skinning placement, bit for bit, and stays within the oracle bounds."""
    for name, V in (("hum64", 700), ("tree1024", 900)):
        par = hsgen.skeleton(name)
        J = len(par)
        keys = hsgen.clips(95, J, 3, 11)
        lay = hsgen.layers(96, 7, 2, 3, 1.0)
        ib = hsgen.inv_bind(97, J)
        mesh = hsgen.mesh(98, par, V)
        sk = hs.Skeleton(par, ib)
        cs = hs.ClipSet(sk, keys, 30.0, 1)
        m = hs.Mesh(sk, *mesh)
        g, s, v = hs.animate_skin(sk, cs, lay, m, skin=True)
        g2, s2 = hs.animate(sk, cs, lay)
        torch.cuda.synchronize()
        assert torch.equal(g, g2) and torch.equal(s, s2)
        G, S = oracle.animate(par, keys, 30.0, 1, lay, ib)
        assert np.abs(v.cpu().numpy() - oracle.skin_vertices(S, *mesh)).max() <= TOL_VERTS


def test_c5_full_size_lbs_sampled():
    """Scan + bind + LBS of a 1000-vertex mesh at C5's full size in bench.py
    --skin-mesh 1000's configuration (AUTO placement per type): sampled characters'
    vertices against the oracle's LBS of its own fp64 skin poses."""
    for name, n, seed, type_, ib_seed in hsgen.CONFIGS[5]:
        par = hsgen.skeleton(name)
        J = len(par)
        ib = hsgen.inv_bind(ib_seed, J)
        sk = hs.Skeleton(par, ib)
        mesh_np = hsgen.mesh(200 + type_, par, 1000, type_=type_)
        m = hs.Mesh(sk, *mesh_np)
        x = torch.empty((n, J, 3, 4), device="cuda")
        assert hsgen.lib_cuda().hsg_cuda_local_poses(seed, type_, J, 0, n, x.data_ptr(),
                                                     torch.cuda.current_stream().cuda_stream) == 0
        g, s, v = hs.scan_skin(sk, m, x, skin=True)
        torch.cuda.synchronize()
        idx = np.unique(np.r_[0, np.linspace(0, n - 1, 8).astype(np.int64), n - 1])
        host = x[idx].cpu().numpy()
        G, S = oracle.scan(par, host, ib)
        err = float(np.abs(v[idx].cpu().numpy() - oracle.skin_vertices(S, *mesh_np)).max())
        print(f"{name} x {n}: vertices sampled max err {err:.3e}")
        assert err <= TOL_VERTS
        del x, g, s, v
        torch.cuda.empty_cache()
