"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Bar (BASELINE.json north_star): max |element| error <= 1e-4 for G and S on
rigid inputs with |t| <= 1, depth <= 1024; bitwise on the exact-arithmetic
family (every product exact in fp32) and on the cases with no multiply.
All inputs come from hsgen (host generator); expected values from oracle/.
"""
from __future__ import annotations

import numpy as np
import pytest

import hsgen
import oracle
from tests import brute

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2505_06703_b200 as hs  # noqa: E402

TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _built():
    hs.build()
    torch.cuda.init()


def gpu_scan(parents, local, ib=None, algo="auto", max_rounds=-1, skin=True, **create):
    sk = hs.Skeleton(parents, ib, **create)
    x = torch.from_numpy(np.ascontiguousarray(local)).cuda()
    g, s = sk.scan(x, algo=algo, max_rounds=max_rounds, skin=skin)
    torch.cuda.synchronize()
    out = g.cpu().numpy(), (s.cpu().numpy() if s is not None else None)
    sk.close()
    return out


def max_err(a, b):
    return float(np.abs(a.astype(np.float64) - b).max()) if a.size else 0.0


# ------------------------------------------------------------------ configs 1-4, full size
@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_config_parity_full(cfg):
    (name, n_chars, seed, type_, ib_seed), = hsgen.CONFIGS[cfg]
    par = hsgen.skeleton(name)
    J = len(par)
    local = hsgen.local_poses(seed, J, n_chars, type_=type_)
    ib = hsgen.inv_bind(ib_seed, J)
    g, s = gpu_scan(par, local, ib)
    G, S = oracle.scan(par, local, ib)
    eg, es = max_err(g, G), max_err(s, S)
    print(f"config {cfg} {name} x {n_chars}: max err global {eg:.3e} skin {es:.3e}")
    assert eg <= TOL and es <= TOL
    # the root's global equals its local bitwise (no multiply on a root)
    roots = np.where(par < 0)[0]
    assert np.array_equal(g[:, roots], local[:, roots])


# ------------------------------------------------------------------ exact family, every path
EXACT_CASES = [
    ("hum32", {}), ("hum64", {}), ("chain256", {}), ("tree1024", {}),
    ("hum64", {"chunk": 3}), ("chain256", {"chunk": 11}), ("tree1024", {"chunk": 5}),
    ("hum64", {"tile_joints": 200}), ("tree1024", {"stages": 2, "sbufs": 1}),
    ("tree1024", {"pbuf": 2}), ("chain256", {"pbuf": 1}), ("tree1024", {"pbuf": 1, "chunk": 9}),
    ("hum32", {"pbuf": 1, "stages": 3, "sbufs": 2}),
    ("tree1024", {"chunking": 1}), ("hum64", {"chunking": 1, "chunk": 7}),
    ("tree1024", {"force_split": True}), ("chain256", {"force_split": True, "chunk": 3}),
]


@pytest.mark.parametrize("name,create", EXACT_CASES)
def test_exact_family_bitwise(name, create):
    par = hsgen.skeleton(name)
    J = len(par)
    n_chars = 37  # ragged against every tile size
    local = hsgen.exact_poses(31, J, n_chars)
    ib = hsgen.exact_inv_bind(31, J)
    G, S = oracle.scan(par, local, ib)
    g, s = gpu_scan(par, local, ib, **create)
    assert np.array_equal(g, G) and np.array_equal(s, S)


@pytest.mark.parametrize("algo", ["doubling", "gateau", "leaf", "blocked", "compressed"])
@pytest.mark.parametrize("name", ["hum64", "chain256", "tree1024"])
def test_exact_family_comparison_algorithms(algo, name):
    par = hsgen.skeleton(name)
    J = len(par)
    local = hsgen.exact_poses(32, J, 9)
    ib = hsgen.exact_inv_bind(32, J)
    G, S = oracle.scan(par, local, ib)
    g, s = gpu_scan(par, local, ib, algo=algo)
    assert np.array_equal(g, G) and np.array_equal(s, S)


def test_permuted_labels():
    """Non-topological user order (forward parents): reordered internally."""
    base = hsgen.skeleton("tree1024")
    perm = hsgen.permutation(7, 1024)
    par, _ = hsgen.relabel(base, perm)
    assert hs.Plan(par).query("identity_order") == 0
    local = hsgen.exact_poses(33, 1024, 5)
    ib = hsgen.exact_inv_bind(33, 1024)
    G, S = oracle.scan(par, local, ib)
    for create in ({}, {"force_split": True}):
        g, s = gpu_scan(par, local, ib, **create)
        assert np.array_equal(g, G) and np.array_equal(s, S)
    # rigid inputs, tolerance, and equality with the unpermuted problem
    local = hsgen.local_poses(34, 1024, 50)
    g, _ = gpu_scan(par, local)
    G, _ = oracle.scan(par, local)
    assert max_err(g, G) <= TOL


@pytest.mark.parametrize("algo", ["tiles", "split"])
def test_large_skeleton_multi_cta_path(algo):
    """16,384-joint tree, L = 1024: beyond one CTA -> the multi-tile path (large crowds,
    HS_ALGO_TILES) or the split path (small crowds); both forced here on a few characters."""
    par = hsgen.skeleton("tree16384")
    sk = hs.Skeleton(par)
    assert sk.query("path") == hs.ALGO["tiles"]
    assert sk.query("seq_tiles") >= 16 and sk.query("split_levels") >= 1
    sk.close()
    local = hsgen.exact_poses(35, 16384, 3)
    ib = hsgen.exact_inv_bind(35, 16384)
    G, S = oracle.scan(par, local, ib)
    g, s = gpu_scan(par, local, ib, algo=algo)
    assert np.array_equal(g, G) and np.array_equal(s, S)
    # rigid |t| <= 1 locals and a rigid |t| <= 1 inverse bind: the north star's 1e-4
    # holds for depth <= 1024 (reading R16)
    local = hsgen.local_poses(36, 16384, 4)
    ib = hsgen.inv_bind(36, 16384)
    g, s = gpu_scan(par, local, ib, algo=algo)
    G, S = oracle.scan(par, local, ib)
    eg, es = max_err(g, G), max_err(s, S)
    print(f"16384-joint L=1024 tree ({algo}): max err global {eg:.3e} skin {es:.3e}")
    assert eg <= TOL and es <= TOL


@pytest.mark.parametrize("name", ["tree16384", "tree16384dfs"])
def test_multi_tile_crowd_auto_and_sampled_oracle(name):
    """A crowd larger than the SM count takes the multi-tile path under AUTO; every
    character equals the same character scanned alone (bitwise: one CTA runs a whole
    character, whatever the crowd); sampled characters within 1e-4 of the oracle.  The
    C6 tree in generation order and depth-first (C7: larger tiles, few imports)."""
    par = hsgen.skeleton(name)
    ib = hsgen.inv_bind(38, 16384)
    sk = hs.Skeleton(par, ib)
    n = 2 * torch.cuda.get_device_properties(0).multi_processor_count + 7
    x = torch.empty((n, 16384, 3, 4), device="cuda")
    assert hsgen.lib_cuda().hsg_cuda_local_poses(39, 0, 16384, 0, n, x.data_ptr(),
                                                 torch.cuda.current_stream().cuda_stream) == 0
    g, s = sk.scan(x)
    g2, s2 = torch.empty_like(x), torch.empty_like(x)
    sk.scan_into(x, g2, s2, algo="tiles")
    torch.cuda.synchronize()
    assert torch.equal(g, g2) and torch.equal(s, s2)
    idx = np.array([0, 1, n // 2, n - 1])
    for i in idx:   # alone == in the crowd
        ga, sa = sk.scan(x[i:i + 1].contiguous(), algo="tiles")
        assert torch.equal(ga[0], g[i]) and torch.equal(sa[0], s[i])
    loc = np.concatenate([hsgen.local_poses(39, 16384, 1, char0=int(i)) for i in idx])
    assert np.array_equal(loc, x[idx].cpu().numpy())
    G, S = oracle.scan(par, loc, ib)
    eg, es = max_err(g[idx].cpu().numpy(), G), max_err(s[idx].cpu().numpy(), S)
    print(f"multi-tile crowd of {n} x {name} (F = {sk.query('seq_tile_joints')}): sampled max err "
          f"global {eg:.3e} skin {es:.3e}")
    assert eg <= TOL and es <= TOL


MULTI_TILE_CASES = [
    ("tree1024", {"force_split": True}), ("chain256", {"force_split": True, "chunk": 3}),
    (("rt", 3000, 120), {}), (("rt", 3000, 120), {"tile_joints": 256}), (("rt", 3000, 120), {"chunking": 2}),
    (("rt", 5000, 2500), {"chunk": 7}), (("chain", 4000), {}), (("star", 2000), {}),
    (("perm", 2500, 200), {}),
]


def _skel(spec):
    if isinstance(spec, str):
        return hsgen.skeleton(spec)
    if spec[0] == "rt":
        return hsgen.random_tree(11, spec[1], spec[2])
    if spec[0] == "chain":
        return hsgen.chain(spec[1])
    if spec[0] == "star":
        return np.r_[-1, np.zeros(spec[1] - 1, np.int32)].astype(np.int32)
    base = hsgen.random_tree(12, spec[1], spec[2])
    return hsgen.relabel(base, hsgen.permutation(13, spec[1]))[0]


@pytest.mark.parametrize("spec,create", MULTI_TILE_CASES)
def test_multi_tile_exact_family_bitwise(spec, create):
    """The multi-tile kernel equals the oracle bit for bit on the exact family: chains
    (one import per tile), stars (every joint imports the root), deep random trees,
    small tiles, K = 3 / 7, heavy-path chunking, permuted labels (gathered TMA runs)."""
    par = _skel(spec)
    J = len(par)
    n_chars = 19
    local = hsgen.exact_poses(51, J, n_chars)
    ib = hsgen.exact_inv_bind(51, J)
    sk = hs.Skeleton(par, ib, **create)
    assert sk.query("seq_tiles") >= 1
    sk.close()
    G, S = oracle.scan(par, local, ib)
    g, s = gpu_scan(par, local, ib, algo="tiles", **create)
    assert np.array_equal(g, G) and np.array_equal(s, S)
    g, _ = gpu_scan(par, local, ib, algo="tiles", skin=False, **create)
    assert np.array_equal(g, G)


def test_forced_split_config4_rigid():
    """the multi-CTA path forced on config 4's skeleton at full size
    (20,000 x tree1024, rigid |t| <= 1 locals and inverse bind), against the oracle."""
    (name, n_chars, seed, type_, ib_seed), = hsgen.CONFIGS[4]
    par = hsgen.skeleton(name)
    local = hsgen.local_poses(seed, 1024, n_chars, type_=type_)
    ib = hsgen.inv_bind(ib_seed, 1024)
    sk = hs.Skeleton(par, ib, force_split=True)
    assert sk.query("path") == hs.ALGO["tiles"]
    x = torch.from_numpy(local).cuda()
    G, S = oracle.scan(par, local, ib)
    for algo in ("auto", "split"):   # auto: the multi-tile path (20,000 >= SM count)
        g, s = sk.scan(x, algo=algo)
        torch.cuda.synchronize()
        eg, es = max_err(g.cpu().numpy(), G), max_err(s.cpu().numpy(), S)
        print(f"forced multi-CTA ({algo}), C4 20,000 x tree1024: max err global {eg:.3e} skin {es:.3e}")
        assert eg <= TOL and es <= TOL
    sk.close()


def test_chain1024_stress():
    par = hsgen.chain(1024)
    local = hsgen.local_poses(37, 1024, 200)
    ib = hsgen.inv_bind(37, 1024)
    g, s = gpu_scan(par, local, ib)
    G, S = oracle.scan(par, local, ib)
    eg, es = max_err(g, G), max_err(s, S)
    print(f"chain1024 (|t|<=1 locals and IB): global {eg:.3e} skin {es:.3e}")
    assert eg <= TOL and es <= TOL


# ------------------------------------------------------------------ closed forms / degenerate
def test_identity_locals_bitwise():
    par = hsgen.skeleton("tree1024")
    I = np.zeros((3, 1024, 3, 4), np.float32)
    I[..., 0, 0] = I[..., 1, 1] = I[..., 2, 2] = 1
    ib = hsgen.inv_bind(4, 1024)
    g, s = gpu_scan(par, I, ib)
    assert np.array_equal(g, I) and np.array_equal(s, np.broadcast_to(ib, s.shape))


def test_dyadic_translation_chain_bitwise():
    J = 256
    rng = np.random.default_rng(3)
    t = rng.integers(-8, 9, size=(2, J, 3)) / 8.0
    local = np.zeros((2, J, 3, 4), np.float32)
    local[..., 0, 0] = local[..., 1, 1] = local[..., 2, 2] = 1
    local[..., 3] = t
    g, _ = gpu_scan(hsgen.chain(J), local)
    assert np.array_equal(g[..., 3], np.cumsum(t, axis=1))


@pytest.mark.parametrize("algo", ["auto", "doubling", "gateau", "leaf", "blocked", "compressed"])
def test_single_joint_and_all_roots(algo):
    for par in ([-1], [-1] * 10):
        local = hsgen.local_poses(40, len(par), 33)
        g, s = gpu_scan(par, local, algo=algo)
        assert np.array_equal(g, local) and np.array_equal(s, local)


def test_zero_characters_is_noop():
    sk = hs.Skeleton(hsgen.skeleton("hum32"))
    x = torch.zeros((0, 32, 3, 4), device="cuda")
    g, s = sk.scan(x)
    assert g.shape == (0, 32, 3, 4)


def test_global_only_mode():
    par = hsgen.skeleton("hum64")
    local = hsgen.exact_poses(41, 64, 20)
    g, s = gpu_scan(par, local, skin=False)
    assert s is None
    assert np.array_equal(g, oracle.scan(par, local)[0])


def test_bind_pose_gives_identity_skin():
    """SPEC.md:218 / Acceptance 6: model == bind pose -> skin == I (fp32 bound)."""
    for name in ("hum64", "tree1024"):
        par = hsgen.skeleton(name)
        J = len(par)
        bind_local = hsgen.local_poses(42, J, 1)
        Gb, _ = oracle.scan(par, bind_local)
        ib = np.stack([np.linalg.inv(brute.homog(m))[:3] for m in Gb[0]]).astype(np.float32)
        _, s = gpu_scan(par, bind_local, ib)
        I = np.zeros((3, 4)); I[0, 0] = I[1, 1] = I[2, 2] = 1
        e = max_err(s[0], np.broadcast_to(I, s[0].shape))
        print(f"{name} bind-pose skin vs I: {e:.3e}")
        assert e <= TOL


# ------------------------------------------------------------------ round induction (P6)
def test_doubling_round_induction():
    """after d rounds of Alg. 2 on a 64-chain, each joint equals the
    product of its 2^d nearest chain nodes (computed by the oracle on the sub-chain)."""
    J = 64
    local = hsgen.exact_poses(43, J, 1)
    assert hs.Plan(hsgen.chain(J)).query("rounds") == 6
    for d in range(0, 7):
        g, _ = gpu_scan(hsgen.chain(J), local, algo="doubling", max_rounds=d)
        for i in range(J):
            lo = max(0, i - (1 << d) + 1)
            sub, _ = oracle.scan(hsgen.chain(i - lo + 1), local[0, lo:i + 1])
            assert np.array_equal(g[0, i], sub[-1]), (d, i)


# ------------------------------------------------------------------ determinism / independence
def test_determinism_and_character_independence():
    par = hsgen.skeleton("tree1024")
    local = hsgen.local_poses(44, 1024, 64)
    g1, s1 = gpu_scan(par, local)
    g2, s2 = gpu_scan(par, local)
    assert np.array_equal(g1, g2) and np.array_equal(s1, s2)
    g3, s3 = gpu_scan(par, local[17:18])
    assert np.array_equal(g3[0], g1[17]) and np.array_equal(s3[0], s1[17])
    par = hsgen.skeleton("hum64")
    local = hsgen.local_poses(45, 64, 100)
    ga, _ = gpu_scan(par, local)
    gb, _ = gpu_scan(par, local[50:])
    assert np.array_equal(ga[50:], gb)


@pytest.mark.parametrize("batch_chars", [700, 5000])   # fixed batches / the 8 MB ramp (682, 1364, ...)
def test_host_pipeline_matches_device_path(batch_chars):
    par = hsgen.skeleton("chain256")
    ib = hsgen.inv_bind(3, 256)
    local = hsgen.local_poses(46, 256, 3000)
    g_dev, s_dev = gpu_scan(par, local, ib)
    sk = hs.Skeleton(par, ib)
    pl = hs.Pipeline(batch_bytes=256 * 48 * batch_chars)  # several batches + a ragged one
    hl = torch.from_numpy(local).pin_memory()
    hg = torch.empty_like(hl).pin_memory()
    hsk = torch.empty_like(hl).pin_memory()
    pl.scan_host(sk, hl, hg, hsk)
    assert np.array_equal(hg.numpy(), g_dev) and np.array_equal(hsk.numpy(), s_dev)


def test_host_pipeline_batch_over_types():
    items, want = [], []
    for name, n in (("hum64", 900), ("chain256", 300), ("tree1024", 40)):
        par = hsgen.skeleton(name)
        J = len(par)
        ib = hsgen.inv_bind(5, J)
        local = hsgen.local_poses(47, J, n)
        want.append(gpu_scan(par, local, ib))
        hl = torch.from_numpy(local).pin_memory()
        items.append((hs.Skeleton(par, ib), hl, torch.empty_like(hl).pin_memory(),
                      torch.empty_like(hl).pin_memory()))
    pl = hs.Pipeline(batch_bytes=1 << 20)
    pl.scan_host_batch(items)
    for (_, _, hg, hsk), (g, s) in zip(items, want):
        assert np.array_equal(hg.numpy(), g) and np.array_equal(hsk.numpy(), s)


# ------------------------------------------------------------------ ABI error behaviour
def test_abi_errors():
    sk = hs.Skeleton(hsgen.skeleton("hum32"))
    x = torch.zeros((4, 32, 3, 4), device="cuda")
    y = torch.zeros_like(x)
    with pytest.raises(hs.HSError) as e:
        sk.scan_into(x, x, y)
    assert e.value.status == hs.HS_ERR_INVALID_ARG
    with pytest.raises(hs.HSError) as e:
        sk.scan_into(x.data_ptr() + 4, y, None, n_chars=2)
    assert e.value.status == hs.HS_ERR_INVALID_ARG
    with pytest.raises(hs.HSError) as e:
        sk.scan_into(x, y, None, algo="split")
    assert e.value.status == hs.HS_ERR_UNSUPPORTED
    with pytest.raises(hs.HSError) as e:
        sk.scan_into(x, y, None, algo="chunked", max_rounds=2)
    assert e.value.status == hs.HS_ERR_INVALID_ARG
    for bad, code in (([], hs.HS_ERR_EMPTY), ([0], hs.HS_ERR_CYCLE), ([-1, 9], hs.HS_ERR_OUT_OF_RANGE)):
        with pytest.raises(hs.HSError) as e:
            hs.Skeleton(bad)
        assert e.value.status == code


# ------------------------------------------------------------------ Fig. 7 shape (NEXT-2)
def test_fig7_shape_depth_sweep():
    """The Fig. 7 sweep's cells at depth 15 / 60 / 120: every
    algorithm within 1e-4 of the oracle on the same seeded inputs.  The timing side
    of the sweep is tools/fig7_sweep.py (not asserted here)."""
    import statistics
    res = {}
    for depth in (15, 60, 120):
        par = hsgen.random_tree(100 + depth, 300, depth)
        local = hsgen.local_poses(7, 300, 2000)
        x = torch.from_numpy(local).cuda()
        g, s = torch.empty_like(x), torch.empty_like(x)
        sk = hs.Skeleton(par)
        G, _ = oracle.scan(par, local[:8])
        for algo in ("auto", "gateau", "leaf", "doubling", "blocked", "compressed"):
            sk.scan_into(x, g, s, algo=algo)
            torch.cuda.synchronize()
            assert max_err(g[:8].cpu().numpy(), G) <= TOL
            ts = []
            for _ in range(7):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); sk.scan_into(x, g, s, algo=algo); e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[(depth, algo)] = statistics.median(ts)
        sk.close()
    # timings are printed, not asserted (a noisy box must not fail a parity gate); the
    # sweep with its timing claims is tools/fig7_sweep.py
    print(res)


def test_large_crowd_int64_offsets():
    """Buffers beyond 2^31 floats (9.2 GB each): characters near the end are addressed
    with 64-bit offsets on every path the kernel takes (TMA loads/stores, tiles)."""
    par = hsgen.skeleton("hum32")
    J, n = 32, 6_000_000                       # 6e6 x 32 x 12 floats = 2.3e9 > 2^31
    x = torch.empty((n, J, 3, 4), device="cuda")
    assert hsgen.lib_cuda().hsg_cuda_local_poses(91, 0, J, 0, n, x.data_ptr(),
                                                 torch.cuda.current_stream().cuda_stream) == 0
    ib = hsgen.inv_bind(92, J)
    sk = hs.Skeleton(par, ib)
    g, s = torch.empty_like(x), torch.empty_like(x)
    sk.scan_into(x, g, s)
    torch.cuda.synchronize()
    idx = np.array([0, 1, n // 2, n - 3, n - 2, n - 1])
    loc = np.concatenate([hsgen.local_poses(91, J, 1, char0=int(i)) for i in idx])
    assert np.array_equal(loc, x[idx].cpu().numpy())    # device generator == host generator
    G, S = oracle.scan(par, loc, ib)
    assert np.abs(g[idx].cpu().numpy() - G).max() <= TOL and np.abs(s[idx].cpu().numpy() - S).max() <= TOL
    del x, g, s
    torch.cuda.empty_cache()


def test_scan_and_animate_capture_into_a_cuda_graph():
    """Every launch goes onto the caller's stream with no host synchronisation, so a
    frame (hs_scan, and hs_animate with its stream-ordered workspace) can be captured
    once into a CUDA graph and replayed; replays equal the eager results bit for bit."""
    par = hsgen.skeleton("hum64")
    sk = hs.Skeleton(par, hsgen.inv_bind(5, 64))
    x = torch.from_numpy(hsgen.local_poses(6, 64, 300)).cuda()
    g_ref, s_ref = sk.scan(x)
    cs = hs.ClipSet(sk, hsgen.clips(7, 64, 3, 9), 30.0, 1)
    lay = torch.from_numpy(np.ascontiguousarray(hsgen.layers(8, 300, 2, 3, 1.0)).view(np.int32)
                           .reshape(300, 2, 4)).cuda()
    ga_ref, sa_ref = hs.animate(sk, cs, lay)
    g, s = torch.empty_like(x), torch.empty_like(x)
    ga, sa = torch.empty_like(x), torch.empty_like(x)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        sk.scan_into(x, g, s, stream=st)          # warm (first-use attributes, pool)
        hs.animate(sk, cs, lay, ga, sa, stream=st)
        st.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=st):
            sk.scan_into(x, g, s, stream=st)
            hs.animate(sk, cs, lay, ga, sa, stream=st)
    for t in (g, s, ga, sa):
        t.fill_(float("nan"))
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(g, g_ref) and torch.equal(s, s_ref)
    assert torch.equal(ga, ga_ref) and torch.equal(sa, sa_ref)


def test_c_client_runs():
    """examples/hs_demo.c: a plain C program using only the C ABI (skeleton, host-buffer
    pipeline, query) checks 1000 characters against its own float64 walk."""
    import subprocess

    import __graft_entry__ as ge
    out = ge.build_examples()
    r = subprocess.run([out], capture_output=True, text=True, timeout=120)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "max |err|" in r.stdout


def test_binding_rejects_bad_buffers_before_the_abi():
    """The binding checks what the C ABI cannot (pointer residency, dtype, contiguity,
    size) and raises before any kernel could touch a wrong buffer."""
    sk = hs.Skeleton(hsgen.skeleton("hum32"))
    x = torch.zeros((4, 32, 3, 4), device="cuda")
    g = torch.empty_like(x)
    with pytest.raises(TypeError):
        sk.scan_into(x.cpu(), g)                                   # host tensor as device input
    with pytest.raises(TypeError):
        sk.scan_into(x.double(), g)                                # wrong dtype
    with pytest.raises(ValueError):
        sk.scan_into(x, torch.empty((4, 32, 4, 3), device="cuda").transpose(2, 3))   # strided
    with pytest.raises(ValueError):
        sk.scan_into(x, g[:3])                                     # too small for n_chars = 4
    pl = hs.Pipeline(batch_bytes=1 << 20)
    with pytest.raises(TypeError):
        pl.scan_host(sk, x, x.cpu(), x.cpu())                      # device tensor as host input
    with pytest.raises(ValueError):
        pl.scan_host(sk, x.cpu(), np.empty((3, 32, 3, 4), np.float32), x.cpu())
    sk.scan_into(x, g)                                             # and the good call still works
    torch.cuda.synchronize()
    assert torch.equal(g, x)                                       # zero locals: roots stay zero
    pl.close()


def test_c5_full_size_sampled_parity():
    """C5 at BASELINE.json's full size (1,000,000 characters, 64.5 GB resident), in the
    launch configuration bench.py times (one hs_scan per type, device-generated
    inputs): sampled characters against the fp64 oracle (inputs regenerated on the
    host by the same counter RNG, and checked equal to the device generator's)."""
    worst = 0.0
    for name, n, seed, type_, ib_seed in hsgen.CONFIGS[5]:
        par = hsgen.skeleton(name)
        J = len(par)
        ib = hsgen.inv_bind(ib_seed, J)
        sk = hs.Skeleton(par, ib)
        x = torch.empty((n, J, 3, 4), device="cuda")
        assert hsgen.lib_cuda().hsg_cuda_local_poses(seed, type_, J, 0, n, x.data_ptr(),
                                                     torch.cuda.current_stream().cuda_stream) == 0
        g, s = torch.empty_like(x), torch.empty_like(x)
        sk.scan_into(x, g, s)
        torch.cuda.synchronize()
        idx = np.unique(np.r_[0, 1, np.linspace(0, n - 1, 14).astype(np.int64), n - 2, n - 1])
        host = np.concatenate([hsgen.local_poses(seed, J, 1, char0=int(c), type_=type_) for c in idx])
        assert np.array_equal(host, x[idx].cpu().numpy())
        G, S = oracle.scan(par, host, ib)
        eg = max_err(g[idx].cpu().numpy(), G)
        es = max_err(s[idx].cpu().numpy(), S)
        worst = max(worst, eg, es)
        del x, g, s
        torch.cuda.empty_cache()
    print(f"C5 sampled max err {worst:.3e}")
    assert worst <= TOL


@pytest.mark.parametrize("name", ["hum32", "hum64", "chain256"])
def test_small_crowd_program_is_bitwise_the_default(name):
    """Small crowds run a second program with smaller tiles (more CTAs busy); it keeps
    every character's chunks, so a character's result does not depend on the crowd it
    is scanned in: 1,000 / 37 / 1 characters alone equal the same characters inside a
    20,000-character crowd, bit for bit."""
    par = hsgen.skeleton(name)
    J = len(par)
    sk = hs.Skeleton(par, hsgen.inv_bind(61, J))
    assert 2 <= sk.query("small_tile_chars") < sk.query("tile_chars")
    x = torch.from_numpy(hsgen.local_poses(62, J, 20_000)).cuda()
    g_big, s_big = sk.scan(x)
    for lo, n in ((0, 1000), (4321, 37), (19_999, 1)):
        g, s = sk.scan(x[lo:lo + n].contiguous())
        assert torch.equal(g, g_big[lo:lo + n]) and torch.equal(s, s_big[lo:lo + n])
    torch.cuda.synchronize()
