"""GPU parity of the fused Stage-1 prologue (hs_animate) against
the fp64 oracle (oracle.animate): sampling, blending, TRS, then scan + bind."""
from __future__ import annotations

import numpy as np
import pytest

import hsgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2505_06703_b200 as hs  # noqa: E402

TOL = 1e-4


def stage1_tol(L):
    """End-to-end bound with Stage 1: the north-star 1e-4 at every depth.
    Stage 1 computes each local pose in fp64 and rounds it once to fp32 (the measured
    budget, tests/test_gpu_stage1_budget.py: fp32 Stage-1 arithmetic put 4e-7 rotation
    errors into every local pose, 1.5e-4 after 256 levels; correctly rounded locals carry
    5e-6), so the scan's own bound applies unchanged."""
    return TOL


def levels(par):
    lev = np.zeros(len(par), int)
    for i in hsgen_order(par):
        lev[i] = 1 if par[i] < 0 else lev[par[i]] + 1
    return int(lev.max())


def hsgen_order(par):
    return oracle.kahn_order(par)


def run(par, keys, fps, wrap, lay, ib=None, mode="auto", **create):
    sk = hs.Skeleton(par, ib, **create)
    cs = hs.ClipSet(sk, keys, fps, wrap)
    g, s = hs.animate(sk, cs, lay, mode=mode)
    torch.cuda.synchronize()
    return g.cpu().numpy(), s.cpu().numpy()


@pytest.mark.parametrize("name,n_layers,wrap", [("hum64", 2, 1), ("chain256", 3, 0),
                                                ("tree1024", 2, 1), ("hum32", 1, 1),
                                                ("tree1024", 1, 0)])
@pytest.mark.parametrize("mode", ["fused", "two_pass"])
def test_animate_parity(name, n_layers, wrap, mode):
    par = hsgen.skeleton(name)
    J = len(par)
    keys = hsgen.clips(11, J, 4, 31)
    lay = hsgen.layers(11, 97, n_layers, 4, 1.6)     # times beyond the 1 s duration: wrap
    ib = hsgen.inv_bind(11, J)
    g, s = run(par, keys, 30.0, wrap, lay, ib, mode=mode)
    G, S = oracle.animate(par, keys, 30.0, wrap, lay, ib)
    eg, es = float(np.abs(g - G).max()), float(np.abs(s - S).max())
    tol = stage1_tol(levels(par))
    print(f"{name} layers={n_layers} wrap={wrap}: global {eg:.2e} skin {es:.2e} (tol {tol:.1e})")
    assert eg <= tol and es <= tol


@pytest.mark.parametrize("n_layers", [1, 2, 3])
def test_stage1_local_poses(n_layers):
    """An all-roots skeleton returns the Stage-1 local poses themselves (G = L): they
    match the oracle's fp64 locals to fp32 rounding."""
    J = 256
    par = np.full(J, -1, np.int32)
    keys = hsgen.clips(14, J, 3, 17, scale=(0.8, 1.25))
    lay = hsgen.layers(14, 64, n_layers, 3, 1.3)
    g, _ = run(par, keys, 16.0, 1, lay)
    _, _, Lo = oracle.animate(par, keys, 16.0, 1, lay, return_local=True)
    e = float(np.abs(g - Lo).max())
    print(f"stage-1 locals, {n_layers} layers: max err {e:.2e}")
    # fp64 arithmetic rounded once: within half an fp32 ulp of the oracle's locals
    # (|entries| <= 1.25: ulp 2^-23 at most), up to the fp64 rounding itself
    assert e <= 2 ** -24 * 1.25 * (1 + 1e-9)


def test_animate_key_times_bitwise_on_exact_keys():
    """One layer at exact key times on exact-family keys: Stage 1 returns the key's TRS
    matrix and every product is exact -> bitwise equal to the oracle."""
    par = hsgen.skeleton("tree1024")
    J = len(par)
    keys = np.zeros((2, 5, J, 10), np.float32)
    keys[..., 7:] = 1.0
    rng = np.random.default_rng(5)
    quats = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 1, 0], [0, 0, 0, 1]], np.float32)
    keys[..., 3:7] = quats[rng.integers(0, 4, size=keys.shape[:3])]
    keys[..., :3] = rng.integers(-1, 2, size=keys.shape[:3] + (3,))
    lay = np.zeros((40, 1), hs.LAYER_DTYPE)
    lay["clip"][:, 0] = rng.integers(0, 2, 40)
    lay["time"][:, 0] = rng.integers(0, 5, 40) / 4.0
    lay["weight"][:, 0] = 1.0
    g, s = run(par, keys, 4.0, 0, lay)
    G, S = oracle.animate(par, keys, 4.0, 0, lay)
    assert np.array_equal(g, G) and np.array_equal(s, S)


def test_animate_scaled_shallow_skeleton():
    par = hsgen.skeleton("hum32")
    keys = hsgen.clips(12, 32, 3, 9, scale=(0.8, 1.25))
    lay = hsgen.layers(12, 50, 3, 3, 0.7)
    g, s = run(par, keys, 10.0, 1, lay)
    G, S = oracle.animate(par, keys, 10.0, 1, lay)
    e = max(float(np.abs(g - G).max()), float(np.abs(s - S).max()))
    print(f"hum32 with scales 0.8-1.25: max err {e:.2e} (max |G| {np.abs(G).max():.1f})")
    assert e <= TOL


def test_animate_equals_scan_of_oracle_locals_chunk_variants():
    """Same bits whatever chunking / K the skeleton uses (Stage 1 is per joint)."""
    par = hsgen.skeleton("hum64")
    keys = hsgen.clips(13, 64, 2, 7)
    lay = hsgen.layers(13, 33, 2, 2, 0.5)
    outs = [run(par, keys, 12.0, 1, lay, chunk=k, chunking=c)[0] for k, c in ((5, 1), (7, 2), (3, 3))]
    G, _ = oracle.animate(par, keys, 12.0, 1, lay)
    for g in outs:
        assert float(np.abs(g - G).max()) <= stage1_tol(12)


def test_animate_errors():
    sk = hs.Skeleton(hsgen.skeleton("hum32"))
    cs = hs.ClipSet(sk, hsgen.clips(1, 32, 1, 3), 10.0, 1)
    lay = torch.zeros((4, 9, 4), dtype=torch.int32, device="cuda")
    with pytest.raises(hs.HSError) as e:
        hs.animate(sk, cs, lay)            # 9 layers > 8
    assert e.value.status == hs.HS_ERR_INVALID_ARG
    other = hs.Skeleton(hsgen.skeleton("hum64"))
    with pytest.raises(hs.HSError):
        hs.animate(other, cs, torch.zeros((4, 1, 4), dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("name,n_layers", [("hum64", 3), ("chain256", 1), ("tree1024", 2)])
def test_fused_and_two_pass_bitwise_equal(name, n_layers):
    """Both Stage-1 placements compute the same local poses (same device code) and the
    same scan, so they agree bit for bit; a 3-character workspace forces many batches."""
    par = hsgen.skeleton(name)
    J = len(par)
    keys = hsgen.clips(9, J, 4, 17)
    lay = hsgen.layers(10, 101, n_layers, 4, 2.0)
    sk = hs.Skeleton(par, hsgen.inv_bind(11, J))
    cs = hs.ClipSet(sk, keys, 24.0, 1)
    g1, s1 = hs.animate(sk, cs, lay, mode="fused")
    g2, s2 = hs.animate(sk, cs, lay, mode="two_pass", workspace_bytes=3 * J * 48)
    g3, s3 = hs.animate(sk, cs, lay)
    torch.cuda.synchronize()
    assert torch.equal(g1, g2) and torch.equal(s1, s2) and torch.equal(g1, g3) and torch.equal(s1, s3)


def test_animate_opts_errors():
    sk = hs.Skeleton(hsgen.skeleton("hum32"))
    cs = hs.ClipSet(sk, hsgen.clips(1, 32, 1, 3), 10.0, 1)
    lay = torch.zeros((4, 1, 4), dtype=torch.int32, device="cuda")
    for bad in (dict(mode="fused", workspace_bytes=-1),):
        with pytest.raises(hs.HSError) as e:
            hs.animate(sk, cs, lay, **bad)
        assert e.value.status == hs.HS_ERR_INVALID_ARG


def test_two_pass_on_multi_cta_skeleton():
    """The two-pass placement feeds any skeleton, including the multi-CTA path (the
    fused prologue needs one CTA and says so)."""
    par = hsgen.random_tree(21, 3000, 80)
    J = len(par)
    keys = hsgen.clips(22, J, 3, 9)
    lay = hsgen.layers(23, 5, 2, 3, 1.0)
    ib = hsgen.inv_bind(24, J)
    sk = hs.Skeleton(par, ib)
    assert sk.query("path") == hs.ALGO["tiles"]   # beyond one CTA (5 characters: the split path)
    cs = hs.ClipSet(sk, keys, 30.0, 1)
    g, s = hs.animate(sk, cs, lay)
    torch.cuda.synchronize()
    G, S = oracle.animate(par, keys, 30.0, 1, lay, ib)
    tol = stage1_tol(levels(par))
    assert np.abs(g.cpu().numpy() - G).max() <= tol and np.abs(s.cpu().numpy() - S).max() <= tol
    with pytest.raises(hs.HSError) as e:
        hs.animate(sk, cs, lay, mode="fused")
    assert e.value.status == hs.HS_ERR_UNSUPPORTED


@pytest.mark.parametrize("name,n", [("hum64", 5000), ("tree1024", 300)])
def test_animate_host_pipeline(name, n):
    """hs_animate_host (host layers in, host poses out, batched over 3 streams with a small
    pipeline so many batches run) equals hs_animate on the device bit for bit, and the
    oracle within the Stage-1 bound on sampled characters."""
    par = hsgen.skeleton(name)
    J = len(par)
    keys = hsgen.clips(31, J, 4, 15)
    lay = hsgen.layers(32, n, 2, 4, 1.5)
    ib = hsgen.inv_bind(33, J)
    sk = hs.Skeleton(par, ib)
    cs = hs.ClipSet(sk, keys, 30.0, 1)
    hl = torch.from_numpy(np.ascontiguousarray(lay).view(np.int32).reshape(n, 2, 4)).pin_memory()
    hg = torch.full((n, J, 3, 4), float("nan"), pin_memory=True)
    hsk = torch.full_like(hg, float("nan"), pin_memory=True)
    pl = hs.Pipeline(batch_bytes=2 << 20)
    pl.animate_host(sk, cs, hl, hg, hsk)
    g, s = hs.animate(sk, cs, lay)
    torch.cuda.synchronize()
    assert torch.equal(hg, g.cpu()) and torch.equal(hsk, s.cpu())
    # a numpy LAYER_DTYPE array works as the host buffer too
    hg2, hs2 = np.empty((n, J, 3, 4), np.float32), np.empty((n, J, 3, 4), np.float32)
    pl.animate_host(sk, cs, np.ascontiguousarray(lay), hg2, hs2)
    assert np.array_equal(hg2, hg.numpy()) and np.array_equal(hs2, hsk.numpy())
    idx = np.linspace(0, n - 1, 7).astype(int)
    G, S = oracle.animate(par, keys, 30.0, 1, lay[idx], ib)
    tol = stage1_tol(levels(par))
    assert np.abs(hg.numpy()[idx] - G).max() <= tol and np.abs(hsk.numpy()[idx] - S).max() <= tol
    with pytest.raises(hs.HSError) as e:
        pl.animate_host(sk, cs, hl[:, :0], hg, hsk)
    assert e.value.status == hs.HS_ERR_INVALID_ARG
    pl.close()


def test_workspace_trim_releases_the_pool():
    """The two-pass workspace pool keeps its memory between calls (no per-frame driver
    allocation) until hs_workspace_trim hands the unused part back."""
    par = hsgen.skeleton("hum64")
    sk = hs.Skeleton(par, hsgen.inv_bind(41, 64))
    cs = hs.ClipSet(sk, hsgen.clips(42, 64, 2, 5), 30.0, 1)
    lay = hsgen.layers(43, 5000, 1, 2, 1.0)
    g1, s1 = hs.animate(sk, cs, lay, mode="two_pass")
    torch.cuda.synchronize()
    assert hs.workspace_trim() == 0          # nothing outstanding: everything released
    g2, s2 = hs.animate(sk, cs, lay, mode="two_pass")   # the pool grows again on demand
    torch.cuda.synchronize()
    assert torch.equal(g1, g2) and torch.equal(s1, s2)
    assert hs.workspace_trim() == 0


def test_c5_full_size_stage1_sampled():
    """Stage 1 + scan + bind at C5's full size in bench.py --stage1's configuration (8
    clips of 31 keys per type, 2 layers, two-pass placement): sampled characters
    against the fp64 oracle, within the Stage-1 bound of each skeleton's depth."""
    for name, n, seed, type_, ib_seed in hsgen.CONFIGS[5]:
        par = hsgen.skeleton(name)
        J = len(par)
        ib = hsgen.inv_bind(ib_seed, J)
        keys = hsgen.clips(100 + type_, J, 8, 31, type_=type_)
        lay = hsgen.layers(seed, n, 2, 8, 1.5, type_=type_)
        sk = hs.Skeleton(par, ib)
        cs = hs.ClipSet(sk, keys, 30.0, 1)
        g, s = hs.animate(sk, cs, lay)
        torch.cuda.synchronize()
        idx = np.unique(np.r_[0, np.linspace(0, n - 1, 10).astype(np.int64), n - 1])
        G, S = oracle.animate(par, keys, 30.0, 1, lay[idx], ib)
        tol = stage1_tol(levels(par))
        eg = float(np.abs(g[idx].cpu().numpy() - G).max())
        es = float(np.abs(s[idx].cpu().numpy() - S).max())
        print(f"{name} x {n}: Stage-1 sampled max err {max(eg, es):.3e} (bound {tol:.1e})")
        assert eg <= tol and es <= tol
        del g, s
        torch.cuda.empty_cache()


def test_one_joint_eight_layers_two_pass():
    """a one-joint skeleton with 8 layers puts 2048 characters x 8 layer
    descriptors (256 KB) in one block-tile of the streaming kernel; the launcher shrinks
    the block-tile to fit shared memory.  G = L (a root), against the fp64 oracle."""
    par = np.array([-1], np.int32)
    keys = hsgen.clips(81, 1, 4, 9)
    lay = hsgen.layers(82, 5000, 8, 4, 1.3)
    g, s = run(par, keys, 8.0, 1, lay, mode="two_pass")
    G, S = oracle.animate(par, keys, 8.0, 1, lay)
    e = max(float(np.abs(g - G).max()), float(np.abs(s - S).max()))
    print(f"one joint, 8 layers: max err {e:.2e}")
    assert e <= 2 ** -24 * (1 + 1e-9)
