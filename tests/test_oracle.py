"""Pins for the fp64 oracle.

Nothing here re-types the oracle's formula: each test checks the oracle against
something fixed independently — brute-force Eq. 1 recursion on 4x4 homogeneous
matrices (tests/brute.py), closed forms (cumsum, summed angles, polylines),
Cayley's formula, SPEC worked values (tests/golden/), numpy's multi_dot, and
invariants.  CPU only.
"""
from __future__ import annotations

import functools
import itertools
import json
import os

import numpy as np
import pytest

import hsgen
import oracle
from tests import brute

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                     "spec_worked_values.json")))
I34 = np.hstack([np.eye(3), np.zeros((3, 1))])


def _rng_affine(rng, n, rigid=False):
    if rigid:
        q = rng.normal(size=(n, 4))
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        w, x, y, z = q.T
        R = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                      2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                      2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
                     axis=1).reshape(n, 3, 3)
    else:
        R = rng.uniform(-1, 1, size=(n, 3, 3))
    t = rng.uniform(-1, 1, size=(n, 3, 1))
    return np.concatenate([R, t], axis=2).astype(np.float32)


def _all_parent_arrays(n):
    return np.array(list(itertools.product(range(-1, n), repeat=n)), dtype=np.int32)


def _vectorised_is_forest(P):
    M, n = P.shape
    v = np.tile(np.arange(n), (M, 1))
    rows = np.arange(M)[:, None]
    for _ in range(n):
        nxt = np.where(v >= 0, P[rows, np.maximum(v, 0)], -1)
        v = nxt
    return np.all(v == -1, axis=1)


# ---------------------------------------------------------------- P1 brute force
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_validate_all_parent_arrays_and_cayley(n):
    """Every candidate parent array with entries in {-1..n-1}: the oracle's
    validator agrees with the brute-force root walk, and the number of valid ones
    is Cayley's count of labelled rooted forests, (n+1)^(n-1)."""
    P = _all_parent_arrays(n)
    assert len(P) == (n + 1) ** n
    forest = _vectorised_is_forest(P)
    assert forest.sum() == (n + 1) ** (n - 1)
    got = np.array([oracle.validate(p) == "ok" for p in P])
    assert np.array_equal(got, forest)
    assert all(oracle.validate(p) == "cycle" for p in P[~forest][:200])


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_oracle_equals_brute_force_on_every_forest(n):
    """All (n+1)^(n-1) forests with n <= 6: oracle == brute-force Eq. 1 within 1e-12."""
    rng = np.random.default_rng(100 + n)
    P = _all_parent_arrays(n)
    P = P[_vectorised_is_forest(P)]
    worst = 0.0
    for p in P:
        local = _rng_affine(rng, n)
        ib = _rng_affine(rng, n)
        g, s = oracle.scan(p, local, ib, nthreads=1)
        G = brute.global_pose(p, local)
        S = np.stack([G[i] @ brute.homog(ib[i]) for i in range(n)])
        worst = max(worst, np.abs(g - G[:, :3, :]).max(), np.abs(s - S[:, :3, :]).max())
    assert worst < 1e-12, worst


def test_oracle_equals_root_path_product_random_trees():
    """Random trees up to 64 joints (random labels): oracle vs Eq. 1 root-path product."""
    rng = np.random.default_rng(7)
    for trial in range(40):
        n = int(rng.integers(1, 65))
        parents = np.full(n, -1, np.int32)
        for i in range(1, n):
            parents[i] = rng.integers(-1 if rng.random() < 0.05 else 0, i)
        perm = rng.permutation(n).astype(np.int32)
        parents, _ = hsgen.relabel(parents, perm)
        local = _rng_affine(rng, n, rigid=bool(trial % 2))
        g, _ = oracle.scan(parents, local, nthreads=1)
        for i in range(n):
            assert np.abs(g[i] - brute.root_path_product(parents, local, i)[:3]).max() < 1e-12


# ---------------------------------------------------------------- P2 closed forms
def test_identity_locals_give_identity_and_inv_bind_bitwise():
    parents = hsgen.skeleton("tree1024")
    local = np.broadcast_to(I34.astype(np.float32), (2, 1024, 3, 4)).copy()
    ib = hsgen.inv_bind(4, 1024)
    g, s = oracle.scan(parents, local, ib)
    assert np.array_equal(g, np.broadcast_to(I34, g.shape))
    assert np.array_equal(s, np.broadcast_to(ib.astype(np.float64), s.shape))


def test_dyadic_translation_chain_is_cumsum_bitwise():
    """Pure-translation chain with translations in multiples of 1/8: exact prefix sums."""
    rng = np.random.default_rng(3)
    J = 300
    t = rng.integers(-8, 9, size=(J, 3)) / 8.0
    local = np.broadcast_to(I34, (J, 3, 4)).astype(np.float32).copy()
    local[:, :, 3] = t
    g, s = oracle.scan(hsgen.chain(J), local)
    assert np.array_equal(g[:, :, 3], np.cumsum(t, axis=0))
    assert np.array_equal(g[:, :, :3], np.broadcast_to(np.eye(3), (J, 3, 3)))
    assert np.array_equal(s, g)  # identity inverse bind


def _rz(theta, scale=1.0):
    """scale * (2x2 rotation by theta) in the xy block, 1 on z."""
    c, s = scale * np.cos(theta), scale * np.sin(theta)
    return np.array([[c, -s, 0], [s, c, 0], [0, 0, 1.0]])


def test_z_rotation_chain_is_summed_angle():
    rng = np.random.default_rng(4)
    J = 256
    theta32 = rng.uniform(-np.pi, np.pi, J).astype(np.float32)
    local = np.zeros((J, 3, 4), np.float32)
    # the fp32 input matrices; the closed form uses the exact angle of each input
    local[:, 0, 0] = np.cos(theta32); local[:, 0, 1] = -np.sin(theta32)
    local[:, 1, 0] = np.sin(theta32); local[:, 1, 1] = np.cos(theta32)
    local[:, 2, 2] = 1
    ang = np.arctan2(local[:, 1, 0].astype(np.float64), local[:, 0, 0].astype(np.float64))
    scale = np.hypot(local[:, 1, 0].astype(np.float64), local[:, 0, 0].astype(np.float64))
    g, _ = oracle.scan(hsgen.chain(J), local)
    cum_ang, cum_scale = np.cumsum(ang), np.cumprod(scale)
    for i in range(J):
        assert np.abs(g[i, :, :3] - _rz(cum_ang[i], cum_scale[i])).max() < 1e-12
        assert np.all(g[i, :, 3] == 0)


def test_planar_chain_polyline():
    """z-rotations + xy-translations: t_i = sum_k Rz(sum_{m<k} theta_m) t_k."""
    rng = np.random.default_rng(5)
    J = 120
    th = rng.uniform(-1, 1, J)
    tr = np.zeros((J, 3)); tr[:, :2] = rng.uniform(-1, 1, (J, 2))
    local = np.zeros((J, 3, 4))
    for i in range(J):
        local[i, :, :3] = _rz(th[i]); local[i, :, 3] = tr[i]
    local = local.astype(np.float32)
    # closed form in the fp32-rounded inputs' own angles/translations
    ang = np.arctan2(local[:, 1, 0].astype(np.float64), local[:, 0, 0].astype(np.float64))
    sc = np.hypot(local[:, 1, 0].astype(np.float64), local[:, 0, 0].astype(np.float64))
    t64 = local[:, :, 3].astype(np.float64)
    g, _ = oracle.scan(hsgen.chain(J), local)
    pos = np.zeros(3); a = 0.0; s = 1.0
    for i in range(J):
        pos = pos + _rz(a, s) @ t64[i]
        a += ang[i]; s *= sc[i]
        assert np.abs(g[i, :, 3] - pos).max() < 1e-12
        assert np.abs(g[i, :, :3] - _rz(a, s)).max() < 1e-12


# ---------------------------------------------------------------- SPEC worked values
def _m(x):
    return I34.copy() if x == "identity" else np.array(x, np.float64)


def test_golden_compose():
    for case in GOLDEN["compose"]:
        c = oracle.compose(_m(case["a"]), _m(case["b"]))
        if "expect" in case:
            assert np.array_equal(c, _m(case["expect"])), case["cite"]
        else:
            origin = c @ np.array([0, 0, 0, 1.0])
            assert np.allclose(origin, case["expect_origin_maps_to"], atol=0), case["cite"]


def test_golden_scan():
    for case in GOLDEN["scan"]:
        p = np.array(case["parents"], np.int32)
        local = np.broadcast_to(_m(case["local_all"]), (len(p), 3, 4)).astype(np.float32)
        g, _ = oracle.scan(p, local)
        if "expect_tx" in case:
            assert np.array_equal(g[:, 0, 3], case["expect_tx"]), case["cite"]
        else:
            assert np.array_equal(g, np.broadcast_to(I34, g.shape)), case["cite"]


def test_golden_bind():
    cases = {c.get("case", "chain"): c for c in GOLDEN["bind"]}
    # model == bind pose -> skin identity (exact family keeps it bitwise)
    p = hsgen.skeleton("hum64")
    bind_local = hsgen.exact_poses(9, 64, 1)[0]
    gb, _ = oracle.scan(p, bind_local)
    ib = np.stack([np.linalg.inv(brute.homog(m))[:3] for m in gb]).astype(np.float32)
    _, s = oracle.scan(p, bind_local, ib)
    assert np.array_equal(s, np.broadcast_to(I34, s.shape)), cases["model_equals_bind"]["cite"]
    # identity inverse bind -> skin == model
    local = hsgen.local_poses(9, 64, 2)
    g, s = oracle.scan(p, local, None)
    assert np.array_equal(g, s), cases["identity_inverse_bind"]["cite"]
    # chain-3 rest pose + root translate(0,1,0) -> every skin == translate(0,1,0)
    c = cases["chain"]
    p3 = np.array(c["parents"], np.int32)
    rest = np.broadcast_to(_m(c["rest_local"]), (3, 3, 4)).astype(np.float32).copy()
    grest, _ = oracle.scan(p3, rest)
    ib3 = np.stack([np.linalg.inv(brute.homog(m))[:3] for m in grest]).astype(np.float32)
    moved = rest.copy()
    moved[0] = (brute.homog(_m(c["root_extra"])) @ brute.homog(rest[0]))[:3]
    _, s3 = oracle.scan(p3, moved, ib3)
    assert np.array_equal(s3, np.broadcast_to(_m(c["expect_skin_all"]), s3.shape)), c["cite"]


def test_golden_topology_validation():
    for case in GOLDEN["topology"]:
        st = oracle.validate(case["parents"]) if case["parents"] else "empty"
        if case["valid"]:
            assert st == "ok", case["cite"]
        else:
            assert st == case["error"], case["cite"]


def test_kahn_order_is_topological_bfs():
    for name in ("hum32", "hum64", "tree1024"):
        p = hsgen.skeleton(name)
        perm = hsgen.permutation(11, len(p))
        q, _ = hsgen.relabel(p, perm)
        order = oracle.kahn_order(q)
        assert sorted(order) == list(range(len(q)))
        pos = np.empty(len(q), int); pos[order] = np.arange(len(q))
        assert all(q[i] == -1 or pos[q[i]] < pos[i] for i in range(len(q)))
        lev = np.zeros(len(q), int)
        for i in order:
            lev[i] = 1 if q[i] < 0 else lev[q[i]] + 1
        assert np.all(np.diff(lev[order]) >= 0)  # BFS: levels non-decreasing


# ---------------------------------------------------------------- P3 exact family
def test_exact_family_bitwise_vs_brute():
    """Signed-permutation rotations, integer translations: every product is exact,
    so the oracle must equal the brute-force recursion bitwise."""
    for name in ("hum64", "tree1024"):
        p = hsgen.skeleton(name)
        J = len(p)
        local = hsgen.exact_poses(13, J, 3)
        ib = hsgen.exact_inv_bind(13, J)
        g, s = oracle.scan(p, local, ib)
        for c in range(3):
            G = brute.global_pose(p, local[c])
            assert np.array_equal(g[c], G[:, :3])
            S = np.einsum("jab,jbc->jac", G, np.stack([brute.homog(m) for m in ib]))
            assert np.array_equal(s[c], S[:, :3])


def test_exact_family_generator_properties():
    sp = hsgen.signed_perms()
    assert len({m.tobytes() for m in sp}) == 24
    assert np.allclose(np.linalg.det(sp.astype(np.float64)), 1.0)
    e = hsgen.exact_poses(1, 64, 10)
    assert set(np.unique(e[..., 3])) <= {-1.0, 0.0, 1.0}


# ---------------------------------------------------------------- P4 library case
def test_chain_equals_multi_dot():
    rng = np.random.default_rng(8)
    J = 256
    local = _rng_affine(rng, J, rigid=True)
    g, _ = oracle.scan(hsgen.chain(J), local)
    H = [brute.homog(m) for m in local]
    for i in (1, 2, 17, 128, 255):
        ref = np.linalg.multi_dot(H[: i + 1]) if i >= 2 else functools.reduce(np.matmul, H[: i + 1])
        assert np.abs(g[i] - ref[:3]).max() < 1e-12


# ---------------------------------------------------------------- P5 invariants
def test_root_global_equals_local_bitwise():
    p = hsgen.skeleton("hum64")
    local = hsgen.local_poses(2, 64, 4)
    g, _ = oracle.scan(p, local)
    assert np.array_equal(g[:, 0], local[:, 0].astype(np.float64))
    forest = np.full(10, -1, np.int32)
    loc = hsgen.local_poses(3, 10, 2)
    g, _ = oracle.scan(forest, loc)
    assert np.array_equal(g, loc.astype(np.float64))


def test_label_permutation_invariance_bitwise():
    p = hsgen.skeleton("tree1024")
    local = hsgen.local_poses(4, 1024, 2)
    ib = hsgen.inv_bind(4, 1024)
    g, s = oracle.scan(p, local, ib)
    perm = hsgen.permutation(5, 1024)
    q, _ = hsgen.relabel(p, perm)
    g2, s2 = oracle.scan(q, local[:, perm], ib[perm])
    assert np.array_equal(g2, g[:, perm]) and np.array_equal(s2, s[:, perm])


def test_forest_is_disjoint_union():
    a, b = hsgen.skeleton("hum32"), hsgen.chain(40)
    union = np.concatenate([a, np.where(b >= 0, b + 32, -1)]).astype(np.int32)
    la, lb = hsgen.local_poses(6, 32, 2), hsgen.local_poses(7, 40, 2)
    gu, _ = oracle.scan(union, np.concatenate([la, lb], axis=1))
    ga, _ = oracle.scan(a, la)
    gb, _ = oracle.scan(b, lb)
    assert np.array_equal(gu[:, :32], ga) and np.array_equal(gu[:, 32:], gb)


def test_local_recovery_from_globals():
    """G_parent^-1 G_i == L_i (rigid inputs) — the O(1)/joint check usable at any size."""
    p = hsgen.skeleton("tree1024")
    local = hsgen.local_poses(4, 1024, 1)
    g, _ = oracle.scan(p, local)
    g = g[0]
    for i in range(1, 1024):
        rec = np.linalg.inv(brute.homog(g[p[i]])) @ brute.homog(g[i])
        assert np.abs(rec[:3] - local[0, i]).max() < 1e-12


def test_threads_do_not_change_results():
    p = hsgen.skeleton("hum64")
    local = hsgen.local_poses(2, 64, 37)
    g1, s1 = oracle.scan(p, local, nthreads=1)
    g8, s8 = oracle.scan(p, local, nthreads=8)
    assert np.array_equal(g1, g8) and np.array_equal(s1, s8)
    cs = oracle.scan_discard(p, local, nthreads=3)
    assert np.isfinite(cs)


def test_errors():
    with pytest.raises(oracle.OracleError):
        oracle.scan([1, 0], np.zeros((2, 3, 4), np.float32))
    with pytest.raises(oracle.OracleError):
        oracle.scan([-1, 7], np.zeros((2, 3, 4), np.float32))
