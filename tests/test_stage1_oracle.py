"""Pins for the Stage-1 oracle (oracle/stage1.c): SPEC worked
values for trs_to_matrix / sample_clip / blend (tests/golden/), closed forms and
invariants, and an independent numpy re-derivation of the quaternion rotation
(Hamilton product q v q*, not the matrix formula).  CPU only."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import hsgen
import oracle
from tests import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "spec_worked_values.json")))["stage1"]


def _qmul(a, b):
    w1, x1, y1, z1 = a
    w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def _rotate(q, v):
    qc = np.array([q[0], -q[1], -q[2], -q[3]])
    return _qmul(_qmul(q, np.array([0.0, *v])), qc)[1:]


def _keys(n_keys, J=1):
    k = np.zeros((n_keys, J, 10), np.float32)
    k[..., 3] = 1.0
    k[..., 7:] = 1.0
    return k


def test_golden_trs_to_matrix():
    for case in GOLD["trs_to_matrix"]:
        m = oracle.trs_to_matrix(case["trs"])
        if "expect" in case:
            assert np.array_equal(m, np.array(case["expect"], float)), case["cite"]
        if "expect_translation" in case:
            assert np.array_equal(m[:, 3], case["expect_translation"]), case["cite"]
        if "expect_upper_left" in case:
            assert np.allclose(m[:2, :2], case["expect_upper_left"], atol=1e-15), case["cite"]


def test_trs_matches_hamilton_product():
    """R(q) diag(s) applied to basis vectors == s_c * (q e_c q*), for random q and s."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        q = rng.normal(size=4); q /= np.linalg.norm(q)
        s = rng.uniform(0.5, 2, 3); t = rng.uniform(-1, 1, 3)
        m = oracle.trs_to_matrix(np.concatenate([t, q, s]))
        for c in range(3):
            e = np.zeros(3); e[c] = 1.0
            assert np.abs(m[:, c] - s[c] * _rotate(q, e)).max() < 1e-14
        assert np.array_equal(m[:, 3], t)


def test_golden_sample_clip():
    cases = GOLD["sample_clip"]
    # key time exact (bitwise), for several keys / joints, clamp and loop
    keys = hsgen.clips(3, 5, 1, 7)[0]
    for wrap in (0, 1):
        for k in range(6):
            for j in range(5):
                got = oracle.sample(keys, 2.0, wrap, k / 2.0, j)
                assert np.array_equal(got, keys[k, j].astype(np.float64)), cases[0]["cite"]
    c = cases[1]
    k = _keys(2); k[:, 0, 0] = c["keys_x"]
    assert oracle.sample(k, c["fps"], 0, c["t"], 0)[0] == c["expect_x"], c["cite"]
    c = cases[2]
    k = _keys(2); k[0, 0, 3:7] = c["q0"]; k[1, 0, 3:7] = c["q1"]
    q = oracle.sample(k, c["fps"], 0, c["t"], 0)[3:7]
    ang = np.degrees(2 * np.arctan2(q[3], q[0]))
    assert abs(ang - c["expect_angle_deg"]) < c["tol"], c["cite"]


def test_sample_shortest_arc_and_wrap():
    k = _keys(2)
    k[1, 0, 3:7] = [-1, 0, 0, 0]          # same rotation, opposite sign: no motion
    q = oracle.sample(k, 1.0, 0, 0.3, 0)[3:7]
    assert np.allclose(q, [1, 0, 0, 0], atol=1e-15)
    # loop: t + duration samples the same as t; clamp holds the ends
    keys = hsgen.clips(4, 3, 1, 9)[0]
    for t in (0.13, 0.77, 1.9):
        a = oracle.sample(keys, 4.0, 1, t, 2)
        b = oracle.sample(keys, 4.0, 1, t + 2.0, 2)   # duration = 8 / 4
        assert np.allclose(a, b, atol=1e-6)
    assert np.array_equal(oracle.sample(keys, 4.0, 0, 99.0, 1), keys[-1, 1].astype(np.float64))
    assert np.array_equal(oracle.sample(keys, 4.0, 0, -3.0, 1), keys[0, 1].astype(np.float64))


def test_golden_blend():
    rng = np.random.default_rng(2)
    P = np.concatenate([rng.uniform(-1, 1, 3), (lambda q: q / np.linalg.norm(q))(rng.normal(size=4)),
                        rng.uniform(0.5, 2, 3)])
    c = {x.get("case", "x"): x for x in GOLD["blend"]}
    assert np.array_equal(oracle.blend([P], [0.37]), P), c["single"]["cite"]
    assert np.abs(oracle.blend([P, P], [0.2, 0.9]) - P).max() < 1e-15, c["idempotent"]["cite"]
    x = c["x"]
    A = np.array([x["x"][0], 0, 0, 1, 0, 0, 0, 1, 1, 1.0])
    B = np.array([x["x"][1], 0, 0, 1, 0, 0, 0, 1, 1, 1.0])
    assert oracle.blend([A, B], x["weights"])[0] == x["expect_x"], x["cite"]


def test_blend_invariants():
    rng = np.random.default_rng(3)
    for _ in range(50):
        n = int(rng.integers(2, 6))
        P = np.concatenate([rng.uniform(-1, 1, (n, 3)), rng.normal(size=(n, 4)),
                            rng.uniform(0.5, 2, (n, 3))], axis=1)
        P[:, 3:7] /= np.linalg.norm(P[:, 3:7], axis=1, keepdims=True)
        w = rng.uniform(0.1, 1, n)
        a = oracle.blend(P, w)
        assert np.abs(oracle.blend(P, 7.5 * w) - a).max() < 1e-14        # weight scaling
        Q = P.copy(); Q[1:, 3:7] *= -1                                    # sign-aligned quats
        assert np.abs(oracle.blend(Q, w) - a).max() < 1e-14
        assert abs(np.linalg.norm(a[3:7]) - 1) < 1e-15


def test_animate_equals_stage1_then_brute_scan():
    """orc_animate's locals equal sample -> blend -> trs composed here from the pinned
    pieces; its globals equal the brute-force Eq. 1 recursion on those locals."""
    par = hsgen.skeleton("hum64")
    J = len(par)
    keys = hsgen.clips(5, J, 4, 11)
    lay = hsgen.layers(5, 6, 3, 4, 3.5)
    ib = hsgen.inv_bind(5, J)
    G, S, Lo = oracle.animate(par, keys, 3.0, 1, lay, ib, return_local=True)
    for c in range(6):
        for j in range(J):
            poses = [oracle.sample(keys[l["clip"]], 3.0, 1, l["time"], j) for l in lay[c]]
            m = oracle.trs_to_matrix(oracle.blend(poses, [l["weight"] for l in lay[c]]))
            assert np.array_equal(Lo[c, j], m)
        Gb = brute.global_pose(par, Lo[c])
        assert np.abs(G[c] - Gb[:, :3]).max() < 1e-12
        Sb = np.stack([Gb[i] @ brute.homog(ib[i]) for i in range(J)])
        assert np.abs(S[c] - Sb[:, :3]).max() < 1e-12


def test_single_layer_at_key_time_equals_key_pose():
    """One layer at an exact key time: Stage 1 yields the key's TRS matrix exactly."""
    par = hsgen.chain(16)
    keys = hsgen.clips(6, 16, 2, 5)
    lay = np.zeros((1, 1), oracle.LAYER_DTYPE)
    lay[0, 0] = (1, 3 / 2.0, 0.5, 0)     # key 3 at fps 2
    _, _, Lo = oracle.animate(par, keys, 2.0, 0, lay, return_local=True)
    for j in range(16):
        assert np.array_equal(Lo[0, j], oracle.trs_to_matrix(keys[1, 3, j].astype(np.float64)))
