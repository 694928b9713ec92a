"""Pins for the LBS oracle (oracle/lbs.c, R24), each
from an independent formula: identity palette, single influence == the homogeneous
4x4 matrix-vector product (numpy), translation-only palette closed form, linearity
in the weights, rigid single influence preserves distances.  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

import hsgen
import oracle


def _rot(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def _palette(rng, n, J, rigid=True):
    S = np.zeros((n, J, 3, 4))
    for c in range(n):
        for j in range(J):
            S[c, j, :, :3] = _rot(rng) if rigid else rng.normal(size=(3, 3))
            S[c, j, :, 3] = rng.uniform(-1, 1, 3)
    return S


def test_identity_palette_returns_weighted_rest_position():
    par = hsgen.skeleton("hum64")
    pos, jt, w = hsgen.mesh(3, par, 500)
    S = np.zeros((2, 64, 3, 4))
    S[..., 0, 0] = S[..., 1, 1] = S[..., 2, 2] = 1.0
    out = oracle.skin_vertices(S, pos, jt, w)
    want = pos.astype(np.float64) * w.astype(np.float64).sum(1, keepdims=True)
    assert np.abs(out - want[None]).max() < 1e-15


def test_single_influence_is_homogeneous_matvec():
    rng = np.random.default_rng(1)
    J, V = 10, 200
    S = _palette(rng, 3, J, rigid=False)
    pos = rng.uniform(-1, 1, (V, 3)).astype(np.float32)
    jt = rng.integers(0, J, (V, 4)).astype(np.int32)
    w = np.zeros((V, 4), np.float32)
    w[:, 0] = 1.0
    out = oracle.skin_vertices(S, pos, jt, w)
    H = np.zeros((3, J, 4, 4))
    H[:, :, :3, :] = S
    H[:, :, 3, 3] = 1.0
    ph = np.concatenate([pos.astype(np.float64), np.ones((V, 1))], axis=1)
    want = np.einsum("cvab,vb->cva", H[:, jt[:, 0]], ph)[..., :3]
    assert np.abs(out - want).max() < 1e-13


def test_translation_palette_closed_form():
    rng = np.random.default_rng(2)
    J, V = 7, 300
    S = np.zeros((1, J, 3, 4))
    S[..., 0, 0] = S[..., 1, 1] = S[..., 2, 2] = 1.0
    S[..., 3] = rng.uniform(-1, 1, (1, J, 3))
    pos, jt, w = hsgen.mesh(5, np.arange(-1, J - 1), V)
    out = oracle.skin_vertices(S, pos, jt, w)[0]
    wd = w.astype(np.float64)
    want = pos * wd.sum(1, keepdims=True) + np.einsum("vk,vkr->vr", wd, S[0, jt, :, 3])
    assert np.abs(out - want).max() < 1e-14


def test_linear_in_weights_and_rigid_distances():
    rng = np.random.default_rng(3)
    J, V = 12, 100
    S = _palette(rng, 2, J)
    pos = rng.uniform(-1, 1, (V, 3)).astype(np.float32)
    jt = rng.integers(0, J, (V, 4)).astype(np.int32)
    w1 = rng.uniform(0, 1, (V, 4)).astype(np.float32)
    w2 = rng.uniform(0, 1, (V, 4)).astype(np.float32)
    a = oracle.skin_vertices(S, pos, jt, w1)
    b = oracle.skin_vertices(S, pos, jt, w2)
    ab = oracle.skin_vertices(S, pos, jt, w1 + w2)
    assert np.abs(ab - (a + b)).max() < 1e-6          # w1 + w2 is rounded once to fp32
    # a single rigid influence keeps pairwise distances between vertices on that joint
    jt1 = np.zeros((V, 4), np.int32)
    w = np.zeros((V, 4), np.float32)
    w[:, 0] = 1
    out = oracle.skin_vertices(S, pos, jt1, w)[0]
    d0 = np.linalg.norm(pos[:, None].astype(np.float64) - pos[None], axis=-1)
    d1 = np.linalg.norm(out[:, None] - out[None], axis=-1)
    assert np.abs(d0 - d1).max() < 1e-12


def test_bad_joint_index_rejected():
    pos = np.zeros((1, 3), np.float32)
    with pytest.raises(oracle.OracleError):
        oracle.skin_vertices(np.zeros((4, 3, 4)), pos, np.array([[0, 1, 2, 4]], np.int32),
                             np.ones((1, 4), np.float32))
