"""fp64 CPU oracle for the Hierarchy-Scan + Bind MeshPose path (ctypes binding).

TEST INFRASTRUCTURE ONLY — only tests/, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this.
The product package ``paper_2505_06703_b200`` never imports it.

The arithmetic lives in ``oracle/oracle.c`` (see its header for the PAPER.md
passages it follows: §1 steps 2-3, Eq. 1, Alg. 1's parent-left update, Bind
MeshPose).  This module only marshals numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "stage1.c"), os.path.join(_HERE, "lbs.c")]

STATUS = {0: "ok", 2: "empty", 3: "out_of_range", 4: "cycle", 6: "nomem"}


def build(force: bool = False) -> str:
    """Compile oracle.c with -O2 -ffp-contract=off (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_SO) or any(os.path.getmtime(_SO) < os.path.getmtime(s)
                                                for s in _SRCS):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-shared",
               "-fPIC", "-pthread", "-o", _SO, *_SRCS, "-lm"]
        subprocess.run(cmd, check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.orc_validate.argtypes = [i32p, ctypes.c_int32]
        L.orc_validate.restype = ctypes.c_int
        L.orc_kahn_order.argtypes = [i32p, ctypes.c_int32, i32p]
        L.orc_kahn_order.restype = ctypes.c_int
        L.orc_compose.argtypes = [ctypes.c_void_p] * 3
        L.orc_compose.restype = None
        L.orc_scan.argtypes = [i32p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                               ctypes.POINTER(ctypes.c_double)]
        L.orc_scan.restype = ctypes.c_int
        vp = ctypes.c_void_p
        L.orc_key_index.argtypes = [ctypes.c_float, ctypes.c_int32, ctypes.c_float, ctypes.c_int32,
                                    ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_float)]
        L.orc_key_index.restype = None
        L.orc_sample.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_float, ctypes.c_int32,
                                 ctypes.c_float, ctypes.c_int32, vp]
        L.orc_sample.restype = None
        L.orc_blend.argtypes = [ctypes.c_int32, vp, vp, vp]
        L.orc_blend.restype = None
        L.orc_trs_to_matrix.argtypes = [vp, vp]
        L.orc_trs_to_matrix.restype = None
        L.orc_animate.argtypes = [i32p, ctypes.c_int32, vp, ctypes.c_int32, ctypes.c_float,
                                  ctypes.c_int32, vp, ctypes.c_int32, vp, ctypes.c_int64, vp, vp, vp,
                                  ctypes.c_int]
        L.orc_animate.restype = ctypes.c_int
        L.orc_skin_vertices.argtypes = [vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, vp]
        L.orc_skin_vertices.restype = ctypes.c_int
        _lib = L
    return _lib


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


class OracleError(ValueError):
    def __init__(self, status: int):
        super().__init__(f"oracle: {STATUS.get(status, status)}")
        self.status = STATUS.get(status, status)


def validate(parents) -> str:
    p, pp = _i32(parents)
    return STATUS[lib().orc_validate(pp, len(p))]


def kahn_order(parents) -> np.ndarray:
    p, pp = _i32(parents)
    out = np.empty(len(p), np.int32)
    st = lib().orc_kahn_order(pp, len(p), out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    if st:
        raise OracleError(st)
    return out


def compose(a, b) -> np.ndarray:
    """fp64 affine compose of two 3x4 matrices (parent on the left)."""
    a = np.ascontiguousarray(a, np.float64).reshape(12)
    b = np.ascontiguousarray(b, np.float64).reshape(12)
    c = np.empty(12, np.float64)
    lib().orc_compose(a.ctypes.data, b.ctypes.data, c.ctypes.data)
    return c.reshape(3, 4)


def scan(parents, local, inv_bind=None, nthreads: int | None = None):
    """Oracle Hierarchy-Scan + bind.

    parents: [J] int (-1 = root, any order); local: [n_chars, J, 3, 4] (or [J,3,4])
    float32; inv_bind: [J, 3, 4] float32 or None (identity).
    Returns (global, skin) fp64 arrays of local's shape.
    """
    p, pp = _i32(parents)
    J = len(p)
    local = np.ascontiguousarray(local, dtype=np.float32)
    squeeze = local.ndim == 3
    if squeeze:
        local = local[None]
    assert local.shape[1:] == (J, 3, 4), local.shape
    n_chars = local.shape[0]
    ib = None
    if inv_bind is not None:
        ib = np.ascontiguousarray(inv_bind, dtype=np.float32)
        assert ib.shape == (J, 3, 4)
    g = np.empty(local.shape, np.float64)
    s = np.empty(local.shape, np.float64)
    st = lib().orc_scan(pp, J, local.ctypes.data, None if ib is None else ib.ctypes.data,
                        n_chars, g.ctypes.data, s.ctypes.data, nthreads or os.cpu_count() or 1,
                        None)
    if st:
        raise OracleError(st)
    if squeeze:
        return g[0], s[0]
    return g, s


def scan_discard(parents, local, inv_bind=None, nthreads: int | None = None) -> float:
    """Timed-baseline mode: same arithmetic, outputs kept in per-thread scratch only.
    Returns a checksum of the results so the work is observable."""
    p, pp = _i32(parents)
    J = len(p)
    local = np.ascontiguousarray(local, dtype=np.float32)
    n_chars = local.shape[0]
    ib = None if inv_bind is None else np.ascontiguousarray(inv_bind, dtype=np.float32)
    cs = ctypes.c_double(0.0)
    st = lib().orc_scan(pp, J, local.ctypes.data, None if ib is None else ib.ctypes.data,
                        n_chars, None, None, nthreads or os.cpu_count() or 1, ctypes.byref(cs))
    if st:
        raise OracleError(st)
    return cs.value


# ---------------------------------------------------------------- Stage 1 (NEXT-1)
LAYER_DTYPE = np.dtype([("clip", "<i4"), ("time", "<f4"), ("weight", "<f4"), ("pad", "<i4")])


def key_index(t: float, n_keys: int, fps: float, wrap: int):
    k = ctypes.c_int32()
    a = ctypes.c_float()
    lib().orc_key_index(t, n_keys, fps, wrap, ctypes.byref(k), ctypes.byref(a))
    return k.value, a.value


def sample(clip_keys, fps: float, wrap: int, t: float, joint: int) -> np.ndarray:
    """clip_keys: [n_keys, J, 10] fp32 (one clip) -> fp64 Trs (t3, q wxyz, s3)."""
    ck = np.ascontiguousarray(clip_keys, np.float32)
    out = np.empty(10, np.float64)
    lib().orc_sample(ck.ctypes.data, ck.shape[0], ck.shape[1], fps, wrap, t, joint, out.ctypes.data)
    return out


def blend(poses, weights) -> np.ndarray:
    p = np.ascontiguousarray(poses, np.float64).reshape(-1, 10)
    w = np.ascontiguousarray(weights, np.float64)
    out = np.empty(10, np.float64)
    lib().orc_blend(len(p), p.ctypes.data, w.ctypes.data, out.ctypes.data)
    return out


def trs_to_matrix(trs) -> np.ndarray:
    t = np.ascontiguousarray(trs, np.float64)
    out = np.empty(12, np.float64)
    lib().orc_trs_to_matrix(t.ctypes.data, out.ctypes.data)
    return out.reshape(3, 4)


def animate(parents, keys, fps: float, wrap: int, layers, inv_bind=None, nthreads=None,
            return_local=False):
    """Stage 1 + scan + bind in fp64.  keys: [n_clips, n_keys, J, 10] fp32; layers:
    structured [n_chars, n_layers] of LAYER_DTYPE.  Returns (G, S[, L])."""
    p, pp = _i32(parents)
    J = len(p)
    k = np.ascontiguousarray(keys, np.float32)
    assert k.shape[2] == J and k.shape[3] == 10
    lay = np.ascontiguousarray(layers, LAYER_DTYPE)
    n_chars, n_layers = lay.shape
    ib = None if inv_bind is None else np.ascontiguousarray(inv_bind, np.float32)
    g = np.empty((n_chars, J, 3, 4), np.float64)
    s = np.empty_like(g)
    loc = np.empty_like(g) if return_local else None
    st = lib().orc_animate(pp, J, k.ctypes.data, k.shape[1], fps, wrap, lay.ctypes.data, n_layers,
                           None if ib is None else ib.ctypes.data, n_chars, g.ctypes.data,
                           s.ctypes.data, None if loc is None else loc.ctypes.data,
                           nthreads or os.cpu_count() or 1)
    if st:
        raise OracleError(st)
    return (g, s, loc) if return_local else (g, s)


# ---------------------------------------------------------------- LBS (NEXT-4)
def skin_vertices(skin, pos, joints, weights) -> np.ndarray:
    """Linear blend skinning in fp64.  skin: [n_chars, J, 3, 4] (or [J, 3, 4]) skin
    matrices; pos [V, 3], joints [V, 4], weights [V, 4].  Returns [n_chars, V, 3]."""
    S = np.ascontiguousarray(skin, np.float64)
    squeeze = S.ndim == 3
    if squeeze:
        S = S[None]
    n, J = S.shape[0], S.shape[1]
    p = np.ascontiguousarray(pos, np.float32)
    jt = np.ascontiguousarray(joints, np.int32)
    w = np.ascontiguousarray(weights, np.float32)
    V = p.shape[0]
    out = np.empty((n, V, 3), np.float64)
    st = lib().orc_skin_vertices(S.ctypes.data, n, J, V, p.ctypes.data, jt.ctypes.data, w.ctypes.data,
                                 out.ctypes.data)
    if st:
        raise OracleError(st)
    return out[0] if squeeze else out
