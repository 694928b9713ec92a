"""Seeded counter-based synthetic inputs (skeletons, local poses, inverse binds).

TEST/BENCH INFRASTRUCTURE, shared by both sides of the parity check: it holds
none of the method's arithmetic (see hsgen/gen.c for the recipe).  Skeleton
templates follow SURVEY.md §8(d) "Exact template parent arrays".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libhsgen.so")
_SRC = os.path.join(_HERE, "gen.c")
_CU = os.path.join(_HERE, "gen_cuda.cu")
_SO_CUDA = os.path.join(_HERE, "libhsgen_cuda.so")

# --- skeleton templates -----------------------------------
HUM32 = [-1, 0, 1, 2, 3, 4, 5, 3, 7, 8, 9, 8, 9, 3, 13, 14, 15, 14, 15, 0, 19, 19, 21, 22, 23,
         0, 25, 25, 27, 28, 29, 0]
HUM64 = HUM32 + [10, 32, 33, 10, 35, 36, 10, 38, 39, 10, 41, 42, 10, 44, 45, 46, 16, 48, 49, 16,
                 51, 52, 16, 54, 55, 16, 57, 58, 16, 60, 61, 62]

# purposes (stream = 8*type + purpose)
P_LOCAL_ROT, P_LOCAL_TR, P_INV_BIND, P_SKELETON, P_EXACT, P_PERM, P_EXACT_IB = range(7)


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.run(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread", "-o", _SO, _SRC,
                        "-lm"], check=True)
    return _SO


def build_cuda(force: bool = False) -> str:
    if force or not os.path.exists(_SO_CUDA) or os.path.getmtime(_SO_CUDA) < os.path.getmtime(_CU):
        subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                        "-Xcompiler", "-fPIC", "-o", _SO_CUDA, _CU], check=True)
    return _SO_CUDA


_lib = None
_libc = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        u64 = ctypes.c_uint64
        L.hsg_sm64.argtypes = [u64]
        L.hsg_sm64.restype = u64
        L.hsg_raw.argtypes = [u64] * 6
        L.hsg_raw.restype = u64
        L.hsg_u.argtypes = [u64] * 6
        L.hsg_u.restype = ctypes.c_double
        for name in ("hsg_local_poses", "hsg_exact_poses"):
            getattr(L, name).argtypes = [u64, u64, u64, u64, u64, ctypes.c_void_p, ctypes.c_int]
            getattr(L, name).restype = None
        for name in ("hsg_inv_bind", "hsg_exact_inv_bind"):
            getattr(L, name).argtypes = [u64, u64, u64, ctypes.c_void_p]
            getattr(L, name).restype = None
        L.hsg_random_tree.argtypes = [u64, u64, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
        L.hsg_random_tree.restype = ctypes.c_int
        L.hsg_permutation.argtypes = [u64, u64, ctypes.c_int32, ctypes.c_void_p]
        L.hsg_permutation.restype = None
        L.hsg_signed_perm.argtypes = [ctypes.c_int, ctypes.c_void_p]
        L.hsg_signed_perm.restype = None
        L.hsg_clips.argtypes = [u64, u64, u64, u64, u64, ctypes.c_float, ctypes.c_float,
                                ctypes.c_void_p]
        L.hsg_clips.restype = None
        L.hsg_layers.argtypes = [u64, u64, u64, u64, u64, u64, ctypes.c_float, ctypes.c_void_p]
        L.hsg_layers.restype = None
        L.hsg_mesh.argtypes = [u64, u64, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.hsg_mesh.restype = None
        _lib = L
    return _lib


def lib_cuda():
    global _libc
    if _libc is None:
        build_cuda()
        L = ctypes.CDLL(_SO_CUDA)
        u64 = ctypes.c_uint64
        L.hsg_cuda_local_poses.argtypes = [u64, u64, u64, u64, u64, ctypes.c_void_p,
                                           ctypes.c_void_p]
        L.hsg_cuda_local_poses.restype = ctypes.c_int
        _libc = L
    return _libc


def _threads(n):
    return n or min(32, os.cpu_count() or 1)


def sm64(x: int) -> int:
    return lib().hsg_sm64(x)


def u(seed, stream, c, J, j, k) -> float:
    return lib().hsg_u(seed, stream, c, J, j, k)


def local_poses(seed: int, J: int, n_chars: int, char0: int = 0, type_: int = 0,
                nthreads: int | None = None) -> np.ndarray:
    """Haar rotations + unit-ball translations: [n_chars, J, 3, 4] float32."""
    out = np.empty((n_chars, J, 3, 4), np.float32)
    if n_chars:
        lib().hsg_local_poses(seed, type_, J, char0, n_chars, out.ctypes.data, _threads(nthreads))
    return out


def exact_poses(seed: int, J: int, n_chars: int, char0: int = 0, type_: int = 0,
                nthreads: int | None = None) -> np.ndarray:
    """Exact-arithmetic family: signed-permutation rotations, translations in {-1,0,1}."""
    out = np.empty((n_chars, J, 3, 4), np.float32)
    if n_chars:
        lib().hsg_exact_poses(seed, type_, J, char0, n_chars, out.ctypes.data, _threads(nthreads))
    return out


def inv_bind(seed: int, J: int, type_: int = 0) -> np.ndarray:
    out = np.empty((J, 3, 4), np.float32)
    lib().hsg_inv_bind(seed, type_, J, out.ctypes.data)
    return out


def exact_inv_bind(seed: int, J: int, type_: int = 0) -> np.ndarray:
    out = np.empty((J, 3, 4), np.float32)
    lib().hsg_exact_inv_bind(seed, type_, J, out.ctypes.data)
    return out


def random_tree(seed: int, J: int, depth: int, type_: int = 0) -> np.ndarray:
    """SPEC random_tree: a depth-`depth` path then uniform attachment (max level == depth)."""
    out = np.empty(J, np.int32)
    if lib().hsg_random_tree(seed, type_, J, depth, out.ctypes.data):
        raise ValueError("random_tree: bad arguments")
    return out


def permutation(seed: int, n: int, type_: int = 0) -> np.ndarray:
    out = np.empty(n, np.int32)
    lib().hsg_permutation(seed, type_, n, out.ctypes.data)
    return out


def signed_perms() -> np.ndarray:
    out = np.empty((24, 3, 3), np.float32)
    for i in range(24):
        lib().hsg_signed_perm(i, out[i].ctypes.data)
    return out


def chain(J: int) -> np.ndarray:
    return np.arange(-1, J - 1, dtype=np.int32)


def relabel(parents, perm):
    """Relabel a parent array: new joint i is old joint perm[i].
    Returns (new_parents, inv) where inv[old] = new."""
    parents = np.asarray(parents, np.int32)
    perm = np.asarray(perm, np.int32)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm), dtype=np.int32)
    old_par = parents[perm]
    new_par = np.where(old_par >= 0, inv[np.maximum(old_par, 0)], -1).astype(np.int32)
    return new_par, inv


def dfs_labels(parents) -> np.ndarray:
    """The same forest relabelled in depth-first preorder, the largest child subtree
    first (how skeleton files usually list joints); roots in their original order."""
    par = np.asarray(parents, np.int32)
    J = len(par)
    children = [[] for _ in range(J)]
    for j in range(J):
        if par[j] >= 0:
            children[par[j]].append(j)
    size = np.ones(J, np.int64)
    for j in _topo(par)[::-1]:
        if par[j] >= 0:
            size[par[j]] += size[j]
    order, stack = [], [r for r in range(J) if par[r] < 0][::-1]
    while stack:
        v = stack.pop()
        order.append(v)
        stack.extend(sorted(children[v], key=lambda c: size[c]))   # largest popped first
    return relabel(par, np.array(order, np.int32))[0]


def _topo(par):
    """A topological order (parents first) of a forest given as a parent array."""
    J = len(par)
    children = [[] for _ in range(J)]
    for j in range(J):
        if par[j] >= 0:
            children[par[j]].append(j)
    out, stack = [], [r for r in range(J) if par[r] < 0]
    while stack:
        v = stack.pop()
        out.append(v)
        stack.extend(children[v])
    return np.array(out, np.int64)


# --- the BASELINE.json configs ------------------------------
def skeleton(name: str) -> np.ndarray:
    if name == "hum32":
        return np.array(HUM32, np.int32)
    if name == "hum64":
        return np.array(HUM64, np.int32)
    if name == "chain256":
        return chain(256)
    if name == "chain1024":
        return chain(1024)
    if name == "tree1024":
        return random_tree(4, 1024, 300)
    if name == "tree16384":   # the multi-CTA skeleton, 16,384 joints, L = 1024
        return random_tree(77, 16384, 1024)
    if name == "tree16384dfs":   # the same tree with depth-first labels (skeleton-file order)
        return dfs_labels(random_tree(77, 16384, 1024))
    raise KeyError(name)


# config id -> list of (skeleton name, n_chars, pose seed, type, inv_bind seed)
CONFIGS = {
    1: [("hum32", 1_000, 1, 0, 1)],
    2: [("hum64", 100_000, 2, 0, 2)],
    3: [("chain256", 50_000, 3, 0, 3)],
    4: [("tree1024", 20_000, 4, 0, 4)],
    5: [("hum64", 333_334, 5, 0, 2), ("chain256", 333_333, 5, 1, 3),
        ("tree1024", 333_333, 5, 2, 4)],
    # beyond one CTA (SURVEY §7 step 7 / VERDICT r1): the multi-tile path's workload
    6: [("tree16384", 2_000, 6, 0, 6)],
    # the same trees labelled depth-first: few cross-tile parents
    7: [("tree16384dfs", 2_000, 7, 0, 7)],
}


# --- Stage-1 inputs (NEXT-1) -----------------------------------------------------
LAYER_DTYPE = np.dtype([("clip", "<i4"), ("time", "<f4"), ("weight", "<f4"), ("pad", "<i4")])


def clips(seed: int, J: int, n_clips: int, n_keys: int, type_: int = 0,
          scale=(1.0, 1.0)) -> np.ndarray:
    """Keyframes [n_clips, n_keys, J, 10] fp32: t(3), q(w,x,y,z), s(3)."""
    out = np.empty((n_clips, n_keys, J, 10), np.float32)
    lib().hsg_clips(seed, type_, n_clips, n_keys, J, scale[0], scale[1], out.ctypes.data)
    return out


def layers(seed: int, n_chars: int, n_layers: int, n_clips: int, time_span: float,
           char0: int = 0, type_: int = 0) -> np.ndarray:
    """Per-character animation layers [n_chars, n_layers] (clip, time, weight)."""
    out = np.zeros((n_chars, n_layers), LAYER_DTYPE)
    if n_chars:
        lib().hsg_layers(seed, type_, char0, n_chars, n_layers, n_clips, time_span, out.ctypes.data)
    return out


# --- NEXT-4: synthetic skinned meshes --------------------------------------------------
def mesh(seed: int, parents, V: int, type_: int = 0):
    """(pos [V, 3] f32, joints [V, 4] i32, weights [V, 4] f32) for a skeleton."""
    par = np.ascontiguousarray(parents, np.int32)
    pos = np.empty((V, 3), np.float32)
    joints = np.empty((V, 4), np.int32)
    weights = np.empty((V, 4), np.float32)
    lib().hsg_mesh(seed, type_, par.ctypes.data, len(par), V, pos.ctypes.data, joints.ctypes.data,
                   weights.ctypes.data)
    return pos, joints, weights
