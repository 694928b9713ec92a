"""B200-native Hierarchy-Scan + fused Bind MeshPose (arxiv 2505.06703).

Thin ctypes binding over ``libhs.so`` (C ABI in ``include/hs.h``).  Argument
marshalling only: every step of the path runs in the library's sm_100a kernels.
PyTorch supplies device memory and streams.  There is NO CPU fallback: if the
compiled library is missing, importing the bindings raises.

    sk = Skeleton(parents, inv_bind)            # host preprocessor + upload, once
    g, s = sk.scan(local)                       # local: cuda float32 [N, J, 3, 4]
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
LIB_PATH = os.path.join(_HERE, "libhs.so")
# A/B experiments may point the binding at another in-tree build of the same sources.
_LOAD_PATH = os.environ.get("HS_LIB", LIB_PATH)
_SOURCES = [os.path.join(_HERE, "csrc", f) for f in ("plan.cpp", "api.cpp", "kernels.cu", "kernels_aux.cu",
                                                      "kernels_seq.cu")]
_DEPS = _SOURCES + [os.path.join(_HERE, "csrc", f) for f in ("plan.hpp", "kernels.cuh", "device_util.cuh")] + [
    os.path.join(_ROOT, "include", "hs.h")]

NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-shared"]

# hs_status
HS_OK, HS_ERR_INVALID_ARG, HS_ERR_EMPTY, HS_ERR_OUT_OF_RANGE, HS_ERR_CYCLE, HS_ERR_CUDA, \
    HS_ERR_OOM, HS_ERR_WRONG_DEVICE, HS_ERR_UNSUPPORTED = range(9)
# hs_algo
ALGO = {"auto": 0, "chunked": 1, "doubling": 2, "split": 3, "gateau": 4, "leaf": 5, "blocked": 6,
        "tiles": 7, "compressed": 8}
# hs_query
QUERY = {"n_joints": 0, "max_level": 1, "rounds": 2, "path": 3, "chunk": 4, "tile_chars": 5,
         "anchors": 6, "anchor_rounds": 7, "identity_order": 8, "smem_bytes": 9, "threads": 10,
         "stages": 11, "device": 12, "split_levels": 13,
         "pbufs": 15, "sbufs": 16, "chunking": 17, "tile_slots": 18, "tile_rounds_entries": 19,
         "tile_r2": 20, "small_tile_chars": 21, "seq_tiles": 22, "seq_tile_joints": 23,
         "seq_exports": 24, "seq_smem_bytes": 25, "seq_threads": 26, "seq_slots": 27, "seq_r2max": 28,
         "seq_entries": 29, "seq_imports": 30, "seq_runs": 31, "seq_qslots": 32, "seq_chunk": 33,
         "seq_sbufs": 34}
# hs_plan_export_what
EXPORT = {"levels": 0, "order": 1, "lift": 2, "block_of": 3, "mpob": 4, "chunk_src": 5,
          "anchor_link": 6, "chunk_lists": 7, "tile_meta": 8, "tile_p1len": 9,
          "tile_round_off": 10, "tile_rounds": 11, "seq_tiles": 12, "seq_meta": 13, "seq_p1len": 14,
          "seq_round_off": 15, "seq_rounds": 16, "seq_imp": 17, "seq_runs": 18, "seq_ib_user": 19}


def sources_sha256() -> str:
    """Hash of the library's sources (csrc + hs.h): ties a committed ncu capture to the
    build it was taken on (bench.py reports the capture's traffic only on a match)."""
    import hashlib
    h = hashlib.sha256()
    for d in sorted(_DEPS):
        h.update(os.path.basename(d).encode())
        with open(d, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libhs.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    stale = force or not os.path.exists(LIB_PATH) or any(
        os.path.getmtime(LIB_PATH) < os.path.getmtime(d) for d in _DEPS)
    if stale:
        cmd = ["nvcc", *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), *_SOURCES, "-o",
               LIB_PATH]
        subprocess.run(cmd, check=True, cwd=_HERE)
    return LIB_PATH


def build_variant(name: str, defines) -> str:
    """Compile the same sources with extra -D flags into build/<name> (tuning and
    profiling builds, e.g. the HS_PROF_HOOKS=1 phase-profile build) and return the path."""
    out = os.path.join(_ROOT, "build", name)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    if not os.path.exists(out) or any(os.path.getmtime(out) < os.path.getmtime(d) for d in _DEPS):
        subprocess.run(["nvcc", *NVCC_FLAGS, *defines, *_SOURCES, "-o", out], check=True, cwd=_HERE)
    return out


def use_library(path: str) -> None:
    """Load another build of the library (before the first lib() call)."""
    global _LOAD_PATH
    if _lib is not None and _LOAD_PATH != path:
        raise RuntimeError("the library is already loaded")
    _LOAD_PATH = path


class HSError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        detail = _lib.hs_last_error().decode() if _lib is not None else ""
        name = _lib.hs_status_string(status).decode() if _lib is not None else str(status)
        super().__init__(f"{where}: {name}: {detail}")


class _CreateOpts(ctypes.Structure):
    _fields_ = [("chunk", ctypes.c_int32), ("tile_joints", ctypes.c_int32),
                ("force_split", ctypes.c_int32), ("stages", ctypes.c_int32),
                ("sbufs", ctypes.c_int32), ("pbuf", ctypes.c_int32),
                ("chunking", ctypes.c_int32), ("reserved", ctypes.c_int32 * 1)]


class _ScanOpts(ctypes.Structure):
    _fields_ = [("algo", ctypes.c_int32), ("max_rounds", ctypes.c_int32),
                ("tile_ctas", ctypes.c_int32), ("reserved", ctypes.c_int32 * 5)]


_lib = None


def lib():
    """Load libhs.so.  Raises if it has not been built — no fallback exists."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LOAD_PATH):
        raise ImportError(f"{_LOAD_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
    L = ctypes.CDLL(_LOAD_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.hs_skeleton_create.argtypes = [vp, i32, vp, ctypes.POINTER(vp)]
    L.hs_skeleton_create_ex.argtypes = [vp, i32, vp, ctypes.POINTER(_CreateOpts), ctypes.POINTER(vp)]
    L.hs_scan.argtypes = [vp, vp, i64, vp, vp, vp]
    L.hs_scan_ex.argtypes = [vp, vp, i64, vp, vp, vp, ctypes.POINTER(_ScanOpts)]
    L.hs_destroy.argtypes = [vp]
    L.hs_skeleton_query.argtypes = [vp, i32, ctypes.POINTER(i64)]
    L.hs_status_string.argtypes = [ctypes.c_int]
    L.hs_status_string.restype = ctypes.c_char_p
    L.hs_last_error.argtypes = []
    L.hs_last_error.restype = ctypes.c_char_p
    L.hs_plan_create.argtypes = [vp, i32, i32, i32, ctypes.POINTER(vp)]
    L.hs_plan_create_ex.argtypes = [vp, i32, ctypes.POINTER(_CreateOpts), i32, ctypes.POINTER(vp)]
    L.hs_plan_query.argtypes = [vp, i32, ctypes.POINTER(i64)]
    L.hs_plan_export.argtypes = [vp, i32, vp, i64]
    L.hs_plan_destroy.argtypes = [vp]
    L.hs_clipset_create.argtypes = [vp, vp, i32, i32, ctypes.c_float, i32, ctypes.POINTER(vp)]
    L.hs_clipset_destroy.argtypes = [vp]
    L.hs_animate.argtypes = [vp, vp, vp, i32, i64, vp, vp, vp]
    L.hs_animate_ex.argtypes = [vp, vp, vp, i32, i64, vp, vp, vp, ctypes.POINTER(_AnimateOpts)]
    L.hs_scan_batch.argtypes = [ctypes.POINTER(_BatchItem), i32, vp]
    L.hs_scan_varied.argtypes = [vp, vp, vp, i32, i64, vp, vp, vp]
    L.hs_mesh_create.argtypes = [vp, i32, vp, vp, vp, ctypes.POINTER(vp)]
    L.hs_mesh_destroy.argtypes = [vp]
    L.hs_scan_skin.argtypes = [vp, vp, vp, i64, vp, vp, vp, vp]
    L.hs_skin_vertices.argtypes = [vp, vp, i64, vp, vp]
    L.hs_animate_skin.argtypes = [vp, vp, vp, i32, i64, vp, vp, vp, vp, vp]
    L.hs_scan_skin_ex.argtypes = [vp, vp, vp, i64, vp, vp, vp, vp, ctypes.POINTER(_SkinOpts)]
    L.hs_pipeline_create.argtypes = [i64, ctypes.POINTER(vp)]
    L.hs_scan_host.argtypes = [vp, vp, vp, i64, vp, vp]
    L.hs_scan_host_batch.argtypes = [vp, ctypes.POINTER(_BatchItem), i32]
    L.hs_animate_host.argtypes = [vp, vp, vp, vp, i32, i64, vp, vp]
    L.hs_workspace_trim.argtypes = [ctypes.POINTER(ctypes.c_int64)]
    L.hs_pipeline_destroy.argtypes = [vp]
    for f in ("hs_skeleton_create", "hs_skeleton_create_ex", "hs_scan", "hs_scan_ex", "hs_destroy",
              "hs_skeleton_query", "hs_plan_create", "hs_plan_create_ex", "hs_plan_query", "hs_plan_export",
              "hs_plan_destroy", "hs_pipeline_create", "hs_scan_host", "hs_pipeline_destroy",
              "hs_clipset_create", "hs_clipset_destroy", "hs_animate"):
        getattr(L, f).restype = ctypes.c_int
    _lib = L
    return L


def _dev(t, name: str, need: int = 0, dtypes=("float32",)):
    """Device pointer of an argument: None, a raw device pointer (int, trusted), or a
    contiguous CUDA tensor of an accepted dtype holding at least `need` elements."""
    if t is None or isinstance(t, int):
        return t
    if not getattr(t, "is_cuda", False):
        raise TypeError(f"{name} must be a CUDA tensor (or a device pointer as int)")
    if str(t.dtype).replace("torch.", "") not in dtypes:
        raise TypeError(f"{name} must be {' or '.join(dtypes)}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.numel() < need:
        raise ValueError(f"{name} holds {t.numel()} elements, needs {need}")
    return t.data_ptr()


def _host(t, name: str, need_bytes: int = 0):
    """Host pointer of a contiguous CPU tensor or C-contiguous numpy array (pinned memory
    gives the full PCIe rate) of at least `need_bytes` bytes."""
    if hasattr(t, "data_ptr"):
        if t.is_cuda:
            raise TypeError(f"{name} must be a host (CPU) tensor")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        n, p = t.numel() * t.element_size(), t.data_ptr()
    else:
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name} must be C-contiguous")
        n, p = t.nbytes, t.ctypes.data
    if n < need_bytes:
        raise ValueError(f"{name} holds {n} bytes, needs {need_bytes}")
    return p


def _check(status: int, where: str):
    if status != HS_OK:
        raise HSError(status, where)


class Plan:
    """Host-only view of the topology preprocessor (no CUDA)."""

    def __init__(self, parents, chunk: int = 0, block_size: int = 0, chunking: int = 0,
                 tile_joints: int = 0):
        L = lib()
        p = np.ascontiguousarray(np.asarray(parents), dtype=np.int32)
        self.n = len(p)
        h = ctypes.c_void_p()
        o = _CreateOpts(chunk, tile_joints, 0, 0, 0, 0, chunking)
        _check(L.hs_plan_create_ex(p.ctypes.data if self.n else None, self.n, ctypes.byref(o),
                                   block_size, ctypes.byref(h)), "hs_plan_create")
        self._h = h

    def query(self, what: str) -> int:
        v = ctypes.c_int64()
        _check(lib().hs_plan_query(self._h, QUERY[what], ctypes.byref(v)), "hs_plan_query")
        return v.value

    def export(self, what: str) -> np.ndarray:
        if what.startswith("seq_"):
            KT, T, K = self.query("seq_tiles"), self.query("seq_threads"), self.query("chunk")
            F, R2 = self.query("seq_tile_joints"), self.query("seq_r2max")
            dtype, shape = {"seq_tiles": (np.int32, (KT, 12)), "seq_meta": (np.uint64, (KT, T, K)),
                            "seq_p1len": (np.int32, (KT, T)), "seq_round_off": (np.int32, (KT, (R2 + 4) // 4 * 4)),
                            "seq_rounds": (np.uint32, (self.query("seq_entries"),)),
                            "seq_imp": (np.int32, (self.query("seq_imports"), 2)),
                            "seq_runs": (np.int32, (self.query("seq_runs"), 4)),
                            "seq_ib_user": (np.int32, (KT, F))}[what]
            out = np.empty(max(int(np.prod(shape)), 1), dtype)
            _check(lib().hs_plan_export(self._h, EXPORT[what], out.ctypes.data, out.nbytes),
                   "hs_plan_export")
            return out[:int(np.prod(shape))].reshape(shape)
        if what.startswith("tile_"):
            T, K = self.query("threads"), self.query("chunk")
            dtype, size = {"tile_meta": (np.uint64, T * K), "tile_p1len": (np.int32, T),
                           "tile_round_off": (np.int32, self.query("tile_r2") + 1),
                           "tile_rounds": (np.uint32, self.query("tile_rounds_entries"))}[what]
            out = np.empty(max(size, 1), dtype)
            _check(lib().hs_plan_export(self._h, EXPORT[what], out.ctypes.data, out.nbytes),
                   "hs_plan_export")
            out = out[:size]
            return out.reshape(T, K) if what == "tile_meta" else out
        if what == "lift":
            size = self.query("rounds") * self.n
        elif what == "anchor_link":
            size = self.query("anchors")
        elif what == "chunk_lists":
            size = self.query("threads") * self.query("chunk")
        else:
            size = self.n
        out = np.empty(max(size, 1), np.int32)
        _check(lib().hs_plan_export(self._h, EXPORT[what], out.ctypes.data, out.nbytes),
               "hs_plan_export")
        out = out[:size]
        if what == "lift":
            return out.reshape(-1, self.n)
        if what == "chunk_lists":
            return out.reshape(-1, self.query("chunk"))
        return out

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.hs_plan_destroy(self._h)
        self._h = None

    __del__ = close


class Skeleton:
    """A skeleton handle on the current CUDA device (hs_skeleton_create_ex)."""

    def __init__(self, parents, inv_bind=None, *, chunk: int = 0, tile_joints: int = 0,
                 force_split: bool = False, stages: int = 0, sbufs: int = 0, pbuf: int = 0,
                 chunking: int = 0):
        L = lib()
        p = np.ascontiguousarray(np.asarray(parents), dtype=np.int32)
        self.n_joints = len(p)
        ib = None
        if inv_bind is not None:
            ib = np.ascontiguousarray(np.asarray(inv_bind, dtype=np.float32))
            if ib.shape != (self.n_joints, 3, 4):
                raise ValueError(f"inv_bind must be [{self.n_joints}, 3, 4]")
        o = _CreateOpts(chunk, tile_joints, int(force_split), stages, sbufs, pbuf, chunking)
        h = ctypes.c_void_p()
        _check(L.hs_skeleton_create_ex(p.ctypes.data if self.n_joints else None, self.n_joints,
                                       None if ib is None else ib.ctypes.data, ctypes.byref(o),
                                       ctypes.byref(h)), "hs_skeleton_create")
        self._h = h

    @property
    def handle(self):
        return self._h

    def query(self, what: str) -> int:
        v = ctypes.c_int64()
        _check(lib().hs_skeleton_query(self._h, QUERY[what], ctypes.byref(v)), "hs_skeleton_query")
        return v.value

    def scan_into(self, local, global_out, skin_out=None, *, n_chars: int | None = None,
                  stream=None, algo: str = "auto", max_rounds: int = -1, tile_ctas: int = 0):
        """hs_scan_ex on caller-owned CUDA tensors (or raw device pointers as ints)."""
        import torch

        if n_chars is None:
            n_chars = local.shape[0]
        need = n_chars * self.n_joints * 12
        pl, pg, ps = _dev(local, "local", need), _dev(global_out, "global_out", need), _dev(skin_out, "skin_out", need)
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        elif not isinstance(stream, int):
            stream = stream.cuda_stream
        opts = _ScanOpts(ALGO[algo], max_rounds, tile_ctas)
        _check(lib().hs_scan_ex(self._h, pl, n_chars, pg, ps, stream, ctypes.byref(opts)), "hs_scan")

    def scan(self, local, *, skin: bool = True, algo: str = "auto", max_rounds: int = -1,
             tile_ctas: int = 0):
        """local: CUDA float32 [N, J, 3, 4] -> (global, skin) (skin None if skin=False)."""
        import torch
        if local.dtype != torch.float32 or not local.is_cuda:
            raise TypeError("local must be a CUDA float32 tensor")
        local = local.contiguous()
        squeeze = local.dim() == 3
        if squeeze:
            local = local.unsqueeze(0)
        if tuple(local.shape[1:]) != (self.n_joints, 3, 4):
            raise ValueError(f"local must be [N, {self.n_joints}, 3, 4]")
        g = torch.empty_like(local)
        s = torch.empty_like(local) if skin else None
        self.scan_into(local, g, s, algo=algo, max_rounds=max_rounds, tile_ctas=tile_ctas)
        if squeeze:
            return g[0], (s[0] if s is not None else None)
        return g, s

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.hs_destroy(self._h)
        self._h = None

    __del__ = close


MAX_BATCH = 8   # HS_MAX_BATCH


ANIMATE_MODE = {"auto": 0, "fused": 1, "two_pass": 2}


class _AnimateOpts(ctypes.Structure):   # hs_animate_opts
    _fields_ = [("mode", ctypes.c_int32), ("reserved0", ctypes.c_int32),
                ("workspace_bytes", ctypes.c_int64), ("reserved", ctypes.c_int64 * 2)]


class _SkinOpts(ctypes.Structure):   # hs_skin_opts
    _fields_ = [("mode", ctypes.c_int32), ("reserved0", ctypes.c_int32),
                ("workspace_bytes", ctypes.c_int64), ("reserved", ctypes.c_int64 * 2)]


class _BatchItem(ctypes.Structure):
    _fields_ = [("skeleton", ctypes.c_void_p), ("local", ctypes.c_void_p), ("n_chars", ctypes.c_int64),
                ("global_out", ctypes.c_void_p), ("skin_out", ctypes.c_void_p)]


def scan_batch(items, stream=None):
    """hs_scan_batch: one launch over several crowds (NEXT-3).  items: sequence of
    (Skeleton, local, global_out, skin_out-or-None) CUDA tensors (or device pointers
    as ints, then a fifth element n_chars)."""
    import torch

    arr = (_BatchItem * max(1, len(items)))()
    for i, it in enumerate(items):
        sk, loc, g, s = it[:4]
        n = it[4] if len(it) > 4 else loc.shape[0]
        need = n * sk.n_joints * 12
        arr[i] = _BatchItem(sk.handle, _dev(loc, f"items[{i}].local", need), n,
                            _dev(g, f"items[{i}].global_out", need), _dev(s, f"items[{i}].skin_out", need))
    st = torch.cuda.current_stream().cuda_stream if stream is None else (
        stream if isinstance(stream, int) else stream.cuda_stream)
    _check(lib().hs_scan_batch(arr, len(items), st), "hs_scan_batch")


class Mesh:
    """Skinned mesh for one skeleton (hs_mesh_create): pos [V, 3] f32, joints [V, 4]
    int32, weights [V, 4] f32 (NEXT-4)."""

    def __init__(self, sk: "Skeleton", pos, joints, weights):
        p = np.ascontiguousarray(pos, np.float32)
        j = np.ascontiguousarray(joints, np.int32)
        w = np.ascontiguousarray(weights, np.float32)
        V = p.shape[0]
        if p.shape != (V, 3) or j.shape != (V, 4) or w.shape != (V, 4):
            raise ValueError("pos [V, 3], joints [V, 4], weights [V, 4]")
        h = ctypes.c_void_p()
        _check(lib().hs_mesh_create(sk.handle, V, p.ctypes.data, j.ctypes.data, w.ctypes.data,
                                    ctypes.byref(h)), "hs_mesh_create")
        self._h, self.n_vertices = h, V

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.hs_mesh_destroy(self._h)
        self._h = None

    __del__ = close


def skin_vertices(mesh: Mesh, skin, verts_out=None, stream=None):
    """hs_skin_vertices: LBS from skin poses on the device (CUDA float32 [N, J, 3, 4])."""
    import torch
    n = skin.shape[0]
    if verts_out is None:
        verts_out = torch.empty((n, mesh.n_vertices, 3), dtype=torch.float32, device=skin.device)
    st = torch.cuda.current_stream().cuda_stream if stream is None else (
        stream if isinstance(stream, int) else stream.cuda_stream)
    _check(lib().hs_skin_vertices(mesh.handle, _dev(skin, "skin"), n,
                                  _dev(verts_out, "verts_out", n * mesh.n_vertices * 3), st), "hs_skin_vertices")
    return verts_out


SKIN_MODE = {"auto": 0, "fused": 1, "two_pass": 2}


def scan_skin(sk: "Skeleton", mesh: Mesh, local, global_out=None, skin_out=None, verts_out=None,
              stream=None, skin: bool = False, mode: str = "auto", workspace_bytes: int = 0):
    """hs_scan_skin: scan + bind + linear blend skinning.  Returns (global, skin-or-None,
    verts [N, V, 3])."""
    import torch
    n = local.shape[0]
    if global_out is None:
        global_out = torch.empty_like(local)
    if skin_out is None and skin:
        skin_out = torch.empty_like(local)
    if verts_out is None:
        verts_out = torch.empty((n, mesh.n_vertices, 3), dtype=torch.float32, device=local.device)
    st = torch.cuda.current_stream().cuda_stream if stream is None else (
        stream if isinstance(stream, int) else stream.cuda_stream)
    opts = _SkinOpts(SKIN_MODE[mode], 0, workspace_bytes)
    need = n * sk.n_joints * 12
    _check(lib().hs_scan_skin_ex(sk.handle, mesh.handle, _dev(local, "local", need), n,
                                 _dev(global_out, "global_out", need), _dev(skin_out, "skin_out", need),
                                 _dev(verts_out, "verts_out", n * mesh.n_vertices * 3), st,
                                 ctypes.byref(opts)), "hs_scan_skin")
    return global_out, skin_out, verts_out


def scan_varied(parents, local, inv_bind=None, global_out=None, skin_out=None, stream=None,
                skin: bool = True):
    """hs_scan_varied: per-character topology.  parents: CUDA int32 [N, J]; local: CUDA
    float32 [N, J, 3, 4]; inv_bind: CUDA float32 [N, J, 3, 4] or None."""
    import torch
    if parents.dtype != torch.int32 or local.dtype != torch.float32:
        raise TypeError("parents must be int32 and local float32 CUDA tensors")
    if not (parents.is_contiguous() and local.is_contiguous()) or (inv_bind is not None and not inv_bind.is_contiguous()):
        raise ValueError("tensors must be contiguous")
    n, J = parents.shape
    if tuple(local.shape) != (n, J, 3, 4):
        raise ValueError(f"local must be [{n}, {J}, 3, 4]")
    if global_out is None:
        global_out = torch.empty_like(local)
    if skin_out is None and skin:
        skin_out = torch.empty_like(local)
    st = torch.cuda.current_stream().cuda_stream if stream is None else (
        stream if isinstance(stream, int) else stream.cuda_stream)
    need = n * J * 12
    _check(lib().hs_scan_varied(_dev(parents, "parents", n * J, ("int32",)), _dev(local, "local", need),
                                _dev(inv_bind, "inv_bind", need), J, n,
                                _dev(global_out, "global_out", need), _dev(skin_out, "skin_out", need), st),
           "hs_scan_varied")
    return global_out, skin_out


LAYER_DTYPE = np.dtype([("clip", "<i4"), ("time", "<f4"), ("weight", "<f4"), ("pad", "<i4")])


class ClipSet:
    """Animation clips for one skeleton (hs_clipset_create): keys [n_clips, n_keys, J, 10]
    fp32 = t(3), q(w,x,y,z), s(3), uniformly spaced at fps; wrap 0 clamp / 1 loop."""

    def __init__(self, sk: "Skeleton", keys, fps: float, wrap: int = 1):
        k = np.ascontiguousarray(np.asarray(keys, dtype=np.float32))
        if k.ndim != 4 or k.shape[2] != sk.n_joints or k.shape[3] != 10:
            raise ValueError(f"keys must be [n_clips, n_keys, {sk.n_joints}, 10]")
        h = ctypes.c_void_p()
        _check(lib().hs_clipset_create(sk.handle, k.ctypes.data, k.shape[0], k.shape[1], fps, wrap,
                                       ctypes.byref(h)), "hs_clipset_create")
        self._h, self.n_clips, self.n_keys = h, k.shape[0], k.shape[1]

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.hs_clipset_destroy(self._h)
        self._h = None

    __del__ = close


def animate(sk: "Skeleton", clips: ClipSet, layers, global_out=None, skin_out=None, stream=None,
            skin: bool = True, mode: str = "auto", workspace_bytes: int = 0):
    """Stage 1 + Hierarchy-Scan + Bind (hs_animate).  layers: CUDA tensor [N, n_layers, 4]
    int32 / float32 bit pattern of hs_layer, or a numpy LAYER_DTYPE array (copied)."""
    import torch
    if isinstance(layers, np.ndarray):
        layers = torch.from_numpy(np.ascontiguousarray(layers).view(np.int32).reshape(
            layers.shape[0], layers.shape[1], 4)).cuda()
    n, nl = layers.shape[0], layers.shape[1]
    if global_out is None:
        global_out = torch.empty((n, sk.n_joints, 3, 4), dtype=torch.float32, device=layers.device)
    if skin_out is None and skin:
        skin_out = torch.empty_like(global_out)
    st = torch.cuda.current_stream().cuda_stream if stream is None else (
        stream if isinstance(stream, int) else stream.cuda_stream)
    opts = _AnimateOpts(ANIMATE_MODE[mode], 0, workspace_bytes)
    need = n * sk.n_joints * 12
    _check(lib().hs_animate_ex(sk.handle, clips.handle, _dev(layers, "layers", n * nl * 4, ("int32", "float32")),
                               nl, n, _dev(global_out, "global_out", need), _dev(skin_out, "skin_out", need), st,
                               ctypes.byref(opts)),
           "hs_animate")
    return global_out, skin_out


def animate_skin(sk: "Skeleton", clips: "ClipSet", layers, mesh: "Mesh", global_out=None, skin_out=None,
                 verts_out=None, stream=None, skin: bool = False):
    """hs_animate_skin: Stage 1 -> scan -> bind -> skinning.  Returns (global, skin, verts)."""
    import torch
    if isinstance(layers, np.ndarray):
        layers = torch.from_numpy(np.ascontiguousarray(layers).view(np.int32).reshape(
            layers.shape[0], layers.shape[1], 4)).cuda()
    n, nl = layers.shape[0], layers.shape[1]
    if global_out is None:
        global_out = torch.empty((n, sk.n_joints, 3, 4), dtype=torch.float32, device=layers.device)
    if skin_out is None and skin:
        skin_out = torch.empty_like(global_out)
    if verts_out is None:
        verts_out = torch.empty((n, mesh.n_vertices, 3), dtype=torch.float32, device=layers.device)
    st = torch.cuda.current_stream().cuda_stream if stream is None else (
        stream if isinstance(stream, int) else stream.cuda_stream)
    need = n * sk.n_joints * 12
    _check(lib().hs_animate_skin(sk.handle, clips.handle, _dev(layers, "layers", n * nl * 4, ("int32", "float32")),
                                 nl, n, mesh.handle, _dev(global_out, "global_out", need),
                                 _dev(skin_out, "skin_out", need),
                                 _dev(verts_out, "verts_out", n * mesh.n_vertices * 3), st), "hs_animate_skin")
    return global_out, skin_out, verts_out


def workspace_trim() -> int:
    """hs_workspace_trim: return the workspace pool's unused memory on the current device
    to the driver; returns the bytes the pool still reserves."""
    held = ctypes.c_int64(0)
    _check(lib().hs_workspace_trim(ctypes.byref(held)), "hs_workspace_trim")
    return held.value


class Pipeline:
    """Host-buffer entry point (hs_scan_host): H2D, scan, D2H pipelined over batches."""

    def __init__(self, batch_bytes: int = 0):
        h = ctypes.c_void_p()
        _check(lib().hs_pipeline_create(batch_bytes, ctypes.byref(h)), "hs_pipeline_create")
        self._h = h

    def scan_host(self, sk: Skeleton, h_local, h_global, h_skin, n_chars: int | None = None):
        """Host tensors/arrays (pinned for full PCIe rate) -> fills h_global, h_skin."""
        if n_chars is None:
            n_chars = h_local.shape[0]
        need = n_chars * sk.n_joints * 48
        _check(lib().hs_scan_host(self._h, sk.handle, _host(h_local, "h_local", need), n_chars,
                                  _host(h_global, "h_global", need), _host(h_skin, "h_skin", need)),
               "hs_scan_host")

    def animate_host(self, sk: Skeleton, clips: "ClipSet", h_layers, h_global, h_skin):
        """hs_animate_host: host layer states [N, n_layers] (LAYER_DTYPE array or an int32
        [N, n_layers, 4] tensor, pinned for full PCIe rate) -> fills h_global, h_skin."""
        n, nl = h_layers.shape[0], h_layers.shape[1]
        need = n * sk.n_joints * 48
        _check(lib().hs_animate_host(self._h, sk.handle, clips.handle, _host(h_layers, "h_layers", n * nl * 16),
                                     nl, n, _host(h_global, "h_global", need), _host(h_skin, "h_skin", need)),
               "hs_animate_host")

    def scan_host_batch(self, items):
        """hs_scan_host_batch: items = [(Skeleton, h_local, h_global, h_skin), ...] on the
        host; one pipeline over all of them."""
        arr = (_BatchItem * max(1, len(items)))()
        for i, (sk, hl, hg, hsk) in enumerate(items):
            n = hl.shape[0]
            need = n * sk.n_joints * 48
            arr[i] = _BatchItem(sk.handle, _host(hl, f"items[{i}].h_local", need), n,
                                _host(hg, f"items[{i}].h_global", need), _host(hsk, f"items[{i}].h_skin", need))
        _check(lib().hs_scan_host_batch(self._h, arr, len(items)), "hs_scan_host_batch")

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.hs_pipeline_destroy(self._h)
        self._h = None

    __del__ = close


def exported_symbols() -> list[str]:
    """Function names declared in include/hs.h (for the ABI export test)."""
    import re
    src = open(os.path.join(_ROOT, "include", "hs.h")).read()
    return sorted(set(re.findall(r"^\s*(?:hs_status|const char\*)\s+(hs_\w+)\s*\(", src, re.M)))
