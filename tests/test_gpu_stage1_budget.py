"""Stage-1 error budget (NEXT-1): where the end-to-end error of
hs_animate against the fp64 oracle comes from, measured on the bench's Stage-1
workload (C5 skeletons, 8 clips x 31 keys at 30 fps, 2 layers, loop wrap).

Decomposition (every term computed here, printed as one JSON line per skeleton):
  e_repr   floor: the oracle's fp64 locals rounded once to fp32, scanned in fp64,
           against the fp64 scan of the fp64 locals (what any fp32 local pose costs)
  e_local  GPU Stage-1 locals (an all-roots skeleton returns them, G = L) against
           the oracle's fp64 locals, and their rotation blocks' orthonormality
           defect max |R R^T - I| (the normalisation bias shows up here)
  e_prop   the GPU locals scanned in fp64 against the fp64 scan of the fp64 locals
           (local-pose error carried down the root path, no GPU scan rounding)
  e_scan   the GPU's G against the fp64 scan of the GPU's own locals (scan rounding)
  e_total  the GPU's G and S against the oracle (what the tests assert)
"""
from __future__ import annotations

import json

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


def _animate(par, keys, lay, ib):
    sk = hs.Skeleton(par, ib)
    cs = hs.ClipSet(sk, keys, 30.0, 1)
    g, s = hs.animate(sk, cs, lay)
    torch.cuda.synchronize()
    return g.cpu().numpy().astype(np.float64), s.cpu().numpy().astype(np.float64)


def _orth_defect(m):
    R = m[..., :3, :3]
    return float(np.abs(R @ np.swapaxes(R, -1, -2) - np.eye(3)).max())


@pytest.mark.parametrize("name,type_,ib_seed,n", [("chain256", 1, 3, 300), ("tree1024", 2, 4, 100)])
def test_stage1_error_budget(name, type_, ib_seed, n):
    par = hsgen.skeleton(name)
    J = len(par)
    ib = hsgen.inv_bind(ib_seed, J)   # as in bench.py --stage1 (hsgen.CONFIGS[5])
    keys = hsgen.clips(100 + type_, J, 8, 31, type_=type_)
    lay = hsgen.layers(5, n, 2, 8, 1.5, type_=type_)
    G_o, S_o, Lo = oracle.animate(par, keys, 30.0, 1, lay, ib, return_local=True)
    # floor: correctly rounded fp32 locals, scanned exactly
    Lf = Lo.astype(np.float32)
    G_rf, _ = oracle.scan(par, Lf, ib)
    e_repr = float(np.abs(G_rf - G_o).max())
    # the GPU's locals (all-roots skeleton, same keys and layers: G = L)
    Lg, _ = _animate(np.full(J, -1, np.int32), keys, lay, None)
    e_local = float(np.abs(Lg - Lo).max())
    G_gl, _ = oracle.scan(par, Lg.astype(np.float32), ib)
    e_prop = float(np.abs(G_gl - G_o).max())
    # which part of the local error carries down the path: only the translation column
    # of the GPU locals (rotation blocks exact), or only the rotation blocks
    Lt = Lo.copy()
    Lt[..., 3] = Lg[..., 3]
    LR = Lg.copy()
    LR[..., 3] = Lo[..., 3]
    e_prop_t = float(np.abs(oracle.scan(par, Lt, ib)[0] - G_o).max())
    e_prop_R = float(np.abs(oracle.scan(par, LR, ib)[0] - G_o).max())
    G_g, S_g = _animate(par, keys, lay, ib)
    e_scan = float(np.abs(G_g - G_gl).max())
    e_total = max(float(np.abs(G_g - G_o).max()), float(np.abs(S_g - S_o).max()))
    rec = {"skeleton": name, "chars": n, "e_repr": e_repr, "e_local": e_local,
           "orth_gpu_locals": _orth_defect(Lg), "orth_rounded_locals": _orth_defect(Lf.astype(np.float64)),
           "e_prop": e_prop, "e_prop_t_only": e_prop_t, "e_prop_R_only": e_prop_R, "e_scan": e_scan,
           "e_total": e_total}
    print("stage1-budget " + json.dumps(rec))
    # the pieces are consistent (triangle inequality) and the total meets the bound
    assert float(np.abs(G_g - G_o).max()) <= e_prop + e_scan + 1e-12
    assert e_total <= TOL
