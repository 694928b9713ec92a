"""CPU tests of the multi-tile program (HS_ALGO_TILES): the exported
tables, replayed by tests/seq_emulator.py in the kernel's tile order, reproduce the
fp64 oracle BITWISE on the exact-arithmetic family (every product exact), which pins
the tile cut, TMA runs, imports/exports, slot locations and rounds encoding."""
from __future__ import annotations

import numpy as np
import pytest

import hsgen
import oracle
from tests import seq_emulator

hs = pytest.importorskip("paper_2505_06703_b200")


@pytest.fixture(scope="module", autouse=True)
def _built():
    hs.build()
    oracle.build()


def check(par, seed, **plan_kw):
    par = np.asarray(par, np.int32)
    J = len(par)
    plan = hs.Plan(par, **plan_kw)
    assert plan.query("seq_tiles") >= 1
    local = hsgen.exact_poses(seed, J, 1)
    ib = hsgen.exact_inv_bind(seed, J)
    G, S = oracle.scan(par, local, ib)
    g, s = seq_emulator.run(plan, local[0], ib)
    assert np.array_equal(g, G[0]) and np.array_equal(s, S[0])
    return plan


def test_tree16384_depth1024():
    """The multi-CTA bench skeleton: 16,384 joints, L = 1024."""
    plan = check(hsgen.random_tree(77, 16384, 1024), 1)
    assert plan.query("seq_tiles") == 16384 // plan.query("seq_tile_joints") + (
        16384 % plan.query("seq_tile_joints") > 0)
    assert plan.query("seq_runs") == plan.query("seq_tiles")       # topological labels: one run per tile


def test_dfs_labels_are_a_preorder_of_the_same_tree():
    """hsgen.dfs_labels (the C7 workload): a relabelling of the same forest in which every
    subtree is a contiguous label range starting at its root (depth-first preorder)."""
    par = hsgen.random_tree(77, 4000, 300)
    d = hsgen.dfs_labels(par)
    J = len(d)
    assert all(d[j] < j for j in range(J))
    size = np.ones(J, int)
    for j in range(J - 1, 0, -1):
        size[d[j]] += size[j]
    for j in range(J):   # children of j lie inside [j + 1, j + size[j])
        kids = np.nonzero(d == j)[0]
        assert all(j < c < j + size[j] for c in kids)
    # the same tree: sorted child-count and depth profiles agree
    def prof(p):
        lev = np.zeros(len(p), int)
        for j in range(len(p)):
            lev[j] = 0 if p[j] < 0 else lev[p[j]] + 1
        deg = np.bincount(p[p >= 0], minlength=len(p))
        return sorted(lev.tolist()), sorted(deg.tolist())
    assert prof(par) == prof(d)


def test_tree16384_dfs_labels():
    """C7: the bench tree in depth-first labels (K = 3, tiles of up to 672 joints)."""
    plan = check(hsgen.skeleton("tree16384dfs"), 3, chunk=3, tile_joints=672)
    assert plan.query("seq_qslots") < 100            # few cross-tile parents
    assert plan.query("seq_runs") == plan.query("seq_tiles")


@pytest.mark.parametrize("kw", [{}, {"chunking": 1}, {"chunking": 2}, {"chunk": 3}, {"chunk": 7},
                                {"tile_joints": 256}, {"tile_joints": 96, "chunk": 3}])
def test_variants_random_tree(kw):
    check(hsgen.random_tree(5, 3000, 120), 2, **kw)


def test_chain_and_star_and_forest():
    check(hsgen.chain(3000), 3)                                  # every tile imports one parent
    check(np.r_[-1, np.zeros(2999, np.int32)], 4)                # star: all import the root
    f = np.concatenate([hsgen.random_tree(6, 700, 40), hsgen.random_tree(7, 900, 300) + 700])
    f[700] = -1
    check(f, 5, tile_joints=384)                                 # forest, tiles straddle trees


def test_permuted_labels_gather_runs():
    """Non-topological user labels: tiles over the internal DFS order gather their joints
    through many short TMA runs; still bitwise."""
    base = hsgen.random_tree(8, 2500, 200)
    par, _ = hsgen.relabel(base, hsgen.permutation(9, 2500))
    plan = check(par, 6)
    assert plan.query("seq_runs") > plan.query("seq_tiles")
