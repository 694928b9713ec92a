"""Host-side preprocessor (libhs.so, no GPU): SPEC worked values, brute-force
properties of the lift table / block layout / chunk-anchor decomposition, and
that the C ABI library exports every symbol include/hs.h declares.  CPU only."""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np
import pytest

import hsgen
import oracle
import paper_2505_06703_b200 as hs

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                     "spec_worked_values.json")))


@pytest.fixture(scope="module", autouse=True)
def _built():
    hs.build()


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(hs.LIB_PATH)
    names = hs.exported_symbols()
    assert len(names) >= 15
    for name in names:
        assert hasattr(L, name), name


def test_status_strings():
    L = hs.lib()
    for code, name in enumerate(["HS_OK", "HS_ERR_INVALID_ARG", "HS_ERR_EMPTY", "HS_ERR_OUT_OF_RANGE",
                                 "HS_ERR_CYCLE", "HS_ERR_CUDA", "HS_ERR_OOM", "HS_ERR_WRONG_DEVICE",
                                 "HS_ERR_UNSUPPORTED"]):
        assert L.hs_status_string(code).decode() == name


def _status(parents):
    try:
        hs.Plan(parents)
        return "ok"
    except hs.HSError as e:
        return {hs.HS_ERR_EMPTY: "empty", hs.HS_ERR_OUT_OF_RANGE: "out_of_range",
                hs.HS_ERR_CYCLE: "cycle"}[e.status]


def test_golden_topology():
    for case in GOLDEN["topology"]:
        st = _status(case["parents"])
        if case["valid"]:
            assert st == "ok", case["cite"]
            p = hs.Plan(case["parents"])
            assert list(p.export("levels")) == case["levels"], case["cite"]
            assert p.query("max_level") == max(case["levels"])
        else:
            assert st == case["error"], case["cite"]


def test_validation_agrees_with_oracle_on_all_small_arrays():
    import itertools
    for n in range(1, 5):
        for p in itertools.product(range(-1, n), repeat=n):
            assert _status(list(p)) == oracle.validate(list(p)), p


def test_golden_reindex():
    for case in GOLDEN["reindex"]:
        order = hs.Plan(case["parents"]).export("order")   # internal -> user
        if "perm_new_to_old" in case:
            assert list(order) == case["perm_new_to_old"], case["cite"]
        else:
            rank = np.empty_like(order); rank[order] = np.arange(len(order))
            assert list(rank) == case["perm_old_to_new"], case["cite"]
        p = np.asarray(case["parents"])
        ipar = [-1 if p[u] < 0 else int(np.where(order == p[u])[0][0]) for u in order]
        assert ipar == case["dfs_parents"], case["cite"]


def test_golden_lift_and_rounds():
    for case in GOLDEN["lift"]:
        pl = hs.Plan(case["parents"])
        lift = pl.export("lift")
        if "anc" in case:
            R = lift.shape[0]
            want = case["anc"]
            assert list(lift[:, case["joint"]]) == want[:R], case["cite"]
            assert all(a == -1 for a in want[R:]), case["cite"]
        else:
            i, j, want = case["multi_parent"]
            v = i
            for r in range(lift.shape[0]):   # binary decomposition of j (Eq. 2)
                if (j >> r) & 1:
                    v = lift[r, v]
            assert v == want, case["cite"]
    for case in GOLDEN["rounds"]:
        assert hs.Plan(hsgen.chain(case["chain"])).query("rounds") == case["rounds"], case["cite"]


def test_golden_block_layout():
    case = GOLDEN["blocks"][0]
    pl = hs.Plan(hsgen.chain(case["chain"]), block_size=case["block_size"])
    assert pl.export("block_of")[case["joint"]] == case["block_of"], case["cite"]
    assert pl.export("mpob")[case["joint"]] == case["mpob"], case["cite"]


def _random_forest(rng, n, permute=True):
    par = np.full(n, -1, np.int32)
    for i in range(1, n):
        par[i] = rng.integers(-1 if rng.random() < 0.03 else 0, i)
    if permute:
        par, _ = hsgen.relabel(par, rng.permutation(n).astype(np.int32))
    return par


def _walk(par, u, k):
    for _ in range(k):
        if u < 0:
            return -1
        u = par[u]
    return u


@pytest.mark.parametrize("seed", range(6))
def test_lift_table_brute_force(seed):
    rng = np.random.default_rng(seed)
    par = _random_forest(rng, 300)
    pl = hs.Plan(par)
    lift = pl.export("lift")
    lev = pl.export("levels")
    assert lift.shape[0] == int(np.ceil(np.log2(lev.max()))) if lev.max() > 1 else lift.shape[0] == 0
    for r in range(lift.shape[0]):
        for u in range(300):
            assert lift[r, u] == _walk(par, u, 1 << r)
    for u in range(300):
        d, v = 1, u
        while par[v] >= 0:
            v = par[v]; d += 1
        assert lev[u] == d


@pytest.mark.parametrize("seed", range(6))
def test_order_is_topological_and_block_layout_brute_force(seed):
    rng = np.random.default_rng(100 + seed)
    par = _random_forest(rng, 300, permute=bool(seed % 2))
    pl = hs.Plan(par, block_size=64)
    order = pl.export("order")
    assert sorted(order) == list(range(300))
    rank = np.empty(300, int); rank[order] = np.arange(300)
    ipar = np.array([-1 if par[u] < 0 else rank[par[u]] for u in order])
    assert np.all(ipar < np.arange(300))
    if seed % 2 == 0:
        assert pl.query("identity_order") == 1 and np.array_equal(order, np.arange(300))
    mpob = pl.export("mpob")
    for i in range(300):
        a = ipar[i]
        while a >= 0 and a // 64 == i // 64:
            a = ipar[a]
        assert mpob[i] == a


def _chunk_emulation(par, local, K, chunking=3):
    """Emulate this build's chunk/anchor algorithm on the host from
    the exported decomposition, in fp64.  On the exact-arithmetic family every
    association order gives the same bits, so this pins the decomposition."""
    pl = hs.Plan(par, chunk=K, chunking=chunking)
    order = pl.export("order")
    src = pl.export("chunk_src")
    link = pl.export("anchor_link")
    lists = [[int(f) for f in row if f >= 0] for row in pl.export("chunk_lists")]
    n = len(par)
    H = np.zeros((n, 4, 4)); H[:, :3] = local[order]; H[:, 3, 3] = 1
    anchors = sorted(set(int(s) for s in src if s >= 0))
    slot = {a: k for k, a in enumerate(anchors)}
    assert len(anchors) == len(link)
    # phase 1: per-chunk left fold (a RUN joint restarts like a head); publish anchors
    P = np.zeros((len(anchors), 4, 4))
    full = []
    for chunk in lists:
        acc = None
        for f in chunk:
            acc = acc @ H[f] if src[f] == -2 else H[f]
            if f in slot:
                P[slot[f]] = acc
        full.append(acc)
    # phase 2a: a lane whose first joint is RUN (-4) continues the previous lane's run;
    # lift its anchors by the product of the run's earlier lanes (exclusive prefix)
    excl = [None] * len(lists)
    for li, chunk in enumerate(lists):
        if chunk and src[chunk[0]] == -4:
            excl[li] = full[li - 1] if excl[li - 1] is None else excl[li - 1] @ full[li - 1]
            for f in chunk:
                if f in slot:
                    P[slot[f]] = excl[li] @ P[slot[f]]
    # phase 2: pointer jumping over the anchor forest (snapshot semantics)
    lk = link.copy()
    while np.any(lk >= 0):
        Pn = P.copy()
        for s in range(len(anchors)):
            if lk[s] >= 0:
                Pn[s] = P[lk[s]] @ P[s]
        P = Pn
        lk = np.array([lk[lk[s]] if lk[s] >= 0 else -1 for s in range(len(anchors))], np.int32)
    # phase 3: re-fold from the final anchor values (RUN: parent = previous lane's tail)
    G = np.zeros((n, 4, 4))
    for li, chunk in enumerate(lists):
        acc = None
        for f in chunk:
            if src[f] == -2:
                acc = acc @ H[f]
            elif src[f] == -1:
                acc = H[f]
            elif src[f] == -4:
                acc = G[lists[li - 1][-1]] @ H[f]
            else:
                acc = P[slot[src[f]]] @ H[f]
            G[f] = acc
    out = np.zeros((n, 3, 4)); out[order] = G[:, :3]
    return out


@pytest.mark.parametrize("chunking", [1, 2, 3])
@pytest.mark.parametrize("K", [3, 7, 11])
@pytest.mark.parametrize("name", ["hum64", "chain256", "tree1024", "perm_tree"])
def test_chunk_anchor_decomposition_reproduces_oracle_bitwise(name, K, chunking):
    if name == "perm_tree":
        par, _ = hsgen.relabel(hsgen.skeleton("tree1024"), hsgen.permutation(3, 1024))
    else:
        par = hsgen.skeleton(name)
    local = hsgen.exact_poses(21, len(par), 1)[0]
    g_ref, _ = oracle.scan(par, local)
    g = _chunk_emulation(par, local.astype(np.float64), K, chunking)
    assert np.array_equal(g, g_ref)


def test_decomposition_invariants():
    rng = np.random.default_rng(9)
    for trial in range(20):
        par = _random_forest(rng, int(rng.integers(1, 400)), permute=bool(trial % 2))
        K = [3, 5, 7, 9][trial % 4]
        pl = hs.Plan(par, chunk=K, chunking=[1, 2, 3][trial % 3])
        order = pl.export("order")
        n = len(par)
        rank = np.empty(n, int); rank[order] = np.arange(n)
        ipar = np.array([-1 if par[u] < 0 else rank[par[u]] for u in order])
        src = pl.export("chunk_src")
        lists = pl.export("chunk_lists")
        flat = lists[lists >= 0]
        assert sorted(flat) == list(range(n))          # every joint in exactly one list
        assert lists.shape[1] == K
        prev_of = {}
        for row in lists:
            row = [int(f) for f in row if f >= 0]
            for a, b in zip(row, row[1:]):
                prev_of[b] = a
        for f in range(n):
            if src[f] == -1:
                assert ipar[f] == -1
            elif src[f] == -2:
                assert prev_of.get(f) == ipar[f]
            elif src[f] == -4:   # RUN: parent is the previous lane's last joint
                lane = [i for i, row in enumerate(lists) if f in row][0]
                prev = [int(x) for x in lists[lane - 1] if x >= 0]
                assert list(lists[lane]).index(f) == 0 and prev[-1] == ipar[f]
            else:
                assert src[f] == ipar[f] and prev_of.get(f) != ipar[f]
        assert pl.query("anchors") == len(set(int(s) for s in src if s >= 0))


def test_errors_from_plan():
    with pytest.raises(hs.HSError) as e:
        hs.Plan([0])
    assert e.value.status == hs.HS_ERR_CYCLE
    with pytest.raises(hs.HSError) as e:
        hs.Plan([-1, 3])
    assert e.value.status == hs.HS_ERR_OUT_OF_RANGE
    with pytest.raises(hs.HSError) as e:
        hs.Plan([-1, 0], chunk=4)
    assert e.value.status == hs.HS_ERR_INVALID_ARG


@pytest.mark.parametrize("chunking", [1, 2, 3])
@pytest.mark.parametrize("name", ["hum32", "hum64", "chain256", "tree1024", "perm_tree", "forest"])
def test_tile_program_emulation_bitwise(name, chunking):
    """Replay the exact uploaded tile program (ping-pong locations, colouring, round
    order) on the host: bitwise equal to the oracle on the exact family."""
    from tests import tile_emulator
    if name == "perm_tree":
        par, _ = hsgen.relabel(hsgen.skeleton("tree1024"), hsgen.permutation(3, 1024))
    elif name == "forest":   # several long chains + a tree: runs split at warp boundaries
        a, b = hsgen.chain(200), hsgen.skeleton("tree1024")
        par = np.concatenate([a, np.where(a >= 0, a + 200, -1), np.where(b >= 0, b + 400, -1)]).astype(np.int32)
    else:
        par = hsgen.skeleton(name)
    J = len(par)
    local = hsgen.exact_poses(22, J, 1)[0]
    ib = hsgen.exact_inv_bind(22, J)
    G, S = oracle.scan(par, local, ib)
    g, s, _ = tile_emulator.run(hs.Plan(par, chunking=chunking), local, ib)
    assert np.array_equal(g, G) and np.array_equal(s, S)
