// plan.cpp — host topology preprocessor (see plan.hpp and DESIGN.md §5).
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <array>
#include <stdexcept>

namespace hs {

namespace {
constexpr int kOk = 0, kInvalid = 1, kEmpty = 2, kOutOfRange = 3, kCycle = 4, kUnsupported = 8;
constexpr int32_t kMaxJoints = 1 << 20;
}  // namespace

int build_plan(const int32_t* parents, int32_t n, Plan& P, std::string& err) {
    if (n < 0 || (n > 0 && !parents)) { err = "parents is null or n_joints < 0"; return kInvalid; }
    if (n == 0) { err = "n_joints == 0"; return kEmpty; }
    if (n > kMaxJoints) { err = "n_joints above HS_MAX_JOINTS"; return kUnsupported; }
    P = Plan();
    P.n = n;
    P.parents.assign(parents, parents + n);
    for (int32_t j = 0; j < n; ++j)
        if (parents[j] < -1 || parents[j] >= n) {
            err = "parent of joint " + std::to_string(j) + " out of range: " + std::to_string(parents[j]);
            return kOutOfRange;
        }
    // children in ascending label order (CSR)
    std::vector<int32_t> first(n + 1, 0), kids(n);
    for (int32_t j = 0; j < n; ++j) if (parents[j] >= 0) first[parents[j] + 1]++;
    for (int32_t j = 0; j < n; ++j) first[j + 1] += first[j];
    {
        std::vector<int32_t> fill(first.begin(), first.end() - 1);
        for (int32_t j = 0; j < n; ++j) if (parents[j] >= 0) kids[fill[parents[j]]++] = j;
    }
    // DFS preorder from the roots (ascending), children ascending; nodes not
    // reached lie on (or under) a cycle.
    std::vector<int32_t> dfs;
    dfs.reserve(n);
    std::vector<int32_t> stack;
    // roots pushed in descending order so the smallest label is popped first
    for (int32_t r = n - 1; r >= 0; --r) if (parents[r] == -1) stack.push_back(r);
    while (!stack.empty()) {
        int32_t v = stack.back();
        stack.pop_back();
        dfs.push_back(v);
        for (int32_t e = first[v + 1] - 1; e >= first[v]; --e) stack.push_back(kids[e]);
    }
    if ((int32_t)dfs.size() != n) { err = "parent chain contains a cycle"; return kCycle; }

    P.level.assign(n, 0);
    for (int32_t v : dfs) P.level[v] = parents[v] < 0 ? 1 : P.level[parents[v]] + 1;
    P.L = *std::max_element(P.level.begin(), P.level.end());
    P.R = 0;
    while ((1LL << P.R) < P.L) ++P.R;

    P.identity = true;
    for (int32_t j = 0; j < n; ++j) if (parents[j] >= j) { P.identity = false; break; }
    P.order.resize(n);
    if (P.identity) for (int32_t i = 0; i < n; ++i) P.order[i] = i;
    else P.order = dfs;
    P.rank.resize(n);
    for (int32_t i = 0; i < n; ++i) P.rank[P.order[i]] = i;
    P.ipar.resize(n);
    for (int32_t i = 0; i < n; ++i) {
        int32_t q = parents[P.order[i]];
        P.ipar[i] = q < 0 ? -1 : P.rank[q];
    }
    // Eq. 2 lift table, user labels: anc[0] = Parent, anc[r+1][u] = anc[r][anc[r][u]].
    P.lift.assign((size_t)P.R * n, -1);
    for (int r = 0; r < P.R; ++r)
        for (int32_t u = 0; u < n; ++u) {
            int32_t a = r == 0 ? parents[u] : P.lift[(size_t)(r - 1) * n + u];
            if (r > 0 && a >= 0) a = P.lift[(size_t)(r - 1) * n + a];
            P.lift[(size_t)r * n + u] = a;
        }
    for (int32_t u = 0; u < n; ++u) if (first[u + 1] == first[u]) P.leaves.push_back(u);
    return kOk;
}

namespace {

// Heavy paths: walk every root's heavy path (child of largest subtree height,
// smallest index on ties), recursing into the light children.  Each path is a
// parent-to-child chain; together they partition the forest.
std::vector<std::vector<int32_t>> heavy_paths(const std::vector<int32_t>& par) {
    const int32_t F = (int32_t)par.size();
    std::vector<int32_t> first(F + 1, 0), kids(F), height(F, 1);
    for (int32_t f = 0; f < F; ++f) if (par[f] >= 0) first[par[f] + 1]++;
    for (int32_t f = 0; f < F; ++f) first[f + 1] += first[f];
    {
        std::vector<int32_t> fill(first.begin(), first.end() - 1);
        for (int32_t f = 0; f < F; ++f) if (par[f] >= 0) kids[fill[par[f]]++] = f;
    }
    for (int32_t f = F - 1; f >= 0; --f)          // par[f] < f: reverse order is bottom-up
        if (par[f] >= 0) height[par[f]] = std::max(height[par[f]], height[f] + 1);
    std::vector<std::vector<int32_t>> paths;
    std::vector<int32_t> stack;                   // path starts
    for (int32_t f = F - 1; f >= 0; --f) if (par[f] < 0) stack.push_back(f);
    while (!stack.empty()) {
        int32_t v = stack.back();
        stack.pop_back();
        paths.emplace_back();
        for (;;) {
            paths.back().push_back(v);
            int32_t h = -1;
            for (int32_t e = first[v]; e < first[v + 1]; ++e)
                if (h < 0 || height[kids[e]] > height[h]) h = kids[e];
            if (h < 0) break;
            for (int32_t e = first[v + 1] - 1; e >= first[v]; --e)
                if (kids[e] != h) stack.push_back(kids[e]);
            v = h;
        }
    }
    return paths;
}

// Heavy-path pieces of at most K joints (a piece is a parent-to-child chain).
std::vector<std::vector<int32_t>> heavy_pieces(const std::vector<int32_t>& par, int K) {
    std::vector<std::vector<int32_t>> pieces;
    for (auto& path : heavy_paths(par))
        for (size_t i = 0; i < path.size(); i += (size_t)K)
            pieces.emplace_back(path.begin() + (long)i, path.begin() + (long)std::min(path.size(), i + (size_t)K));
    return pieces;
}

// First-fit-decreasing packing of pieces into lists of at most K joints.
std::vector<std::vector<int32_t>> pack_pieces(std::vector<std::vector<int32_t>> pieces, int K) {
    std::stable_sort(pieces.begin(), pieces.end(),
                     [](const std::vector<int32_t>& a, const std::vector<int32_t>& b) { return a.size() > b.size(); });
    std::vector<std::vector<int32_t>> lists;
    std::vector<int> room;
    for (auto& pc : pieces) {
        size_t i = 0;
        while (i < lists.size() && room[i] < (int)pc.size()) ++i;
        if (i == lists.size()) { lists.emplace_back(); room.push_back(K); }
        lists[i].insert(lists[i].end(), pc.begin(), pc.end());
        room[i] -= (int)pc.size();
    }
    return lists;
}

// Pairwise-swap local search over a sequence cut into quarter-warp groups of 8:
// item i contributes residue keys keys[i][d] (d = 0..D-1, -1 = no access); the cost
// of a group is sum_d max_r count(d, r) — the wavefronts its D 128-bit accesses
// take.  Swaps items between groups while the total cost drops.
void swap_search(std::vector<std::vector<int>>& keys, std::vector<int32_t>& perm, int D,
                 const std::vector<char>* movable = nullptr) {
    const int n = (int)perm.size();
    const int G = (n + 7) / 8;
    if (G < 2) return;
    std::vector<int> cnt((size_t)G * D * 8, 0);
    auto at = [&](int g, int d, int r) -> int& { return cnt[((size_t)g * D + d) * 8 + r]; };
    auto gmax = [&](int g, int d) { int m = 0; for (int r = 0; r < 8; ++r) m = std::max(m, at(g, d, r)); return m; };
    for (int i = 0; i < n; ++i)
        for (int d = 0; d < D; ++d)
            if (keys[perm[i]][d] >= 0) at(i / 8, d, keys[perm[i]][d])++;
    const int passes = n > 4096 ? 1 : (n > 1024 ? 3 : 8);   // O(n^2) per pass
    for (int pass = 0; pass < passes; ++pass) {
        bool improved = false;
        for (int i = 0; i < n; ++i)
            for (int j = (i / 8 + 1) * 8; j < n; ++j) {
                if (movable && (!(*movable)[i] || !(*movable)[j])) continue;
                const int gi = i / 8, gj = j / 8;
                int before = 0, after = 0;
                for (int d = 0; d < D; ++d) {
                    const int ki = keys[perm[i]][d], kj = keys[perm[j]][d];
                    if (ki == kj) continue;
                    before += gmax(gi, d) + gmax(gj, d);
                    if (ki >= 0) { at(gi, d, ki)--; at(gj, d, ki)++; }
                    if (kj >= 0) { at(gj, d, kj)--; at(gi, d, kj)++; }
                    after += gmax(gi, d) + gmax(gj, d);
                    if (ki >= 0) { at(gi, d, ki)++; at(gj, d, ki)--; }
                    if (kj >= 0) { at(gj, d, kj)++; at(gi, d, kj)--; }
                }
                if (after < before) {
                    for (int d = 0; d < D; ++d) {
                        const int ki = keys[perm[i]][d], kj = keys[perm[j]][d];
                        if (ki == kj) continue;
                        if (ki >= 0) { at(gi, d, ki)--; at(gj, d, ki)++; }
                        if (kj >= 0) { at(gj, d, kj)--; at(gi, d, kj)++; }
                    }
                    std::swap(perm[i], perm[j]);
                    improved = true;
                }
            }
        if (!improved) break;
    }
}

// Order lists so that each quarter warp (8 consecutive lists = threads) reads, at
// every step, joints whose smem residues (3*pos mod 8, i.e. pos mod 8) differ.
void order_lists(std::vector<std::vector<int32_t>>& lists, const std::vector<int32_t>& pos, int K) {
    std::vector<std::vector<int32_t>> out;
    out.reserve(lists.size());
    std::vector<char> taken(lists.size(), 0);
    size_t left = lists.size();
    while (left) {
        std::vector<std::array<char, 8>> used((size_t)K);
        for (auto& u : used) u.fill(0);
        for (int slot = 0; slot < 8 && left; ++slot) {
            size_t best = 0;
            int best_cost = 1 << 30;
            for (size_t i = 0; i < lists.size(); ++i) {
                if (taken[i]) continue;
                int cost = 0;
                for (size_t s = 0; s < lists[i].size(); ++s) cost += used[s][pos[lists[i][s]] & 7];
                cost = cost * 64 - (int)lists[i].size();     // prefer full lists on ties
                if (cost < best_cost) { best_cost = cost; best = i; }
            }
            taken[best] = 1;
            --left;
            for (size_t s = 0; s < lists[best].size(); ++s) used[s][pos[lists[best][s]] & 7] = 1;
            out.push_back(lists[best]);
        }
    }
    std::vector<std::vector<int>> keys(out.size(), std::vector<int>((size_t)K, -1));
    for (size_t i = 0; i < out.size(); ++i)
        for (size_t s = 0; s < out[i].size(); ++s) keys[i][s] = pos[out[i][s]] & 7;
    std::vector<int32_t> perm(out.size());
    for (size_t i = 0; i < out.size(); ++i) perm[i] = (int32_t)i;
    swap_search(keys, perm, K);
    lists.clear();
    for (int32_t i : perm) lists.push_back(out[i]);
}

// Bank-conflict-aware arrangement of the movable (packed) lanes.  A lane's list is
// a concatenation of pieces; the piece order inside a lane is free (each piece
// starts at an anchor or a root) and decides which joint the lane touches at each
// slot.  The cost is the swap_search model: per quarter-warp group of 8 lanes and
// per slot, the largest number of lanes whose joints share a 16-byte bank group
// (pos mod 8).  Simulated annealing over (a) swaps of two lanes between groups and
// (b) random piece orders of one lane, from a fixed seed (plans are reproducible);
// the best arrangement seen is kept.
void anneal_lists(std::vector<std::vector<int32_t>>& lists, const std::vector<char>& movable,
                  const std::vector<int32_t>& pos, const std::vector<int32_t>& par, int K) {
    const int n = (int)lists.size();
    std::vector<int> mov;
    for (int i = 0; i < n; ++i) if (movable[i]) mov.push_back(i);
    if (mov.size() < 2) return;
    auto key = [&](const std::vector<int32_t>& l, int s) { return s < (int)l.size() ? (pos[l[s]] & 7) : -1; };
    auto group_cost = [&](int g) {
        int cost = 0;
        for (int s = 0; s < K; ++s) {
            int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, m = 0;
            for (int i = 8 * g; i < std::min(n, 8 * g + 8); ++i) {
                const int k = key(lists[i], s);
                if (k >= 0) m = std::max(m, ++cnt[k]);
            }
            cost += m;
        }
        return cost;
    };
    auto pieces_of = [&](const std::vector<int32_t>& l) {
        std::vector<std::vector<int32_t>> pc;
        for (size_t k = 0; k < l.size(); ++k) {
            if (k == 0 || par[l[k]] != l[k - 1]) pc.emplace_back();
            pc.back().push_back(l[k]);
        }
        return pc;
    };
    uint64_t rng = 0x9E3779B97F4A7C15ull;
    auto next = [&]() {   // splitmix64
        uint64_t z = (rng += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    };
    auto uni = [&]() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); };
    int cur = 0;
    for (int g = 0; g < (n + 7) / 8; ++g) cur += group_cost(g);
    int best = cur;
    std::vector<std::vector<int32_t>> best_lists = lists;
    const long iters = std::min<long>(400000, 2000L * (long)mov.size());
    const double t0 = 1.5, t1 = 0.02;
    for (long it = 0; it < iters; ++it) {
        const double temp = t0 * std::pow(t1 / t0, (double)it / (double)iters);
        const int i = mov[next() % mov.size()];
        if (uni() < 0.5) {   // swap two lanes of different groups
            const int j = mov[next() % mov.size()];
            if (i / 8 == j / 8) continue;
            const int before = group_cost(i / 8) + group_cost(j / 8);
            std::swap(lists[i], lists[j]);
            const int delta = group_cost(i / 8) + group_cost(j / 8) - before;
            if (delta <= 0 || uni() < std::exp(-delta / temp)) cur += delta;
            else std::swap(lists[i], lists[j]);
        } else {             // reorder the pieces of one lane
            auto pc = pieces_of(lists[i]);
            if (pc.size() < 2) continue;
            for (size_t k = pc.size() - 1; k > 0; --k) std::swap(pc[k], pc[next() % (k + 1)]);
            std::vector<int32_t> cand;
            for (auto& p : pc) cand.insert(cand.end(), p.begin(), p.end());
            const int before = group_cost(i / 8);
            std::vector<int32_t> old = lists[i];
            lists[i] = cand;
            const int delta = group_cost(i / 8) - before;
            if (delta <= 0 || uni() < std::exp(-delta / temp)) cur += delta;
            else lists[i] = old;
        }
        if (cur < best) { best = cur; best_lists = lists; }
    }
    lists.swap(best_lists);
}

}  // namespace

ChunkDecomp decompose(const std::vector<int32_t>& par, int K, int mode, const std::vector<int32_t>* pos,
                      bool pad_to_warp) {
    const int32_t F = (int32_t)par.size();
    ChunkDecomp d;
    d.K = K;
    if (mode == CHUNK_CONSECUTIVE) {
        for (int32_t f = 0; f < F; f += K) {
            d.lists.emplace_back();
            for (int32_t g = f; g < std::min(F, f + K); ++g) d.lists.back().push_back(g);
        }
    } else if (mode == CHUNK_RUNS) {
        // Paths longer than K become RUNS: their pieces on consecutive lanes, so one
        // warp-shuffle segmented scan joins them (a run restarts at a warp boundary).
        // Shorter paths are packed per lane.  Lanes are per character from lane 0.
        auto paths = heavy_paths(par);
        std::stable_sort(paths.begin(), paths.end(),
                         [](const std::vector<int32_t>& a, const std::vector<int32_t>& b) { return a.size() > b.size(); });
        std::vector<std::vector<int32_t>> shortp;
        for (auto& path : paths) {
            if ((int)path.size() <= K) { shortp.push_back(path); continue; }
            for (size_t i = 0; i < path.size(); i += (size_t)K) {
                const int b = (i > 0 && d.lists.size() % 32 != 0) ? d.run_back.back() + 1 : 0;
                d.lists.emplace_back(path.begin() + (long)i, path.begin() + (long)std::min(path.size(), i + (size_t)K));
                d.run_back.push_back(b);
            }
        }
        const size_t nrun = d.lists.size();
        for (auto& l : pack_pieces(shortp, K)) { d.lists.push_back(l); d.run_back.push_back(0); }
        if (pad_to_warp) {
            d.lists.resize((d.lists.size() + 31) / 32 * 32);
            d.run_back.resize(d.lists.size(), 0);
        }
        if (pos && d.lists.size() > nrun) {   // conflict-aware order of the packed (movable) lanes
            std::vector<std::vector<int>> keys(d.lists.size(), std::vector<int>((size_t)K, -1));
            std::vector<char> movable(d.lists.size(), 0);
            for (size_t i = 0; i < d.lists.size(); ++i) {
                movable[i] = i >= nrun;
                for (size_t s = 0; s < d.lists[i].size(); ++s) keys[i][s] = (*pos)[d.lists[i][s]] & 7;
            }
            std::vector<int32_t> perm(d.lists.size());
            for (size_t i = 0; i < perm.size(); ++i) perm[i] = (int32_t)i;
            swap_search(keys, perm, K, &movable);
            std::vector<std::vector<int32_t>> out;
            for (int32_t i : perm) out.push_back(d.lists[i]);
            d.lists.swap(out);
            anneal_lists(d.lists, movable, *pos, par, K);
        }
    } else {
        d.lists = pack_pieces(heavy_pieces(par, K), K);
        // idle lanes of the last warp are free: empty lists give the ordering room
        if (pad_to_warp) d.lists.resize((d.lists.size() + 31) / 32 * 32);
        if (pos) order_lists(d.lists, *pos, K);
        if (pad_to_warp)   // keep empty lists only where the ordering placed them before a real one
            while (!d.lists.empty() && d.lists.back().empty()) d.lists.pop_back();
    }
    d.src.assign(F, SRC_ROOT);
    d.slot_of.assign(F, -1);
    if (d.run_back.size() != d.lists.size()) d.run_back.assign(d.lists.size(), 0);
    std::vector<int32_t> head(F);
    for (size_t li = 0; li < d.lists.size(); ++li) {
        const auto& L = d.lists[li];
        for (size_t i = 0; i < L.size(); ++i) {
            const int32_t f = L[i], q = par[f];
            if (q < 0) { d.src[f] = SRC_ROOT; head[f] = f; }
            else if (i > 0 && q == L[i - 1]) { d.src[f] = SRC_PREV; head[f] = head[q]; }
            else if (i == 0 && d.run_back[li] > 0) {   // joined by the warp scan: q = previous lane's tail
                d.src[f] = SRC_RUN;
                head[f] = head[q];
            } else { d.src[f] = q; head[f] = f; }
        }
    }
    std::vector<char> is_anchor(F, 0);
    for (int32_t f = 0; f < F; ++f)
        if (d.src[f] >= 0) is_anchor[d.src[f]] = 1;
    for (int32_t f = 0; f < F; ++f)
        if (is_anchor[f]) { d.slot_of[f] = (int32_t)d.slots.size(); d.slots.push_back(f); }
    d.link0.resize(d.slots.size());
    for (size_t s = 0; s < d.slots.size(); ++s) {
        int32_t h = head[d.slots[s]];
        d.link0[s] = d.src[h] >= 0 ? d.slot_of[d.src[h]] : -1;
    }
    d.head = head;
    return d;
}

namespace {

// Bank-conflict-aware numbering of the tile's anchor slots.  A 128-bit shared
// access of a quarter warp (8 lanes) is conflict-free when the 8 addresses fall in
// distinct 16-byte bank groups; a P entry is 48 B = 3 groups, so slot s touches
// groups (3s + k) mod 8 and 8 slots are conflict-free iff their residues mod 8
// differ.  The sets that must differ are: the anchors one quarter warp reads in
// the same phase-3 step, and the anchors it writes in the same phase-1 step.
// Greedy colouring with 8 colours (residues), balanced class sizes; slot =
// colour + 8 * rank within the colour.  Returns the new index of every raw slot
// and the padded slot count (a multiple of 8, so ping-pong buffers keep residues).
std::vector<int32_t> colour_slots(int32_t S, const std::vector<std::vector<int32_t>>& sets,
                                  int32_t* S_out) {
    std::vector<std::vector<int32_t>> member(S);
    for (int32_t k = 0; k < (int32_t)sets.size(); ++k)
        for (int32_t s : sets[k]) member[s].push_back(k);
    std::vector<int32_t> order(S);
    for (int32_t s = 0; s < S; ++s) order[s] = s;
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return member[a].size() > member[b].size(); });
    std::vector<int32_t> colour(S, -1), count(8, 0);
    const int32_t cap = (S + 7) / 8 + 1;
    for (int32_t s : order) {
        int conflicts[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int32_t k : member[s])
            for (int32_t o : sets[k])
                if (o != s && colour[o] >= 0) conflicts[colour[o]]++;
        int best = -1;
        for (int c = 0; c < 8; ++c) {
            if (count[c] >= cap) continue;
            if (best < 0 || conflicts[c] < conflicts[best] ||
                (conflicts[c] == conflicts[best] && count[c] < count[best]))
                best = c;
        }
        colour[s] = best;
        count[best]++;
    }
    int32_t maxc = 0;
    for (int c = 0; c < 8; ++c) maxc = std::max(maxc, count[c]);
    std::vector<int32_t> next(8, 0), idx(S);
    for (int32_t s = 0; s < S; ++s) idx[s] = colour[s] + 8 * next[colour[s]]++;
    *S_out = 8 * maxc;
    return idx;
}

// Order one round's entries so every aligned run of 8 (one quarter warp) has
// distinct self residues and distinct link residues where possible.
void order_round(std::vector<std::array<int32_t, 3>>& ent) {   // {dst, self, link} locations
    std::vector<std::vector<std::array<int32_t, 3>>> bucket(8);
    for (auto& e : ent) bucket[e[1] & 7].push_back(e);
    std::vector<std::array<int32_t, 3>> out;
    out.reserve(ent.size());
    size_t left = ent.size();
    while (left) {
        bool used_s[8] = {}, used_l[8] = {};
        for (int pos = 0; pos < 8 && left; ++pos) {
            int bs = -1;
            size_t bi = 0;
            // 1) an unused self residue with an entry whose link residue is unused
            for (int c = 0; c < 8 && bs < 0; ++c) {
                if (used_s[c]) continue;
                for (size_t i = 0; i < bucket[c].size(); ++i)
                    if (!used_l[bucket[c][i][2] & 7]) { bs = c; bi = i; break; }
            }
            // 2) else any entry with an unused self residue (largest bucket first)
            if (bs < 0) {
                for (int c = 0; c < 8; ++c)
                    if (!used_s[c] && !bucket[c].empty() && (bs < 0 || bucket[c].size() > bucket[bs].size())) bs = c;
                bi = 0;
            }
            // 3) else anything
            if (bs < 0) {
                for (int c = 0; c < 8; ++c)
                    if (!bucket[c].empty() && (bs < 0 || bucket[c].size() > bucket[bs].size())) bs = c;
                bi = 0;
            }
            auto e = bucket[bs][bi];
            bucket[bs].erase(bucket[bs].begin() + (long)bi);
            used_s[e[1] & 7] = true;
            used_l[e[2] & 7] = true;
            out.push_back(e);
            --left;
        }
    }
    std::vector<std::vector<int>> keys(out.size(), std::vector<int>(2));
    for (size_t i = 0; i < out.size(); ++i) { keys[i][0] = out[i][1] & 7; keys[i][1] = out[i][2] & 7; }
    std::vector<int32_t> perm(out.size());
    for (size_t i = 0; i < out.size(); ++i) perm[i] = (int32_t)i;
    swap_search(keys, perm, 2);
    ent.clear();
    for (int32_t i : perm) ent.push_back(out[i]);
}

}  // namespace

TileProgram build_tile_program(const Plan& p, int K, int C, bool pingpong, int mode) {
    // Chunks never straddle characters: every character of a tile runs the same
    // program (same association order), so a character's bits do not depend on
    // its position in the batch, the tile size or the GPU count.
    TileProgram tp;
    const int32_t n = p.n;
    std::vector<int32_t> pos(n);               // smem position (joint index) of internal i
    for (int32_t i = 0; i < n; ++i) pos[i] = p.order[i];
    const ChunkDecomp d = decompose(p.ipar, K, mode, &pos, C == 1 || mode == CHUNK_RUNS);
    const int32_t TC = (int32_t)d.lists.size();   // chunks (threads) per character
    tp.lists_nonempty = 0;
    for (auto& l : d.lists) tp.lists_nonempty += l.empty() ? 0 : 1;
    const int32_t Sc = (int32_t)d.slots.size();
    tp.K = K;
    tp.C = C;
    tp.F = C * n;
    tp.T = C * TC;
    tp.pingpong = pingpong;
    const int32_t Sraw = C * Sc;
    // conflict sets (quarter warp x step) for phase-3 reads and phase-1 writes
    std::vector<std::vector<int32_t>> sets;
    {
        std::vector<std::vector<int32_t>> rd((size_t)((tp.T + 7) / 8) * K), wr(rd.size());
        for (int c = 0; c < C; ++c)
            for (int32_t tc = 0; tc < TC; ++tc) {
                const int32_t t = c * TC + tc;
                for (int s = 0; s < (int)d.lists[tc].size(); ++s) {
                    const int32_t i = d.lists[tc][s];
                    const size_t k = (size_t)(t / 8) * K + s;
                    if (d.src[i] >= 0) rd[k].push_back(c * Sc + d.slot_of[d.src[i]]);
                    if (d.slot_of[i] >= 0) wr[k].push_back(c * Sc + d.slot_of[i]);
                }
            }
        for (auto& v : rd) if (v.size() > 1) sets.push_back(v);
        for (auto& v : wr) if (v.size() > 1) sets.push_back(v);
    }
    int32_t S = 0;
    const std::vector<int32_t> idx = Sraw ? colour_slots(Sraw, sets, &S) : std::vector<int32_t>();
    tp.nslots = S;
    // pointer-jumping rounds over the tile's anchor forest (C disjoint copies)
    std::vector<int32_t> lk(Sraw), latest(Sraw, 0);
    for (int c = 0; c < C; ++c)
        for (int32_t s = 0; s < Sc; ++s) lk[c * Sc + s] = d.link0[s] < 0 ? -1 : c * Sc + d.link0[s];
    tp.round_off.push_back(0);
    for (int r = 0;; ++r) {
        bool any = false;
        for (int32_t s = 0; s < Sraw; ++s) if (lk[s] >= 0) { any = true; break; }
        if (!any) break;
        std::vector<std::array<int32_t, 3>> ent;
        for (int32_t s = 0; s < Sraw; ++s) {
            if (lk[s] < 0) continue;
            // ping-pong: read buffer `latest`, write the other; single buffer: all reads of
            // a round precede its writes (two barriers), so every location is the slot.
            const int32_t wbuf = pingpong ? ((r + 1) & 1) : 0;
            ent.push_back({wbuf * S + idx[s], latest[s] * S + idx[s], latest[lk[s]] * S + idx[lk[s]]});
        }
        order_round(ent);
        // 32-bit descriptor: slot | dst buffer << 14 | self buffer << 15 | link location << 16
        for (auto& e : ent) {
            const uint32_t slot = (uint32_t)(e[1] % S), sbuf = (uint32_t)(e[1] / S), wbuf = (uint32_t)(e[0] / S);
            tp.rounds.push_back(slot | (wbuf << 14) | (sbuf << 15) | ((uint32_t)e[2] << 16));
        }
        tp.max_round_entries = std::max(tp.max_round_entries, (int32_t)ent.size());
        std::vector<int32_t> nl(Sraw, -1);
        for (int32_t s = 0; s < Sraw; ++s) {
            if (lk[s] < 0) continue;
            latest[s] = pingpong ? ((r + 1) & 1) : 0;
            nl[s] = lk[lk[s]];
        }
        lk.swap(nl);
        tp.round_off.push_back((int32_t)tp.rounds.size());
        tp.R2 = r + 1;
    }
    tp.meta.assign((size_t)tp.T * K, 0);
    tp.p1len.assign(tp.T, 0);
    for (int32_t tc = 0; tc < TC; ++tc)
        if (d.run_back[tc] > 0 || (tc + 1 < TC && d.run_back[tc + 1] > 0)) tp.has_runs = true;
    for (int c = 0; c < C; ++c)
        for (int32_t tc = 0; tc < TC; ++tc) {
            const int32_t t = c * TC + tc;
            // lane info: run_back (bits 8..15) and the run head's anchor P location + 1
            // (bits 16..31, 0 = none) for lanes joined by the warp scan
            const bool in_run = d.run_back[tc] > 0 || (tc + 1 < TC && d.run_back[tc + 1] > 0);
            int32_t info = 0;
            if (d.run_back[tc] > 0 && !d.lists[tc].empty()) {
                const int32_t h = d.head[d.lists[tc][0]];
                int32_t loc = -1;
                if (d.src[h] >= 0) {
                    const int32_t raw = c * Sc + d.slot_of[d.src[h]];
                    loc = latest[raw] * S + idx[raw];
                }
                info = (d.run_back[tc] << 8) | ((loc + 1) << 16);
            }
            for (int s = 0; s < K; ++s) {
                const bool has = s < (int)d.lists[tc].size();
                const int32_t i = has ? d.lists[tc][s] : -1;   // internal position within the character
                int32_t src = SRC_NONE, own = -1;
                uint64_t off = 0, ibu = 0;
                if (has) {
                    off = (uint64_t)(c * n + p.order[i]);
                    ibu = (uint64_t)p.order[i];
                    if (d.src[i] >= 0) {
                        const int32_t raw = c * Sc + d.slot_of[d.src[i]];
                        src = latest[raw] * S + idx[raw];
                    } else {
                        src = d.src[i];
                    }
                    own = d.slot_of[i] >= 0 ? idx[c * Sc + d.slot_of[i]] : -1;
                    if (own >= 0 || in_run) tp.p1len[t] = s + 1;   // runs need the whole piece product
                }
                tp.meta[(size_t)t * K + s] = off | (ibu << 16) | ((uint64_t)(uint16_t)(int16_t)src << 32) |
                                             ((uint64_t)(uint16_t)(int16_t)own << 48);
            }
            tp.p1len[t] |= info;
        }
    return tp;
}

SplitProgram build_split_program(const Plan& p, int K) {
    SplitProgram sp;
    sp.K = K;
    const int32_t n = p.n;
    ChunkDecomp d = decompose(p.ipar, K, CHUNK_HEAVY, nullptr, false);
    sp.nslots = (int32_t)d.slots.size();
    sp.nchunks = (int32_t)d.lists.size();
    sp.meta.assign((size_t)sp.nchunks * K * 4, 0);
    for (int32_t c = 0; c < sp.nchunks; ++c)
        for (int s = 0; s < K; ++s) {
            int32_t* m = &sp.meta[((size_t)c * K + s) * 4];
            if (s >= (int)d.lists[c].size()) { m[0] = 0; m[1] = SRC_NONE; m[2] = -1; m[3] = 0; continue; }
            const int32_t f = d.lists[c][s];
            m[0] = p.order[f];
            m[1] = d.src[f] >= 0 ? d.slot_of[d.src[f]] : d.src[f];
            m[2] = d.slot_of[f];
            m[3] = 0;
        }
    sp.anchor_parents = d.link0;
    return sp;
}

bool build_seq_program(const Plan& p, int K, int F, int mode, int max_threads, SeqProgram& sp) {
    // Tiles are runs of F consecutive INTERNAL positions (a topological order), so a
    // joint's parent is in its own tile or an earlier one.  A CTA runs a character's
    // tiles in order; each tile is one chunk/anchor program (build_tile_program with
    // C = 1) over its sub-forest, where
    //   * a joint whose parent is in an earlier tile ("external parent") starts a
    //     segment like a root, but its source is the parent's final global pose in a
    //     Q location (Q nodes are final roots of the anchor forest: pointer jumping
    //     links to them and stops);
    //   * the Q values of tile j: a parent in tile j - 1 is FORWARDED by the thread that
    //     computes it in phase 3 of tile j - 1 (a shared-memory store into tile j's Q
    //     buffer); the parents in tiles <= j - 2 form tile j's INBOX, a contiguous
    //     workspace range ordered by source tile: each source tile i writes its share
    //     (a contiguous sub-range) once it is done (the producer warp, coalesced stores
    //     from the finished tile in shared memory), and the inbox reaches tile j's Q
    //     buffer in ONE bulk copy issued when tile j - 2 is done.  Two Q buffers
    //     alternate with the tile index; inbox entries come first in Q.
    sp = SeqProgram();
    const int32_t n = p.n;
    if (F < 32 || n <= 0) return false;
    sp.K = K;
    sp.F = F;
    sp.KT = (n + F - 1) / F;
    const int KT = sp.KT;
    struct TileTmp {
        ChunkDecomp d;
        std::vector<int32_t> q_of;         // per local node with an external parent: Q index
        std::vector<int32_t> imports;      // Q index -> external parent (internal position)
        std::vector<int32_t> idx;          // raw slot -> coloured slot
        int S = 0;
        int32_t n_inbox = 0;               // imports[0 .. n_inbox): the workspace inbox
        int32_t inbox_base = 0;            // first workspace row of the inbox
    };
    std::vector<TileTmp> tmp(KT);
    for (int k = 0; k < KT; ++k) {
        TileTmp& tt = tmp[k];
        const int32_t a = k * F, nj = std::min(F, n - a);
        std::vector<int32_t> lpar(nj), pos(nj);
        tt.q_of.assign(nj, -1);
        std::vector<int32_t> qmap(a, -1);   // external parent -> Q index
        for (int32_t li = 0; li < nj; ++li) {
            const int32_t q = p.ipar[a + li];
            pos[li] = li;
            lpar[li] = q >= a ? q - a : -1;
            if (q >= 0 && q < a) {
                if (qmap[q] < 0) { qmap[q] = (int32_t)tt.imports.size(); tt.imports.push_back(q); }
                tt.q_of[li] = qmap[q];
            }
        }
        // Q order: the inbox (parents in tiles <= k - 2, by source position: grouped by
        // source tile), then the forwarded parents (tile k - 1)
        {
            std::vector<int32_t> order_q(tt.imports.size());
            for (size_t z = 0; z < order_q.size(); ++z) order_q[z] = (int32_t)z;
            std::stable_sort(order_q.begin(), order_q.end(), [&](int32_t x, int32_t y) {
                const bool fx = tt.imports[x] / F >= k - 1, fy = tt.imports[y] / F >= k - 1;
                if (fx != fy) return !fx;
                return tt.imports[x] < tt.imports[y];
            });
            std::vector<int32_t> newidx(order_q.size()), imp2(order_q.size());
            for (size_t z = 0; z < order_q.size(); ++z) {
                newidx[order_q[z]] = (int32_t)z;
                imp2[z] = tt.imports[order_q[z]];
            }
            tt.imports.swap(imp2);
            for (auto& q : tt.q_of)
                if (q >= 0) q = newidx[q];
            tt.n_inbox = 0;
            for (int32_t q : tt.imports)
                if (q / F < k - 1) ++tt.n_inbox;
        }
        tt.d = decompose(lpar, K, mode, &pos, true);
        const ChunkDecomp& d = tt.d;
        const int32_t T = (int32_t)d.lists.size();
        if (T > max_threads) return false;
        sp.T = std::max(sp.T, (T + 31) / 32 * 32);
        // bank-conflict-aware slot colours (as build_tile_program, one character)
        const int32_t Sraw = (int32_t)d.slots.size();
        std::vector<std::vector<int32_t>> sets;
        {
            std::vector<std::vector<int32_t>> rd((size_t)((T + 7) / 8) * K), wr(rd.size());
            for (int32_t t = 0; t < T; ++t)
                for (int s = 0; s < (int)d.lists[t].size(); ++s) {
                    const int32_t i = d.lists[t][s];
                    const size_t kk = (size_t)(t / 8) * K + s;
                    if (d.src[i] >= 0) rd[kk].push_back(d.slot_of[d.src[i]]);
                    if (d.slot_of[i] >= 0) wr[kk].push_back(d.slot_of[i]);
                }
            for (auto& v : rd) if (v.size() > 1) sets.push_back(v);
            for (auto& v : wr) if (v.size() > 1) sets.push_back(v);
        }
        tt.S = 0;
        if (Sraw) tt.idx = colour_slots(Sraw, sets, &tt.S);
        sp.S = std::max(sp.S, tt.S);
        sp.nQ = std::max(sp.nQ, (int)tt.imports.size());
        if (d.run_back.size() == d.lists.size())
            for (int32_t t = 0; t < T; ++t)
                if (d.run_back[t] > 0) sp.has_runs = true;
    }
    const int32_t S = sp.S, nQ = sp.nQ;
    auto qloc = [&](int k, int32_t z) { return 2 * S + (k & 1) * nQ + z; };
    if (S >= (1 << 12) || 2 * S + 2 * nQ >= (1 << 12) - 8 || F > 1024) return false;   // meta field widths
    // workspace: the inboxes of all tiles, back to back (rows of 48 B per CTA)
    for (int k = 0; k < KT; ++k) {
        tmp[k].inbox_base = sp.n_exp;
        sp.n_exp += tmp[k].n_inbox;
    }
    if (sp.n_exp >= (1 << 24)) return false;
    // encoded meta (seq_meta_* in kernels.cuh): off 10 | src + 8 13 | own + 1 13 | ex 16 | fwd 12
    auto enc = [](int32_t off, int32_t src, int32_t own, int32_t ex, int32_t fwd) {
        return (uint64_t)off | ((uint64_t)(src + 8) << 10) | ((uint64_t)(own + 1) << 23) | ((uint64_t)ex << 36) |
               ((uint64_t)fwd << 52);
    };
    sp.meta.assign((size_t)KT * sp.T * K, enc(0, SRC_NONE, -1, 0, 0));
    sp.p1len.assign((size_t)KT * sp.T, 0);
    sp.ib_user.assign((size_t)KT * F, -1);
    std::vector<std::vector<int32_t>> roff(KT);
    for (int k = 0; k < KT; ++k) {
        TileTmp& tt = tmp[k];
        const ChunkDecomp& d = tt.d;
        const int32_t a = k * F, nj = std::min(F, n - a);
        const int32_t T = (int32_t)d.lists.size();
        const int32_t Sraw = (int32_t)d.slots.size();
        const int32_t nq = (int32_t)tt.imports.size();
        // the next tile's Q index of each of this tile's joints it imports (forwarding)
        std::vector<int32_t> fwd_of(nj, -1);
        if (k + 1 < KT)
            for (size_t z = (size_t)tmp[k + 1].n_inbox; z < tmp[k + 1].imports.size(); ++z) {
                const int32_t q = tmp[k + 1].imports[z];
                if (q >= a) fwd_of[q - a] = (int32_t)z;
            }
        SeqTile st{};
        st.n_early = 0;
        st.nj = nj;
        st.T = T;
        // anchor forest: tile anchors 0..Sraw-1 (ping-pong), Q nodes Sraw..Sraw+nq-1 (final)
        std::vector<int32_t> lk(Sraw + nq, -1), latest(Sraw, 0);
        for (int32_t s = 0; s < Sraw; ++s) {
            const int32_t h = d.head[d.slots[s]];
            if (d.link0[s] >= 0) lk[s] = d.link0[s];
            else if (tt.q_of[h] >= 0) lk[s] = Sraw + tt.q_of[h];
        }
        auto loc = [&](int32_t x) { return x < Sraw ? latest[x] * S + tt.idx[x] : qloc(k, x - Sraw); };
        st.rounds_off = (int32_t)sp.rounds.size();
        roff[k].push_back(0);
        for (int r = 0;; ++r) {
            bool any = false;
            for (int32_t s = 0; s < Sraw; ++s) if (lk[s] >= 0) { any = true; break; }
            if (!any) break;
            std::vector<std::array<int32_t, 3>> ent;
            const int32_t wbuf = (r + 1) & 1;
            for (int32_t s = 0; s < Sraw; ++s)
                if (lk[s] >= 0) ent.push_back({wbuf * S + tt.idx[s], latest[s] * S + tt.idx[s], loc(lk[s])});
            order_round(ent);
            for (auto& e : ent) {
                const uint32_t slot = (uint32_t)(e[1] % S), sbuf = (uint32_t)(e[1] / S), wb = (uint32_t)(e[0] / S);
                sp.rounds.push_back(slot | (wb << 14) | (sbuf << 15) | ((uint32_t)e[2] << 16));
            }
            sp.max_entries = std::max(sp.max_entries, (int)ent.size());
            std::vector<int32_t> nl(lk.size(), -1);
            for (int32_t s = 0; s < Sraw; ++s) {
                if (lk[s] < 0) continue;
                latest[s] = wbuf;
                nl[s] = lk[s] < Sraw ? lk[lk[s]] : -1;   // a Q node is a root: the chain ends
            }
            lk.swap(nl);
            roff[k].push_back((int32_t)sp.rounds.size() - st.rounds_off);
            st.R2 = r + 1;
        }
        st.n_entries = (int32_t)sp.rounds.size() - st.rounds_off;
        while (sp.rounds.size() % 4) sp.rounds.push_back(0);   // 16-byte tile records (TMA)
        sp.R2max = std::max(sp.R2max, st.R2);
        // per-thread program
        for (int32_t t = 0; t < T; ++t) {
            const bool in_run = d.run_back[t] > 0 || (t + 1 < T && d.run_back[t + 1] > 0);
            int32_t info = 0;
            if (d.run_back[t] > 0 && !d.lists[t].empty()) {
                const int32_t h = d.head[d.lists[t][0]];
                int32_t l = -1;
                if (d.src[h] >= 0) l = loc(d.slot_of[d.src[h]]);
                else if (tt.q_of[h] >= 0) l = qloc(k, tt.q_of[h]);
                info = (d.run_back[t] << 8) | ((l + 1) << 16);
            }
            int32_t& p1 = sp.p1len[(size_t)k * sp.T + t];
            for (int s = 0; s < K; ++s) {
                if (s >= (int)d.lists[t].size()) continue;
                const int32_t li = d.lists[t][s];
                int32_t src;
                if (d.src[li] >= 0) src = loc(d.slot_of[d.src[li]]);
                else if (d.src[li] == SRC_ROOT && tt.q_of[li] >= 0) src = qloc(k, tt.q_of[li]);
                else src = d.src[li];
                const int32_t own = d.slot_of[li] >= 0 ? tt.idx[d.slot_of[li]] : -1;
                if (own >= 0 || in_run) p1 = s + 1;
                const int32_t fw = fwd_of[li] + 1;
                sp.meta[((size_t)k * sp.T + t) * K + s] = enc(li, src, own, 0, fw);
            }
            p1 |= info;
        }
        // the inbox (workspace rows read by tile k) and the export list of tile k: for
        // every later tile j >= k + 2, its inbox entries whose parent is in tile k (a
        // contiguous sub-range, rows ascending): (smem offset in tile k, workspace row)
        st.n_imp = tt.n_inbox;
        st.imp_off = tt.inbox_base;
        for (int32_t z = 0; z < tt.n_inbox; ++z)   // the inbox is sorted by parent: a prefix
            if (tt.imports[z] / F <= k - 3) st.n_early = z + 1;
        st.exl_off = (int32_t)sp.exl.size() / 2;
        for (int j = k + 2; j < KT; ++j)
            for (int32_t z = 0; z < tmp[j].n_inbox; ++z) {
                const int32_t q = tmp[j].imports[z];
                if (q / F != k) continue;
                sp.exl.push_back(q - a);
                sp.exl.push_back(tmp[j].inbox_base + z);
                ++st.n_exl;
            }
        while (sp.exl.size() % 4) sp.exl.push_back(0);   // 16-byte tile records (TMA)
        sp.max_exl = std::max(sp.max_exl, (st.n_exl + 1) & ~1);
        st.runs_off = (int32_t)sp.runs.size() / 4;
        for (int32_t li = 0; li < nj;) {
            int32_t len = 1;
            while (li + len < nj && p.order[a + li + len] == p.order[a + li] + len) ++len;
            sp.runs.insert(sp.runs.end(), {p.order[a + li], li, len, 0});
            li += len;
            ++st.n_runs;
        }
        for (int32_t li = 0; li < nj; ++li) sp.ib_user[(size_t)k * F + li] = p.order[a + li];
        sp.max_imp = std::max(sp.max_imp, st.n_imp);
        if (3 * st.n_early > kSeqInboxPiecesPerThread * sp.T ||               // register-staged inbox
            3 * (st.n_imp - st.n_early) > kSeqInboxLatePerThread * sp.T)
            return false;
        sp.max_runs = std::max(sp.max_runs, st.n_runs);
        sp.tiles.push_back(st);
    }
    const int R2P = (sp.R2max + 1 + 3) & ~3;   // round_off rows padded to 16 bytes (TMA)
    sp.round_off.assign((size_t)KT * R2P, 0);
    for (int k = 0; k < KT; ++k)
        for (int r = 0; r < R2P; ++r)
            sp.round_off[(size_t)k * R2P + r] = roff[k][std::min<size_t>(r, roff[k].size() - 1)];
    return true;
}

int64_t seq_max_tile_entries(const SeqProgram& sp) {
    int64_t maxe = 0;
    for (const SeqTile& t : sp.tiles) maxe = std::max<int64_t>(maxe, t.n_entries);
    return maxe;
}

int64_t seq_smem_bytes(const SeqProgram& sp, int stages, int sbufs) {
    // barriers | stages x tile | sbufs x tile | P (2S anchors + 2 x nQ Q buffers) |
    // 2 program buffers (meta | p1 | round_off | rounds | import list) | tile descriptors
    const int64_t tileb = (int64_t)sp.F * 48;
    int64_t b = 256 + (int64_t)(stages + sbufs) * tileb + (int64_t)(2 * sp.S + 2 * sp.nQ) * 48;   // kSeqHeaderBytes
    b += 3 * 4 * seq_prog_words(sp);   // three program buffers
    b += (int64_t)sp.max_exl * 8;      // the export-list buffer
    b += (int64_t)sp.KT * (int64_t)sizeof(SeqTile);
    return b;
}

int64_t seq_prog_words(const SeqProgram& sp) {
    int64_t entp = 0;
    for (const SeqTile& t : sp.tiles) entp = std::max<int64_t>(entp, (t.n_entries + 3) & ~3);
    return 2LL * sp.T * sp.K + sp.T + ((sp.R2max + 1 + 3) & ~3) + entp;
}

void block_layout(const Plan& p, int B, std::vector<int32_t>& block_of, std::vector<int32_t>& mpob) {
    block_of.resize(p.n);
    mpob.assign(p.n, -1);
    for (int32_t i = 0; i < p.n; ++i) block_of[i] = i / B;
    for (int32_t i = 0; i < p.n; ++i) {
        int32_t a = p.ipar[i];
        while (a >= 0 && a / B == i / B) a = p.ipar[a];
        mpob[i] = a;
    }
}

void blocked_tables(const Plan& p, int B, std::vector<int32_t>& lb, std::vector<int32_t>& mpob, int& RB) {
    RB = 0;
    while ((1 << RB) < B) ++RB;
    const int32_t n = p.n;
    std::vector<int32_t> block_of, mi;
    block_layout(p, B, block_of, mi);
    lb.assign((size_t)std::max(RB, 1) * n, -1);
    mpob.assign(n, -1);
    for (int32_t i = 0; i < n; ++i) {
        const int32_t q = p.ipar[i];
        lb[p.order[i]] = (q >= 0 && q / B == i / B) ? p.order[q] : -1;
        mpob[p.order[i]] = mi[i] >= 0 ? p.order[mi[i]] : -1;
    }
    for (int r = 1; r < RB; ++r)
        for (int32_t u = 0; u < n; ++u) {
            const int32_t a = lb[(size_t)(r - 1) * n + u];
            lb[(size_t)r * n + u] = a >= 0 ? lb[(size_t)(r - 1) * n + a] : -1;
        }
}

void compressed_tables(const Plan& p, int B, std::vector<int32_t>& lp, std::vector<int32_t>& l8) {
    const int32_t n = p.n;
    lp.assign(n, -1);
    l8.assign(n, -1);
    for (int32_t i = 0; i < n; ++i) {
        const int32_t q = p.ipar[i];
        lp[p.order[i]] = (q >= 0 && q / B == i / B) ? p.order[q] : -1;
        int32_t a = i;
        for (int d = 0; d < 8 && a >= 0; ++d) {
            a = p.ipar[a];
            if (a >= 0 && a / B != i / B) a = -1;   // left the block: no in-block 8th ancestor
        }
        l8[p.order[i]] = a >= 0 ? p.order[a] : -1;
    }
}

int64_t tile_smem_bytes(const TileProgram& tp, int stages, int sbufs) {
    const int64_t tileb = (int64_t)tp.F * 48, pb = (tp.pingpong ? 2LL : 1LL) * tp.nslots * 48;
    const int64_t tables = ((int64_t)(tp.R2 + 1) * 4 + (int64_t)tp.rounds.size() * 4 + 15) / 16 * 16;
    return 128 + (int64_t)stages * tileb + (int64_t)sbufs * tileb + pb + tables;
}

}  // namespace hs
