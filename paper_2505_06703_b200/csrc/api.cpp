// api.cpp — the C ABI (include/hs.h): skeleton handles, scan dispatch, the
// host-only plan introspection, and the host-buffer pipeline.  DESIGN.md §2.
#include "../../include/hs.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "plan.hpp"

namespace {

thread_local std::string g_err;

hs_status fail(hs_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

hs_status cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? HS_ERR_OOM : HS_ERR_CUDA;
}

template <typename T>
cudaError_t upload(T** dptr, const T* host, size_t count) {
    *dptr = nullptr;
    if (count == 0) return cudaSuccess;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dptr), count * sizeof(T));
    if (e != cudaSuccess) return e;
    return cudaMemcpy(*dptr, host, count * sizeof(T), cudaMemcpyHostToDevice);
}

bool is_valid_k(int k) { return k >= 3 && k <= 11 && (k & 1); }

}  // namespace

struct hs_plan {
    hs::Plan plan;
    int K = 7;
    int block_size = 64;
    hs::ChunkDecomp decomp;
    hs::TileProgram tile;   // the chunked kernel's program for one character (ping-pong P)
    hs::SeqProgram seq;     // the multi-tile program (empty if no tile size fits)
    bool seq_ok = false;
};

struct hs_skeleton {
    int device = 0;
    hs::Plan plan;
    int K = 7;
    bool chunked = false;          // single-CTA chunked path fits
    hs::TileProgram tp;
    int stages = 0, sbufs = 0, threads = 0, chunking = 1;
    int64_t smem = 0;
    int smem_optin = 0;
    hs::SplitProgram sp;
    hs_skeleton* sub = nullptr;    // anchor skeleton of the split path
    hs_skeleton* small = nullptr;  // the same chunk program in smaller tiles, for small crowds
    int split_levels = 0;
    // device tables
    float* d_ib = nullptr;
    int32_t* d_parents = nullptr;
    int32_t* d_lift = nullptr;
    int32_t* d_blk_lift = nullptr;    // Alg. 3 comparison kernel: in-block lift [RB][n]
    int32_t* d_blk_mpob = nullptr;    //   and MaxParentOutBlock [n], user labels
    int32_t blk_rounds = 0;
    int32_t* d_cmp_lp = nullptr;      // Alg. 4 comparison kernel: in-block parent [n]
    int32_t* d_cmp_l8 = nullptr;      //   and in-block 8th ancestor [n], user labels
    uint64_t* d_meta = nullptr;
    int32_t* d_p1len = nullptr;
    int32_t* d_round_off = nullptr;
    uint32_t* d_rounds = nullptr;
    int32_t* d_split_meta = nullptr;
    int32_t* d_path_off = nullptr;
    int32_t* d_path = nullptr;
    int32_t n_leaves = 0;
    // multi-tile path (HS_ALGO_TILES): skeletons beyond one CTA
    bool seq_ok = false;
    hs::SeqProgram seq;
    int seq_stages = 0, seq_sbufs = 0, seq_threads = 0, seq_max_entries = 0, seq_K = 3, seq_helpers = 1;
    int64_t seq_smem = 0;
    hs::SeqTileDev* d_seq_tiles = nullptr;
    uint64_t* d_seq_meta = nullptr;
    int32_t* d_seq_p1len = nullptr;
    int32_t* d_seq_round_off = nullptr;
    uint32_t* d_seq_rounds = nullptr;
    int32_t* d_seq_imp = nullptr;
    int32_t* d_seq_runs = nullptr;
    float* d_seq_ib = nullptr;
};

struct hs_clipset {
    int device = 0;
    int32_t n_clips = 0, n_keys = 0, n_joints = 0, wrap = 0;
    float fps = 0.f, duration = 0.f;
    float* d_keys = nullptr;   // [n_clips][n_keys] rows of 10 * Jp floats (see hs_clipset_create)
};

struct hs_mesh {
    int device = 0;
    int32_t n_joints = 0, n_verts = 0;
    float4* d_a = nullptr;     // [V] (px, py, pz, w0)
    float4* d_b = nullptr;     // [V] (w1, w2, w3, 0)
    int2* d_j = nullptr;       // [V] packed 16-bit joint indices
    float4* d_sa = nullptr;    // the same three arrays sorted by joints (two-pass kernel);
    float4* d_sb = nullptr;    //   d_sb.w holds the output index bits
    int2* d_sj = nullptr;
};

struct hs_pipeline {
    int device = 0;
    int64_t batch_bytes = 0;
    cudaStream_t st[3] = {nullptr, nullptr, nullptr};
    float* d_in[3] = {nullptr, nullptr, nullptr};
    float* d_g[3] = {nullptr, nullptr, nullptr};
    float* d_s[3] = {nullptr, nullptr, nullptr};
};

namespace {

void free_skeleton(hs_skeleton* sk) {
    if (!sk) return;
    free_skeleton(sk->sub);
    free_skeleton(sk->small);
    cudaFree(sk->d_ib);
    cudaFree(sk->d_parents);
    cudaFree(sk->d_lift);
    cudaFree(sk->d_blk_lift);
    cudaFree(sk->d_blk_mpob);
    cudaFree(sk->d_cmp_lp);
    cudaFree(sk->d_cmp_l8);
    cudaFree(sk->d_meta);
    cudaFree(sk->d_p1len);
    cudaFree(sk->d_round_off);
    cudaFree(sk->d_rounds);
    cudaFree(sk->d_split_meta);
    cudaFree(sk->d_path_off);
    cudaFree(sk->d_path);
    cudaFree(sk->d_seq_tiles);
    cudaFree(sk->d_seq_meta);
    cudaFree(sk->d_seq_p1len);
    cudaFree(sk->d_seq_round_off);
    cudaFree(sk->d_seq_rounds);
    cudaFree(sk->d_seq_imp);
    cudaFree(sk->d_seq_runs);
    cudaFree(sk->d_seq_ib);
    delete sk;
}

// The multi-tile program (HS_ALGO_TILES) of a skeleton that does not fit one CTA.
// Defaults measured on C6 / C7 (2,000 x tree16384 in generation / depth-first label
// order; tools/tune_tiles.py): chunk K = 3, three load stages, two skin buffers (the
// next tile's inverse binds load during this tile), the largest tile up to 672 joints
// whose program fits 224 compute threads and whose shared memory fits the device (C6's
// many cross-tile parents need Q space: 576; C7: 672, 17 % faster than 576); chunking RUNS or HEAVY, whichever needs fewer phase-2
// descriptors.  Explicit options override each choice.
hs_status build_seq(hs_skeleton* sk, const hs_create_opts& o, const std::vector<float>& ib) {
    const hs::Plan& P = sk->plan;
    const int K = o.chunk ? o.chunk : 3;
    const int stages = o.stages ? o.stages : 3;
    const int f0 = o.tile_joints ? std::min(o.tile_joints, 1024) : 672;
    const int modes[2] = {hs::CHUNK_RUNS, hs::CHUNK_HEAVY};
    const int nmodes = o.chunking == 0 ? 2 : 1;
    const int sb_cand[2] = {o.sbufs ? o.sbufs : 2, o.sbufs ? o.sbufs : 1};
    for (int sbufs : sb_cand) {
        for (int F = f0 - f0 % 32; F >= 64 && !sk->seq_ok; F -= 32) {
            hs::SeqProgram best;
            bool have = false;
            for (int mi = 0; mi < nmodes; ++mi) {
                const int mode = o.chunking == 0 ? modes[mi]
                                 : (o.chunking == 1 ? hs::CHUNK_CONSECUTIVE
                                                    : (o.chunking == 3 ? hs::CHUNK_RUNS : hs::CHUNK_HEAVY));
                hs::SeqProgram sp;
                if (!hs::build_seq_program(P, K, F, mode, 224, sp)) continue;   // + the producer warp
                if (hs::seq_smem_bytes(sp, stages, sbufs) > sk->smem_optin) continue;
                if (!have || sp.rounds.size() < best.rounds.size()) { best = std::move(sp); have = true; }
            }
            if (!have) continue;
            sk->seq = std::move(best);
            sk->seq_ok = true;
            sk->seq_sbufs = sbufs;
        }
        if (sk->seq_ok) break;
    }
    if (!sk->seq_ok) return HS_OK;   // the split path remains
    const hs::SeqProgram& sp = sk->seq;
    sk->seq_stages = stages;
    sk->seq_K = K;
    sk->seq_smem = hs::seq_smem_bytes(sp, stages, sk->seq_sbufs);
    sk->seq_threads = sp.T + 32;   // consumers and the TMA producer warp
    sk->seq_max_entries = (int)hs::seq_max_tile_entries(sp);
    std::vector<hs::SeqTileDev> tiles(sp.tiles.size());
    static_assert(sizeof(hs::SeqTileDev) == sizeof(hs::SeqTile), "SeqTile layout");
    std::memcpy(tiles.data(), sp.tiles.data(), tiles.size() * sizeof(hs::SeqTile));
    std::vector<float> ibt((size_t)sp.KT * sp.F * 12, 0.f);
    for (size_t i = 0; i < sp.ib_user.size(); ++i)
        if (sp.ib_user[i] >= 0) std::memcpy(&ibt[i * 12], &ib[(size_t)sp.ib_user[i] * 12], 48);
    cudaError_t e;
    if ((e = upload(&sk->d_seq_tiles, tiles.data(), tiles.size())) != cudaSuccess ||
        (e = upload(&sk->d_seq_meta, sp.meta.data(), sp.meta.size())) != cudaSuccess ||
        (e = upload(&sk->d_seq_p1len, sp.p1len.data(), sp.p1len.size())) != cudaSuccess ||
        (e = upload(&sk->d_seq_round_off, sp.round_off.data(), sp.round_off.size())) != cudaSuccess ||
        (e = upload(&sk->d_seq_rounds, sp.rounds.data(), sp.rounds.size())) != cudaSuccess ||
        (e = upload(&sk->d_seq_imp, sp.exl.data(), sp.exl.size())) != cudaSuccess ||
        (e = upload(&sk->d_seq_runs, sp.runs.data(), sp.runs.size())) != cudaSuccess ||
        (e = upload(&sk->d_seq_ib, ibt.data(), ibt.size())) != cudaSuccess ||
        (e = hs::prepare_seq(K)) != cudaSuccess)
        return cuda_fail(e, "multi-tile program");
    return HS_OK;
}

hs_status create_impl(const int32_t* parents, int32_t n, const float* inv_bind,
                      const hs_create_opts& o, hs_skeleton** out, int depth) {
    if (!out) return fail(HS_ERR_INVALID_ARG, "out is null");
    if ((o.chunk && !is_valid_k(o.chunk)) || o.tile_joints < 0 || (o.stages && (o.stages < 2 || o.stages > 3)) ||
        (o.sbufs && (o.sbufs < 1 || o.sbufs > 2)) || o.force_split < 0 || o.force_split > 1 ||
        o.pbuf < 0 || o.pbuf > 2 || o.chunking < 0 || o.chunking > 3 || o.reserved[0])
        return fail(HS_ERR_INVALID_ARG, "invalid hs_create_opts");
    if (depth > 32) return fail(HS_ERR_UNSUPPORTED, "split recursion too deep");
    hs_skeleton* sk = new (std::nothrow) hs_skeleton();
    if (!sk) return fail(HS_ERR_OOM, "host allocation failed");
    std::string err;
    int st = hs::build_plan(parents, n, sk->plan, err);
    if (st != 0) { delete sk; return fail((hs_status)st, err); }
    cudaError_t e = cudaGetDevice(&sk->device);
    if (e != cudaSuccess) { delete sk; return cuda_fail(e, "cudaGetDevice"); }
    int smem_optin = 0;
    e = cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, sk->device);
    if (e != cudaSuccess) { delete sk; return cuda_fail(e, "cudaDeviceGetAttribute"); }
    sk->smem_optin = smem_optin;

    const hs::Plan& P = sk->plan;
    sk->K = o.chunk ? o.chunk : 5;
    // --- chunked (single-CTA) program: C characters per tile, ~tile_target joints
    const int tile_target = o.tile_joints ? o.tile_joints : 1024;
    int C = std::max(1, tile_target / std::max(1, n));
    // chunk construction: heavy-path pieces cut anchors on branchy skeletons, but may need
    // more threads per character (smaller tiles); auto keeps them only when they do not
    int mode = o.chunking == 1 ? hs::CHUNK_CONSECUTIVE : (o.chunking == 3 ? hs::CHUNK_RUNS : hs::CHUNK_HEAVY);
    if (o.chunking == 0) {
        const hs::TileProgram a1 = hs::build_tile_program(P, sk->K, 1, true, hs::CHUNK_CONSECUTIVE);
        const hs::TileProgram a2 = hs::build_tile_program(P, sk->K, 1, true, hs::CHUNK_HEAVY);
        const bool fewer = a2.rounds.size() < a1.rounds.size();
        mode = (fewer && a2.lists_nonempty <= a1.lists_nonempty) ? hs::CHUNK_HEAVY : hs::CHUNK_CONSECUTIVE;
        // runs pad every character to whole warps; worth it for one-character tiles
        // whose pointer jumping they cut by half or more (measured: tree1024 -8%, and a
        // loss on 64/256-joint skeletons packed several per tile)
        const int tile_target = o.tile_joints ? o.tile_joints : 1024;
        if (tile_target / std::max(1, n) <= 1) {
            const hs::TileProgram a3 = hs::build_tile_program(P, sk->K, 1, true, hs::CHUNK_RUNS);
            const size_t best = std::min(a1.rounds.size(), a2.rounds.size());
            if (a3.rounds.size() * 2 <= best && a3.T <= 224) mode = hs::CHUNK_RUNS;
        }
    }
    sk->chunking = mode;
    const int64_t TC = hs::build_tile_program(P, sk->K, 1, true, mode).T;  // chunks per character
    const int max_chunks = 224;  // compute threads per CTA (launch bounds 256 with the producer warp)
    while (C > 1 && C * TC > max_chunks) --C;
    if (!(o.force_split && depth == 0) && C * TC <= max_chunks && (int64_t)C * n <= 65535) {
        // candidates in preference order: (stages, sbufs, ping-pong P)
        // (ping-pong P measured faster than the single buffer: one barrier per round)
        const int cand[][3] = {{3, 2, 1}, {3, 1, 1}, {2, 2, 1}, {2, 1, 1},
                               {3, 2, 0}, {3, 1, 0}, {2, 2, 0}, {2, 1, 0}};
        const int workers = (int)(((C * TC) + 31) / 32 * 32);
        hs::TileProgram tp_pp = hs::build_tile_program(P, sk->K, C, true, mode);
        hs::TileProgram tp_sb = hs::build_tile_program(P, sk->K, C, false, mode);
        const bool single_ok = tp_sb.max_round_entries <= 4 * workers;
        for (auto& c : cand) {
            if (o.stages && c[0] != o.stages) continue;
            if (o.sbufs && c[1] != o.sbufs) continue;
            if (o.pbuf && (c[2] ? 2 : 1) != o.pbuf) continue;
            if (!c[2] && !single_ok) continue;
            const hs::TileProgram& tp = c[2] ? tp_pp : tp_sb;
            const int64_t b = hs::tile_smem_bytes(tp, c[0], c[1]);
            if (b <= smem_optin && 2 * tp.nslots < 32768) {
                sk->tp = tp;
                sk->stages = c[0];
                sk->sbufs = c[1];
                sk->smem = b;
                sk->chunked = true;
                break;
            }
        }
    }

    // --- device tables shared by all paths
    std::vector<float> ib((size_t)n * 12);
    if (inv_bind) std::memcpy(ib.data(), inv_bind, ib.size() * sizeof(float));
    else
        for (int32_t j = 0; j < n; ++j)
            for (int k = 0; k < 12; ++k) ib[(size_t)j * 12 + k] = (k == 0 || k == 5 || k == 10) ? 1.f : 0.f;
    if ((e = upload(&sk->d_ib, ib.data(), ib.size())) != cudaSuccess ||
        (e = upload(&sk->d_parents, P.parents.data(), P.parents.size())) != cudaSuccess ||
        (e = upload(&sk->d_lift, P.lift.data(), P.lift.size())) != cudaSuccess) {
        free_skeleton(sk);
        return cuda_fail(e, "upload skeleton tables");
    }
    {   // the paper's 64-joint blocks for the Alg. 3 comparison kernel
        std::vector<int32_t> lb, mp;
        hs::blocked_tables(P, 64, lb, mp, sk->blk_rounds);
        std::vector<int32_t> lp, l8;
        hs::compressed_tables(P, 64, lp, l8);
        if ((e = upload(&sk->d_blk_lift, lb.data(), lb.size())) != cudaSuccess ||
            (e = upload(&sk->d_blk_mpob, mp.data(), mp.size())) != cudaSuccess ||
            (e = upload(&sk->d_cmp_lp, lp.data(), lp.size())) != cudaSuccess ||
            (e = upload(&sk->d_cmp_l8, l8.data(), l8.size())) != cudaSuccess) {
            free_skeleton(sk);
            return cuda_fail(e, "upload block tables");
        }
    }
    // root -> leaf paths for the KIYA leaf kernel (comparison algorithm)
    {
        std::vector<int32_t> off{0}, path;
        size_t total = 0;
        for (int32_t leaf : P.leaves) total += P.level[leaf];
        if (total <= (size_t)64 << 20) {
            std::vector<int32_t> tmp;
            for (int32_t leaf : P.leaves) {
                tmp.clear();
                for (int32_t v = leaf; v >= 0; v = P.parents[v]) tmp.push_back(v);
                path.insert(path.end(), tmp.rbegin(), tmp.rend());
                off.push_back((int32_t)path.size());
            }
            sk->n_leaves = (int32_t)P.leaves.size();
            if ((e = upload(&sk->d_path_off, off.data(), off.size())) != cudaSuccess ||
                (e = upload(&sk->d_path, path.data(), path.size())) != cudaSuccess) {
                free_skeleton(sk);
                return cuda_fail(e, "upload leaf paths");
            }
        }
    }
    if (sk->chunked) {
        const hs::TileProgram& tp = sk->tp;
        sk->threads = ((tp.T + 31) / 32) * 32 + 32;
        if ((e = upload(&sk->d_meta, tp.meta.data(), tp.meta.size())) != cudaSuccess ||
            (e = upload(&sk->d_p1len, tp.p1len.data(), tp.p1len.size())) != cudaSuccess ||
            (e = upload(&sk->d_round_off, tp.round_off.data(), tp.round_off.size())) != cudaSuccess ||
            (e = upload(&sk->d_rounds, tp.rounds.data(), tp.rounds.size())) != cudaSuccess ||
            (e = hs::prepare_chunked(sk->K, sk->smem)) != cudaSuccess) {
            free_skeleton(sk);
            return cuda_fail(e, "chunked program");
        }
        // Small crowds leave SMs idle with multi-character tiles (C1: 1,000 x hum32 is
        // 46 tiles of 22): a second program with the same chunks in tiles of
        // max(2n, 256) joints, used per call when the default tiles would not cover
        // the SMs (6.65 -> 5.24 us).  Same chunking and K, so every
        // character's arithmetic is identical: results do not depend on which runs.
        if (depth == 0 && sk->tp.C >= 4 && !o.tile_joints && sk->chunking != hs::CHUNK_RUNS) {
            hs_create_opts so = o;
            so.chunk = sk->K;
            so.chunking = sk->chunking + 1;
            so.tile_joints = std::max(2 * n, 256);
            hs_skeleton* small = nullptr;
            if (create_impl(parents, n, inv_bind, so, &small, depth + 1) == HS_OK) {
                if (small->chunked && small->tp.C >= 2 && small->tp.C < sk->tp.C && small->K == sk->K &&
                    small->chunking == sk->chunking)
                    sk->small = small;
                else
                    free_skeleton(small);
            }
        }
    } else {
        if (depth == 0) {
            hs_status s3 = build_seq(sk, o, ib);
            if (s3 != HS_OK) { free_skeleton(sk); return s3; }
        }
        sk->sp = hs::build_split_program(P, sk->K);
        if ((e = upload(&sk->d_split_meta, sk->sp.meta.data(), sk->sp.meta.size())) != cudaSuccess) {
            free_skeleton(sk);
            return cuda_fail(e, "split program");
        }
        if (sk->sp.nslots > 0) {
            hs_create_opts so = o;
            so.force_split = 0;
            hs_status s2 = create_impl(sk->sp.anchor_parents.data(), sk->sp.nslots, nullptr, so, &sk->sub,
                                       depth + 1);
            if (s2 != HS_OK) { free_skeleton(sk); return s2; }
            sk->split_levels = 1 + sk->sub->split_levels;
        } else {
            sk->split_levels = 1;
        }
    }
    *out = sk;
    return HS_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Common checks of a scan's pose buffers (hs_scan rules): non-null input and global
// output, 16-byte alignment, no aliasing between input and outputs, sizes in int64.
hs_status check_pose_buffers(const float* local, int64_t n_chars, int32_t n_joints, const float* gout,
                             const float* sout) {
    if (!local || !gout) return fail(HS_ERR_INVALID_ARG, "null buffer");
    if (!aligned16(local) || !aligned16(gout) || (sout && !aligned16(sout)))
        return fail(HS_ERR_INVALID_ARG, "buffers must be 16-byte aligned");
    if (local == gout || (sout && (local == sout || gout == sout)))
        return fail(HS_ERR_INVALID_ARG, "output aliases an input or the other output");
    if (n_chars > (INT64_MAX / 64) / std::max<int32_t>(n_joints, 1))
        return fail(HS_ERR_INVALID_ARG, "size overflow");
    return HS_OK;
}

// Stream-ordered workspaces (split path, two-pass Stage 1) come from a library-owned
// pool per device that keeps its memory (release threshold = max): after the first
// frame a workspace costs no driver allocation.  The process's default pool and
// PyTorch's allocator are left alone.
cudaMemPool_t g_pools[64] = {};
std::mutex g_pools_mu;

cudaError_t ws_alloc(void** p, size_t bytes, cudaStream_t st) {
    cudaMemPool_t* pools = g_pools;
    std::mutex& mu = g_pools_mu;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, st);
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool;
        if ((e = cudaMemPoolCreate(&pool, &props)) != cudaSuccess) return e;
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        pools[dev] = pool;
    }
    return cudaMallocFromPoolAsync(p, bytes, pools[dev], st);
}

static_assert(HS_MAX_BATCH <= hs::kMaxSegs, "one kernel segment per batch item");
static_assert(hs::kSeqInboxPiecesPerThread == hs::kSeqInboxPieces && hs::kSeqInboxLatePerThread == hs::kSeqInboxLate,
              "multi-tile inbox staging width");

struct ChunkItem {
    const hs_skeleton* sk;
    const float* local;
    int64_t n_chars;
    float* gout;
    float* sout;
};

// Segments + shared-memory layout of one chunked launch: stage and
// S buffers sized for the largest tile, P for the largest anchor set, tables for the
// largest program.  For one segment this is tile_smem_bytes() exactly.
void chunked_layout(const ChunkItem* items, int n, int stages, int sbufs, hs::ChunkedArgs& a) {
    int64_t tiles = 0;
    int max_f = 0, p_floats = 0, r2_max = 0, rounds_max = 0, max_t = 0;
    bool runs = false;
    a.nseg = n;
    for (int i = 0; i < n; ++i) {
        const hs_skeleton* sk = items[i].sk;
        const hs::TileProgram& tp = sk->tp;
        hs::SegArgs& s = a.seg[i];
        s.local = items[i].local; s.gout = items[i].gout; s.sout = items[i].sout; s.ib = sk->d_ib;
        s.meta = sk->d_meta; s.p1len = sk->d_p1len; s.round_off = sk->d_round_off; s.rounds = sk->d_rounds;
        s.n_chars = items[i].n_chars;
        s.tile_base = tiles;
        s.J = sk->plan.n; s.C = tp.C; s.F = tp.F; s.T = tp.T;
        s.nslots = tp.nslots; s.R2 = tp.R2;
        s.n_rounds_entries = (int32_t)tp.rounds.size();
        s.p_single = tp.pingpong ? 0 : 1;
        tiles += (items[i].n_chars + tp.C - 1) / tp.C;
        max_f = std::max(max_f, tp.F);
        p_floats = std::max(p_floats, (tp.pingpong ? 2 : 1) * tp.nslots * 12);
        r2_max = std::max(r2_max, tp.R2);
        rounds_max = std::max(rounds_max, (int)tp.rounds.size());
        max_t = std::max(max_t, tp.T);
        runs = runs || tp.has_runs;
    }
    a.total_tiles = tiles;
    a.tile_f = max_f * 12;
    a.p_floats = p_floats;
    a.r2_max = r2_max;
    a.stages = stages;
    a.sbufs = sbufs;
    const int64_t tables = ((int64_t)(r2_max + 1) * 4 + (int64_t)rounds_max * 4 + 15) / 16 * 16;
    a.smem_bytes = 128 + (int64_t)(stages + sbufs) * max_f * 48 + (int64_t)p_floats * 4 + tables;
    a.threads = ((max_t + 31) / 32) * 32 + 32;
    a.has_runs = runs ? 1 : 0;
    a.bulk_piece = HS_BULK_PIECE;   // compile-time (kernels.cuh); tuning builds pass -DHS_BULK_PIECE=...
}

// Launch one chunked program (with the HS_DEBUG_PROF phase profile when set).
hs_status run_chunked(hs::ChunkedArgs& a, int K, cudaStream_t st) {
    a.prof = nullptr;
    if (HS_PROF_HOOKS && std::getenv("HS_DEBUG_PROF")) {   // profiling builds only: per-phase cycle split, synchronising
        cudaMalloc(reinterpret_cast<void**>(&a.prof), 10 * sizeof(unsigned long long));
        cudaMemsetAsync(a.prof, 0, 10 * sizeof(unsigned long long), st);
    }
    cudaError_t e = hs::launch_chunked(K, a, st);
    if (e != cudaSuccess) {
        char buf[256];
        std::snprintf(buf, sizeof(buf), "chunked launch (K=%d threads=%d smem=%lld stages=%d sbufs=%d)",
                      K, a.threads, (long long)a.smem_bytes, a.stages, a.sbufs);
        return cuda_fail(e, buf);
    }
    if (a.prof) {
        unsigned long long h[10];
        cudaMemcpyAsync(h, a.prof, sizeof(h), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        if (!h[5]) std::fprintf(stderr, "[hs prof] no samples: build with -DHS_PROF_HOOKS=1 (tools/prof_scan.py does)\n");
        const double n = h[5] ? (double)h[5] : 1.0;
        std::fprintf(stderr,
                     "[hs prof] J=%d tiles=%llu cycles/tile: wait_full %.0f stage1 %.0f phase1 %.0f phase2 %.0f "
                     "wait_sbuf %.0f phase3 %.0f (thread 0: fold %.0f scan+lift %.0f)\n",
                     a.seg[0].J, h[5], h[0] / n, h[8] / n, (h[1] + h[6] + h[7]) / n, h[2] / n, h[3] / n, h[4] / n,
                     h[6] / n, h[7] / n);
        cudaFree(a.prof);
    }
    return HS_OK;
}

hs_status scan_impl(const hs_skeleton* sk, const float* local, int64_t n_chars, float* gout,
                    float* sout, cudaStream_t st, int algo, int max_rounds, int tile_ctas,
                    const hs_clipset* cs = nullptr, const void* layers = nullptr, int n_layers = 0) {
    const int32_t J = sk->plan.n;
    cudaError_t e = cudaSuccess;
    if (algo == HS_ALGO_AUTO)
        algo = sk->chunked ? HS_ALGO_CHUNKED
                           : (sk->seq_ok && n_chars >= hs::sm_count() ? HS_ALGO_TILES : HS_ALGO_SPLIT);
    switch (algo) {
        case HS_ALGO_CHUNKED: {
            if (!sk->chunked) return fail(HS_ERR_UNSUPPORTED, "skeleton does not fit the single-CTA path");
            if (!layers && tile_ctas == 0 && sk->small && (n_chars + sk->tp.C - 1) / sk->tp.C < hs::sm_count())
                return scan_impl(sk->small, local, n_chars, gout, sout, st, algo, max_rounds, tile_ctas);
            hs::ChunkedArgs a{};
            const ChunkItem item{sk, local, n_chars, gout, sout};
            chunked_layout(&item, 1, sk->stages, sk->sbufs, a);
            a.ctas_per_sm = tile_ctas;
            a.layers = layers;
            a.keys = cs ? cs->d_keys : nullptr;
            a.n_layers = n_layers;
            a.n_keys = cs ? cs->n_keys : 0;
            a.wrap = cs ? cs->wrap : 0;
            a.fps = cs ? cs->fps : 0.f;
            a.duration = cs ? cs->duration : 0.f;
            a.desc_off = 0;
            if (layers) {
                // Stage 1: a [stages][C * n_layers] int4 descriptor ring after the tables;
                // a third stage is dropped if the ring does not fit beside it
                for (;;) {
                    const int64_t base = hs::tile_smem_bytes(sk->tp, a.stages, a.sbufs);
                    const int64_t need = base + (int64_t)a.stages * sk->tp.C * n_layers * 16;
                    if (need <= sk->smem_optin) {
                        a.desc_off = (int32_t)base;
                        a.smem_bytes = need;
                        break;
                    }
                    if (a.stages <= 2)
                        return fail(HS_ERR_UNSUPPORTED, "no shared memory left for the Stage-1 descriptors");
                    --a.stages;
                    chunked_layout(&item, 1, a.stages, a.sbufs, a);
                }
            }
            if (hs_status r = run_chunked(a, sk->K, st); r != HS_OK) return r;
            break;
        }
        case HS_ALGO_DOUBLING:
            if (J > 1024) return fail(HS_ERR_UNSUPPORTED, "doubling kernel needs n_joints <= 1024");
            e = hs::launch_doubling(local, gout, sout, sk->d_ib, sk->d_lift, J, sk->plan.R, max_rounds,
                                    n_chars, st);
            break;
        case HS_ALGO_BLOCKED:
            if (J > 1024) return fail(HS_ERR_UNSUPPORTED, "blocked kernel needs n_joints <= 1024");
            e = hs::launch_blocked(local, gout, sout, sk->d_ib, sk->d_blk_lift, sk->d_blk_mpob, J, sk->blk_rounds,
                                   n_chars, st);
            break;
        case HS_ALGO_COMPRESSED:
            if (J > 1024) return fail(HS_ERR_UNSUPPORTED, "compressed kernel needs n_joints <= 1024");
            e = hs::launch_compressed(local, gout, sout, sk->d_ib, sk->d_cmp_lp, sk->d_cmp_l8, sk->d_blk_mpob, J,
                                      n_chars, st);
            break;
        case HS_ALGO_GATEAU:
            e = hs::launch_gateau(local, gout, sout, sk->d_ib, sk->d_parents, J, n_chars, st);
            break;
        case HS_ALGO_LEAF:
            if (!sk->d_path) return fail(HS_ERR_UNSUPPORTED, "leaf paths too large");
            e = hs::launch_leaf(local, gout, sout, sk->d_ib, sk->d_path_off, sk->d_path, sk->n_leaves, J,
                                n_chars, st);
            break;
        case HS_ALGO_TILES: {
            if (!sk->seq_ok) return fail(HS_ERR_UNSUPPORTED, "skeleton has no multi-tile program (create with force_split=1)");
            const hs::SeqProgram& sp = sk->seq;
            hs::SeqArgs a{};
            a.local = local; a.gout = gout; a.sout = sout;
            a.ib = sk->d_seq_ib;
            a.tiles = sk->d_seq_tiles;
            a.meta = sk->d_seq_meta;
            a.p1len = sk->d_seq_p1len;
            a.round_off = sk->d_seq_round_off;
            a.rounds = sk->d_seq_rounds;
            a.exl = reinterpret_cast<const int2*>(sk->d_seq_imp);
            a.runs = reinterpret_cast<const int4*>(sk->d_seq_runs);
            a.n_chars = n_chars;
            a.J = J; a.KT = sp.KT; a.F = sp.F; a.T = sp.T; a.S = sp.S; a.nQ = sp.nQ; a.n_exp = sp.n_exp;
            a.r2max = sp.R2max; a.max_imp = sp.max_imp; a.max_entries = sk->seq_max_entries;
            a.p_floats = (2 * sp.S + 2 * sp.nQ) * 12;
            a.r2p = (sp.R2max + 1 + 3) & ~3;
            a.max_exl = sp.max_exl;
            a.entp = 0;
            for (const hs::SeqTile& tl : sp.tiles) a.entp = std::max(a.entp, (tl.n_entries + 3) & ~3);
            a.stages = sk->seq_stages; a.sbufs = sk->seq_sbufs; a.threads = sk->seq_threads;
            a.has_runs = sp.has_runs ? 1 : 0;
            a.bulk_piece = HS_BULK_PIECE;
            a.smem_bytes = sk->seq_smem;
            a.ctas_per_sm = tile_ctas > 0 ? tile_ctas : 1;
            // workspace: one character's exported poses per CTA (stays in L2)
            const int64_t grid = std::min<int64_t>(n_chars, (int64_t)hs::sm_count() * a.ctas_per_sm);
            float* ws = nullptr;
            if (sp.n_exp > 0) {
                e = ws_alloc(reinterpret_cast<void**>(&ws), (size_t)(grid * sp.n_exp * 48), st);
                if (e != cudaSuccess) return cuda_fail(e, "multi-tile workspace");
            }
            a.ws = ws;
            a.prof = nullptr;
            if (HS_PROF_HOOKS && std::getenv("HS_DEBUG_PROF")) {   // profiling builds only (synchronising)
                cudaMalloc(reinterpret_cast<void**>(&a.prof), 12 * sizeof(unsigned long long));
                cudaMemsetAsync(a.prof, 0, 12 * sizeof(unsigned long long), st);
            }
            e = hs::launch_seq(sk->seq_K, a, st);
            if (ws) cudaFreeAsync(ws, st);
            if (a.prof) {
                unsigned long long h[12];
                cudaMemcpyAsync(h, a.prof, sizeof(h), cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                const double nt = h[9] ? (double)h[9] : 1.0;
                std::fprintf(stderr,
                             "[hs prof seq] tiles=%llu cycles/tile: wait_prog %.0f read_prog %.0f wait_full %.0f "
                             "phase1 %.0f bar %.0f phase2 %.0f (mark) %.0f wait_ib %.0f phase3 %.0f "
                             "final_bar %.0f exports %.0f\n",
                             h[9], h[0] / nt, h[1] / nt, h[2] / nt, h[3] / nt, h[4] / nt, h[10] / nt, h[5] / nt,
                             h[6] / nt, h[7] / nt, h[8] / nt, h[11] / nt);
                cudaFree(a.prof);
            }
            break;
        }
        case HS_ALGO_SPLIT: {
            if (sk->chunked) {
                // forced split on a skeleton that fits one CTA: build on the fly is not
                // allowed (no host work on the hot path) — the handle has no split program.
                return fail(HS_ERR_UNSUPPORTED, "skeleton has no split program (create with force_split=1)");
            }
            const hs::SplitProgram& sp = sk->sp;
            const int64_t per_char = std::max<int64_t>(1, (int64_t)sp.nslots * 48);
            int64_t batch = std::max<int64_t>(1, ((int64_t)1 << 30) / per_char);
            batch = std::min(batch, n_chars);
            float* ws = nullptr;
            if (sp.nslots > 0) {
                e = ws_alloc(reinterpret_cast<void**>(&ws), (size_t)(2 * batch * per_char), st);
                if (e != cudaSuccess) return cuda_fail(e, "split workspace");
            }
            float* pg = ws;
            float* pf = ws ? ws + batch * sp.nslots * 12 : nullptr;
            for (int64_t c0 = 0; c0 < n_chars && e == cudaSuccess; c0 += batch) {
                const int64_t nb = std::min(batch, n_chars - c0);
                const float* lc = local + c0 * J * 12;
                if (sp.nslots > 0) {
                    e = hs::launch_split_p1(sk->K, lc, pg, sk->d_split_meta, sp.nchunks, J, sp.nslots, nb, st);
                    if (e != cudaSuccess) break;
                    hs_status s2 = scan_impl(sk->sub, pg, nb, pf, nullptr, st, HS_ALGO_AUTO, -1, tile_ctas);
                    if (s2 != HS_OK) { if (ws) cudaFreeAsync(ws, st); return s2; }
                }
                e = hs::launch_split_p3(sk->K, lc, gout + c0 * J * 12, sout ? sout + c0 * J * 12 : nullptr,
                                        sk->d_ib, pf, sk->d_split_meta, sp.nchunks, J, sp.nslots, nb, st);
            }
            if (ws) cudaFreeAsync(ws, st);
            break;
        }
        default:
            return fail(HS_ERR_INVALID_ARG, "unknown algo");
    }
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    return HS_OK;
}

}  // namespace

extern "C" {

hs_status hs_skeleton_create_ex(const int32_t* parents, int32_t n_joints, const float* inv_bind,
                                const hs_create_opts* opts, hs_skeleton** out) {
    hs_create_opts o;
    std::memset(&o, 0, sizeof(o));
    if (opts) o = *opts;
    try {
        return create_impl(parents, n_joints, inv_bind, o, out, 0);
    } catch (const std::bad_alloc&) {
        return fail(HS_ERR_OOM, "host allocation failed");
    } catch (...) {
        return fail(HS_ERR_INVALID_ARG, "unexpected exception in hs_skeleton_create");
    }
}

hs_status hs_skeleton_create(const int32_t* parents, int32_t n_joints, const float* inv_bind,
                             hs_skeleton** out) {
    return hs_skeleton_create_ex(parents, n_joints, inv_bind, nullptr, out);
}

hs_status hs_scan_ex(const hs_skeleton* sk, const float* local, int64_t n_chars, float* global_out,
                     float* skin_out, void* cuda_stream, const hs_scan_opts* opts) {
    if (!sk) return fail(HS_ERR_INVALID_ARG, "skeleton is null");
    if (n_chars < 0) return fail(HS_ERR_INVALID_ARG, "n_chars < 0");
    if (n_chars == 0) return HS_OK;
    if (hs_status r = check_pose_buffers(local, n_chars, sk->plan.n, global_out, skin_out); r != HS_OK) return r;
    int algo = HS_ALGO_AUTO, max_rounds = -1, tile_ctas = 0;
    if (opts) {
        algo = opts->algo;
        max_rounds = opts->max_rounds;
        tile_ctas = opts->tile_ctas;
        for (int i = 0; i < 5; ++i)
            if (opts->reserved[i]) return fail(HS_ERR_INVALID_ARG, "reserved option fields must be zero");
        if (max_rounds >= 0 && algo != HS_ALGO_DOUBLING)
            return fail(HS_ERR_INVALID_ARG, "max_rounds applies to HS_ALGO_DOUBLING only");
    }
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev != sk->device) return fail(HS_ERR_WRONG_DEVICE, "handle belongs to another device");
    return scan_impl(sk, local, n_chars, global_out, skin_out, static_cast<cudaStream_t>(cuda_stream),
                     algo, max_rounds, tile_ctas);
}

hs_status hs_scan_varied(const int32_t* parents, const float* local, const float* inv_bind, int32_t n_joints,
                         int64_t n_chars, float* global_out, float* skin_out, void* cuda_stream) {
    if (n_chars < 0 || n_joints < 0) return fail(HS_ERR_INVALID_ARG, "negative size");
    if (n_chars == 0 || n_joints == 0) return n_joints == 0 && n_chars > 0 ? fail(HS_ERR_EMPTY, "n_joints == 0")
                                                                          : HS_OK;
    if (n_joints > 1024) return fail(HS_ERR_UNSUPPORTED, "per-character topology needs n_joints <= 1024");
    if (!parents || !local || !global_out) return fail(HS_ERR_INVALID_ARG, "null buffer");
    if (!aligned16(local) || !aligned16(global_out) || (skin_out && !aligned16(skin_out)) ||
        (inv_bind && !aligned16(inv_bind)) || (reinterpret_cast<uintptr_t>(parents) & 3))
        return fail(HS_ERR_INVALID_ARG, "buffers must be 16-byte aligned (parents 4-byte)");
    if (local == global_out || (skin_out && (local == skin_out || global_out == skin_out)))
        return fail(HS_ERR_INVALID_ARG, "output aliases an input or the other output");
    if (n_chars > (INT64_MAX / 64) / n_joints) return fail(HS_ERR_INVALID_ARG, "size overflow");
    const cudaError_t e = hs::launch_varied(parents, local, inv_bind, n_joints, n_chars, global_out, skin_out,
                                            static_cast<cudaStream_t>(cuda_stream));
    return e == cudaSuccess ? HS_OK : cuda_fail(e, "varied-topology launch");
}

hs_status hs_scan_batch(const hs_batch_item* items, int32_t n_items, void* cuda_stream) {
    if (n_items < 0 || n_items > HS_MAX_BATCH) return fail(HS_ERR_INVALID_ARG, "n_items must be in 0..HS_MAX_BATCH");
    if (n_items > 0 && !items) return fail(HS_ERR_INVALID_ARG, "items is null");
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    ChunkItem segs[HS_MAX_BATCH];
    int n = 0, K = 0, stages = 3, sbufs = 2, optin = 0;
    for (int32_t i = 0; i < n_items; ++i) {
        const hs_batch_item& it = items[i];
        const hs_skeleton* sk = it.skeleton;
        if (!sk) return fail(HS_ERR_INVALID_ARG, "item skeleton is null");
        if (it.n_chars < 0) return fail(HS_ERR_INVALID_ARG, "n_chars < 0");
        if (it.n_chars == 0) continue;
        if (hs_status r = check_pose_buffers(it.local, it.n_chars, sk->plan.n, it.global_out, it.skin_out);
            r != HS_OK)
            return r;
        if (dev != sk->device) return fail(HS_ERR_WRONG_DEVICE, "handle belongs to another device");
        if (!sk->chunked) return fail(HS_ERR_UNSUPPORTED, "batched skeletons must fit the single-CTA path");
        if (K && sk->K != K) return fail(HS_ERR_UNSUPPORTED, "batched skeletons must share the chunk size K");
        K = sk->K;
        stages = std::min(stages, sk->stages);
        sbufs = std::min(sbufs, sk->sbufs);
        optin = sk->smem_optin;
        segs[n++] = ChunkItem{sk, it.local, it.n_chars, it.global_out, it.skin_out};
    }
    if (n == 0) return HS_OK;
    // small crowds: when the default tiles of all items together would leave SMs idle,
    // the small-tile twins (same chunks, bitwise the same results) take their place
    int64_t tiles = 0;
    for (int i = 0; i < n; ++i) tiles += (segs[i].n_chars + segs[i].sk->tp.C - 1) / segs[i].sk->tp.C;
    if (tiles < hs::sm_count())
        for (int i = 0; i < n; ++i)
            if (const hs_skeleton* s = segs[i].sk->small) {
                segs[i].sk = s;
                stages = std::min(stages, s->stages);
                sbufs = std::min(sbufs, s->sbufs);
            }
    hs::ChunkedArgs a{};
    for (;;) {   // the common layout of the largest tile / anchor set / program
        chunked_layout(segs, n, stages, sbufs, a);
        if (a.smem_bytes <= optin) break;
        if (sbufs > 1) --sbufs;
        else if (stages > 2) { --stages; sbufs = 2; }
        else return fail(HS_ERR_UNSUPPORTED, "batched programs do not fit shared memory together");
    }
    return run_chunked(a, K, static_cast<cudaStream_t>(cuda_stream));
}

hs_status hs_mesh_create(const hs_skeleton* sk, int32_t n_vertices, const float* pos, const int32_t* joints,
                         const float* weights, hs_mesh** out) {
    if (!sk || !pos || !joints || !weights || !out) return fail(HS_ERR_INVALID_ARG, "null argument");
    if (n_vertices < 1 || n_vertices > (1 << 24)) return fail(HS_ERR_INVALID_ARG, "n_vertices must be in 1..2^24");
    const int32_t J = sk->plan.n;
    if (J > 65535) return fail(HS_ERR_UNSUPPORTED, "meshes need n_joints <= 65535");
    const size_t V = (size_t)n_vertices;
    std::vector<float4> A(V), B(V);
    std::vector<int2> Jt(V);
    for (size_t v = 0; v < V; ++v) {
        for (int k = 0; k < 4; ++k) {
            const int32_t j = joints[4 * v + k];
            if (j < 0 || j >= J) return fail(HS_ERR_OUT_OF_RANGE, "mesh joint index out of range");
        }
        A[v] = make_float4(pos[3 * v], pos[3 * v + 1], pos[3 * v + 2], weights[4 * v]);
        B[v] = make_float4(weights[4 * v + 1], weights[4 * v + 2], weights[4 * v + 3], 0.f);
        Jt[v] = make_int2((int)((uint32_t)joints[4 * v] | ((uint32_t)joints[4 * v + 1] << 16)),
                          (int)((uint32_t)joints[4 * v + 2] | ((uint32_t)joints[4 * v + 3] << 16)));
    }
    // a second copy in processing order for the two-pass kernel: vertices sorted by
    // their joints (a quarter warp then mostly reads the same palette matrices:
    // shared-memory broadcasts), each record carrying its output index in B.w; that
    // kernel stages a character's vertices in smem and writes them out in order
    std::vector<int32_t> order(V);
    for (size_t v = 0; v < V; ++v) order[v] = (int32_t)v;
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
        for (int k = 0; k < 4; ++k)
            if (joints[4 * (size_t)x + k] != joints[4 * (size_t)y + k])
                return joints[4 * (size_t)x + k] < joints[4 * (size_t)y + k];
        return false;
    });
    std::vector<float4> SA(V), SBv(V);
    std::vector<int2> SJ(V);
    for (size_t i = 0; i < V; ++i) {
        const size_t v = (size_t)order[i];
        SA[i] = A[v];
        SBv[i] = B[v];
        const int32_t out_idx = (int32_t)v;
        std::memcpy(&SBv[i].w, &out_idx, 4);
        SJ[i] = Jt[v];
    }
    hs_mesh* m = new (std::nothrow) hs_mesh();
    if (!m) return fail(HS_ERR_OOM, "host allocation failed");
    cudaGetDevice(&m->device);
    m->n_joints = J;
    m->n_verts = n_vertices;
    cudaError_t e;
    if ((e = upload(&m->d_a, A.data(), V)) != cudaSuccess || (e = upload(&m->d_b, B.data(), V)) != cudaSuccess ||
        (e = upload(&m->d_j, Jt.data(), V)) != cudaSuccess || (e = upload(&m->d_sa, SA.data(), V)) != cudaSuccess ||
        (e = upload(&m->d_sb, SBv.data(), V)) != cudaSuccess || (e = upload(&m->d_sj, SJ.data(), V)) != cudaSuccess) {
        hs_mesh_destroy(m);
        return cuda_fail(e, "mesh upload");
    }
    *out = m;
    return HS_OK;
}

hs_status hs_mesh_destroy(hs_mesh* m) {
    if (!m) return HS_OK;
    cudaFree(m->d_a);
    cudaFree(m->d_b);
    cudaFree(m->d_j);
    cudaFree(m->d_sa);
    cudaFree(m->d_sb);
    cudaFree(m->d_sj);
    delete m;
    return HS_OK;
}

hs_status hs_scan_skin_ex(const hs_skeleton* sk, const hs_mesh* mesh, const float* local, int64_t n_chars,
                          float* global_out, float* skin_out, float* verts_out, void* cuda_stream,
                          const hs_skin_opts* opts) {
    if (!sk || !mesh) return fail(HS_ERR_INVALID_ARG, "null handle");
    if (n_chars < 0) return fail(HS_ERR_INVALID_ARG, "n_chars < 0");
    int mode = HS_SKIN_AUTO;
    int64_t ws_bytes = (int64_t)1 << 30;
    if (opts) {
        if (opts->mode < HS_SKIN_AUTO || opts->mode > HS_SKIN_TWO_PASS || opts->reserved0 || opts->reserved[0] ||
            opts->reserved[1] || opts->workspace_bytes < 0)
            return fail(HS_ERR_INVALID_ARG, "invalid hs_skin_opts");
        mode = opts->mode;
        if (opts->workspace_bytes) ws_bytes = opts->workspace_bytes;
    }
    if (n_chars == 0) return HS_OK;
    if (!local || !global_out || !verts_out) return fail(HS_ERR_INVALID_ARG, "null buffer");
    if (!aligned16(local) || !aligned16(global_out) || (skin_out && !aligned16(skin_out)) ||
        (reinterpret_cast<uintptr_t>(verts_out) & 3))
        return fail(HS_ERR_INVALID_ARG, "pose buffers must be 16-byte aligned, vertices 4-byte");
    if (local == global_out || (skin_out && (local == skin_out || global_out == skin_out)) ||
        verts_out == local || verts_out == global_out || verts_out == skin_out)
        return fail(HS_ERR_INVALID_ARG, "output aliases an input or another output");
    if (mesh->n_joints != sk->plan.n) return fail(HS_ERR_INVALID_ARG, "mesh built for another skeleton");
    if (n_chars > (INT64_MAX / 64) / std::max(sk->plan.n, mesh->n_verts))
        return fail(HS_ERR_INVALID_ARG, "size overflow");
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != sk->device || dev != mesh->device) return fail(HS_ERR_WRONG_DEVICE, "device mismatch");
    const cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    const int32_t J = sk->plan.n;
    // AUTO: two-pass when the mesh has at least twice as many vertices as the skeleton
    // has joints (its joint-sorted vertex order turns palette reads into broadcasts and
    // repays the extra 48 B/joint S round trip: hum64 / chain256 with 1000 vertices are
    // 24 % / 17 % faster), else the fused epilogue (tree1024: 13 % faster fused); and
    // two-pass wherever the fused path does not exist (multi-CTA skeletons)
    if (mode == HS_SKIN_AUTO) {
        const bool fits = (int64_t)J * 48 + (int64_t)mesh->n_verts * 12 <= 227 * 1024;
        mode = (!sk->chunked || (fits && mesh->n_verts >= 2 * J)) ? HS_SKIN_TWO_PASS : HS_SKIN_FUSED;
    }
    if (mode == HS_SKIN_FUSED) {
        if (!sk->chunked) return fail(HS_ERR_UNSUPPORTED, "the fused LBS epilogue needs a single-CTA skeleton");
        // small crowds: the small-tile twin (same chunks and vertices, more CTAs busy)
        const hs_skeleton* ps =
            sk->small && (n_chars + sk->tp.C - 1) / sk->tp.C < hs::sm_count() ? sk->small : sk;
        hs::ChunkedArgs a{};
        const ChunkItem item{ps, local, n_chars, global_out, skin_out};
        chunked_layout(&item, 1, ps->stages, ps->sbufs, a);
        a.mesh_a = mesh->d_a;
        a.mesh_b = mesh->d_b;
        a.mesh_j = mesh->d_j;
        a.verts = verts_out;
        a.n_verts = mesh->n_verts;
        return run_chunked(a, ps->K, st);
    }
    // two-pass: the scan writes S (to skin_out, or to a pooled workspace in
    // batches when the caller does not want S), then lbs_kernel skins from it
    if ((int64_t)J * 48 + (int64_t)mesh->n_verts * 12 > 227 * 1024)
        return fail(HS_ERR_UNSUPPORTED, "palette + vertices do not fit shared memory");
    const int64_t per_char = (int64_t)J * 48;
    const int64_t batch = skin_out ? n_chars : std::max<int64_t>(1, std::min<int64_t>(n_chars, ws_bytes / per_char));
    float* ws = nullptr;
    cudaError_t e = cudaSuccess;
    if (!skin_out && (e = ws_alloc(reinterpret_cast<void**>(&ws), (size_t)(batch * per_char), st)) != cudaSuccess)
        return cuda_fail(e, "LBS workspace");
    hs_status r = HS_OK;
    for (int64_t c0 = 0; c0 < n_chars && r == HS_OK; c0 += batch) {
        const int64_t nb = std::min(batch, n_chars - c0);
        float* sb = skin_out ? skin_out + c0 * J * 12 : ws;
        r = scan_impl(sk, local + c0 * J * 12, nb, global_out + c0 * J * 12, sb, st, HS_ALGO_AUTO, -1, 0);
        if (r == HS_OK &&
            (e = hs::launch_lbs(sb, nb, J, mesh->d_sa, mesh->d_sb, mesh->d_sj, mesh->n_verts,
                                verts_out + c0 * (int64_t)mesh->n_verts * 3, st)) != cudaSuccess)
            r = cuda_fail(e, "LBS launch");
    }
    if (ws) cudaFreeAsync(ws, st);
    return r;
}

hs_status hs_skin_vertices(const hs_mesh* mesh, const float* skin, int64_t n_chars, float* verts_out,
                           void* cuda_stream) {
    if (!mesh) return fail(HS_ERR_INVALID_ARG, "null handle");
    if (n_chars < 0) return fail(HS_ERR_INVALID_ARG, "n_chars < 0");
    if (n_chars == 0) return HS_OK;
    if (!skin || !verts_out) return fail(HS_ERR_INVALID_ARG, "null buffer");
    if (!aligned16(skin) || (reinterpret_cast<uintptr_t>(verts_out) & 3))
        return fail(HS_ERR_INVALID_ARG, "skin must be 16-byte aligned, vertices 4-byte");
    if (n_chars > (INT64_MAX / 64) / std::max(mesh->n_joints, mesh->n_verts))
        return fail(HS_ERR_INVALID_ARG, "size overflow");
    if ((int64_t)mesh->n_joints * 48 + (int64_t)mesh->n_verts * 12 > 227 * 1024)
        return fail(HS_ERR_UNSUPPORTED, "palette + vertices do not fit shared memory");
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != mesh->device) return fail(HS_ERR_WRONG_DEVICE, "device mismatch");
    const cudaError_t e = hs::launch_lbs(skin, n_chars, mesh->n_joints, mesh->d_sa, mesh->d_sb, mesh->d_sj,
                                         mesh->n_verts, verts_out, static_cast<cudaStream_t>(cuda_stream));
    return e == cudaSuccess ? HS_OK : cuda_fail(e, "LBS launch");
}

hs_status hs_scan_skin(const hs_skeleton* sk, const hs_mesh* mesh, const float* local, int64_t n_chars,
                       float* global_out, float* skin_out, float* verts_out, void* cuda_stream) {
    return hs_scan_skin_ex(sk, mesh, local, n_chars, global_out, skin_out, verts_out, cuda_stream, nullptr);
}

hs_status hs_clipset_create(const hs_skeleton* sk, const float* keys, int32_t n_clips, int32_t n_keys,
                            float fps, int32_t wrap, hs_clipset** out) {
    if (!sk || !keys || !out) return fail(HS_ERR_INVALID_ARG, "null argument");
    if (n_clips <= 0 || n_keys <= 0 || !(fps > 0.f) || wrap < 0 || wrap > 1)
        return fail(HS_ERR_INVALID_ARG, "n_clips, n_keys, fps must be positive; wrap 0 or 1");
    const int32_t J = sk->plan.n;
    const int64_t Jp = J + (J & 1);   // planes padded to 16 bytes
    if ((int64_t)n_clips * n_keys * Jp * 10 >= ((int64_t)1 << 31))   // int32 float offsets
        return fail(HS_ERR_INVALID_ARG, "clip set too large");
    hs_clipset* cs = new (std::nothrow) hs_clipset();
    if (!cs) return fail(HS_ERR_OOM, "host allocation failed");
    cudaGetDevice(&cs->device);
    cs->n_clips = n_clips; cs->n_keys = n_keys; cs->n_joints = J; cs->wrap = wrap; cs->fps = fps;
    cs->duration = (float)(n_keys - 1) / fps;   // same fp32 operation as the oracle (R20)
    // planar layout, 40 B per (key, joint): per (clip, key) row of 10 * Jp floats,
    // [Jp][4] {t, qw} | [Jp][4] {q.xyz, sx} | [Jp][2] {sy, sz} — consecutive joints on
    // consecutive lanes read contiguous bytes
    std::vector<float> packed((size_t)n_clips * n_keys * Jp * 10, 0.f);
    for (size_t row = 0; row < (size_t)n_clips * n_keys; ++row)
        for (int32_t j = 0; j < J; ++j) {
            const float* s = keys + (row * J + j) * 10;
            float* r = packed.data() + row * Jp * 10;
            for (int e = 0; e < 4; ++e) r[(size_t)j * 4 + e] = s[e];
            for (int e = 0; e < 4; ++e) r[(size_t)Jp * 4 + (size_t)j * 4 + e] = s[4 + e];
            for (int e = 0; e < 2; ++e) r[(size_t)Jp * 8 + (size_t)j * 2 + e] = s[8 + e];
        }
    cudaError_t e = upload(&cs->d_keys, packed.data(), packed.size());
    if (e != cudaSuccess) { delete cs; return cuda_fail(e, "clip upload"); }
    *out = cs;
    return HS_OK;
}

hs_status hs_clipset_destroy(hs_clipset* cs) {
    if (!cs) return HS_OK;
    cudaFree(cs->d_keys);
    delete cs;
    return HS_OK;
}

static hs_status animate_impl(const hs_skeleton* sk, const hs_clipset* cs, const void* layers, int32_t n_layers,
                       int64_t n_chars, float* global_out, float* skin_out, void* cuda_stream,
                       const hs_animate_opts* opts, const hs_mesh* mesh, float* verts_out) {
    if (!sk || !cs) return fail(HS_ERR_INVALID_ARG, "null handle");
    if (n_chars < 0) return fail(HS_ERR_INVALID_ARG, "n_chars < 0");
    int mode = HS_ANIMATE_AUTO;
    int64_t ws_bytes = (int64_t)1 << 30;
    if (opts) {
        if (opts->mode < HS_ANIMATE_AUTO || opts->mode > HS_ANIMATE_TWO_PASS || opts->reserved0 ||
            opts->reserved[0] || opts->reserved[1] || opts->workspace_bytes < 0)
            return fail(HS_ERR_INVALID_ARG, "invalid hs_animate_opts");
        mode = opts->mode;
        if (opts->workspace_bytes) ws_bytes = opts->workspace_bytes;
    }
    if (n_chars == 0) return HS_OK;
    if (!layers || !global_out) return fail(HS_ERR_INVALID_ARG, "null buffer");
    if (n_layers < 1 || n_layers > 8) return fail(HS_ERR_INVALID_ARG, "n_layers must be in 1..8");
    if (cs->n_joints != sk->plan.n) return fail(HS_ERR_INVALID_ARG, "clip set built for another skeleton");
    if (!aligned16(layers) || !aligned16(global_out) || (skin_out && !aligned16(skin_out)))
        return fail(HS_ERR_INVALID_ARG, "buffers must be 16-byte aligned");
    if (skin_out == global_out) return fail(HS_ERR_INVALID_ARG, "outputs alias");
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != sk->device || dev != cs->device) return fail(HS_ERR_WRONG_DEVICE, "device mismatch");
    const cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    if (mesh && mode == HS_ANIMATE_FUSED)
        return fail(HS_ERR_UNSUPPORTED, "Stage 1 + skinning runs the two-pass placement");
    if (mode == HS_ANIMATE_FUSED) {
        if (!sk->chunked) return fail(HS_ERR_UNSUPPORTED, "the fused Stage 1 needs a single-CTA skeleton");
        return scan_impl(sk, nullptr, n_chars, global_out, skin_out, st, HS_ALGO_CHUNKED, -1, 0, cs, layers,
                         n_layers);
    }
    // two-pass (and AUTO, measured faster on B200: DESIGN.md §5.1b): Stage 1 streams the
    // local poses of a batch of characters into a stream-ordered workspace, then the
    // plain chunked scan reads them back
    const int32_t J = sk->plan.n;
    const int64_t per_char = (int64_t)J * 48;
    const int64_t batch = std::max<int64_t>(1, std::min<int64_t>(n_chars, ws_bytes / per_char));
    float* ws = nullptr;
    cudaError_t e = ws_alloc(reinterpret_cast<void**>(&ws), (size_t)(batch * per_char), st);
    if (e != cudaSuccess) return cuda_fail(e, "Stage-1 workspace");
    hs::ChunkedArgs s1{};   // the Stage-1 kernel reads only seg[0].J and the Stage-1 fields
    s1.nseg = 1;
    s1.seg[0].J = J;
    s1.seg[0].n_chars = n_chars;
    s1.layers = layers;
    s1.keys = cs->d_keys;
    s1.n_layers = n_layers;
    s1.n_keys = cs->n_keys;
    s1.wrap = cs->wrap;
    s1.fps = cs->fps;
    s1.duration = cs->duration;
    hs_status r = HS_OK;
    for (int64_t c0 = 0; c0 < n_chars && r == HS_OK; c0 += batch) {
        const int64_t nb = std::min(batch, n_chars - c0);
        if ((e = hs::launch_stage1(s1, c0, nb, ws, st)) != cudaSuccess) { r = cuda_fail(e, "Stage-1 launch"); break; }
        if (mesh)   // scan + bind + skinning of the batch (fused or two-pass LBS, AUTO)
            r = hs_scan_skin_ex(sk, mesh, ws, nb, global_out + c0 * J * 12,
                                skin_out ? skin_out + c0 * J * 12 : nullptr,
                                verts_out + c0 * (int64_t)mesh->n_verts * 3, cuda_stream, nullptr);
        else
            r = scan_impl(sk, ws, nb, global_out + c0 * J * 12, skin_out ? skin_out + c0 * J * 12 : nullptr,
                          st, HS_ALGO_AUTO, -1, 0);   // single-CTA or multi-CTA path
    }
    cudaFreeAsync(ws, st);
    return r;
}

hs_status hs_animate_ex(const hs_skeleton* sk, const hs_clipset* cs, const void* layers, int32_t n_layers,
                        int64_t n_chars, float* global_out, float* skin_out, void* cuda_stream,
                        const hs_animate_opts* opts) {
    return animate_impl(sk, cs, layers, n_layers, n_chars, global_out, skin_out, cuda_stream, opts, nullptr,
                        nullptr);
}

hs_status hs_animate_skin(const hs_skeleton* sk, const hs_clipset* cs, const void* layers, int32_t n_layers,
                          int64_t n_chars, const hs_mesh* mesh, float* global_out, float* skin_out,
                          float* verts_out, void* cuda_stream) {
    if (!mesh || !verts_out) return fail(HS_ERR_INVALID_ARG, "null mesh or vertex buffer");
    if (mesh->n_joints != (sk ? sk->plan.n : -1)) return fail(HS_ERR_INVALID_ARG, "mesh built for another skeleton");
    return animate_impl(sk, cs, layers, n_layers, n_chars, global_out, skin_out, cuda_stream, nullptr, mesh,
                        verts_out);
}

hs_status hs_animate(const hs_skeleton* sk, const hs_clipset* cs, const void* layers, int32_t n_layers,
                     int64_t n_chars, float* global_out, float* skin_out, void* cuda_stream) {
    return hs_animate_ex(sk, cs, layers, n_layers, n_chars, global_out, skin_out, cuda_stream, nullptr);
}

hs_status hs_scan(const hs_skeleton* sk, const float* local, int64_t n_chars, float* global_out,
                  float* skin_out, void* cuda_stream) {
    return hs_scan_ex(sk, local, n_chars, global_out, skin_out, cuda_stream, nullptr);
}

hs_status hs_destroy(hs_skeleton* sk) {
    free_skeleton(sk);
    return HS_OK;
}

hs_status hs_skeleton_query(const hs_skeleton* sk, int32_t what, int64_t* v) {
    if (!sk || !v) return fail(HS_ERR_INVALID_ARG, "null argument");
    switch (what) {
        case HS_Q_N_JOINTS: *v = sk->plan.n; break;
        case HS_Q_MAX_LEVEL: *v = sk->plan.L; break;
        case HS_Q_ROUNDS: *v = sk->plan.R; break;
        case HS_Q_PATH: *v = sk->chunked ? HS_ALGO_CHUNKED : (sk->seq_ok ? HS_ALGO_TILES : HS_ALGO_SPLIT); break;
        case HS_Q_CHUNK: *v = sk->K; break;
        case HS_Q_TILE_CHARS: *v = sk->chunked ? sk->tp.C : 0; break;
        case HS_Q_SMALL_TILE_CHARS: *v = sk->small ? sk->small->tp.C : 0; break;
        case HS_Q_ANCHORS: *v = sk->chunked ? sk->tp.nslots : sk->sp.nslots; break;
        case HS_Q_ANCHOR_ROUNDS: *v = sk->chunked ? sk->tp.R2 : (sk->sub ? sk->sub->plan.R : 0); break;
        case HS_Q_IDENTITY_ORDER: *v = sk->plan.identity ? 1 : 0; break;
        case HS_Q_SMEM_BYTES: *v = sk->smem; break;
        case HS_Q_THREADS: *v = sk->threads; break;
        case HS_Q_STAGES: *v = sk->stages; break;
        case HS_Q_DEVICE: *v = sk->device; break;
        case HS_Q_SPLIT_LEVELS: *v = sk->split_levels; break;
        case HS_Q_SBUFS: *v = sk->sbufs; break;
        case HS_Q_CHUNKING: *v = sk->chunking == hs::CHUNK_CONSECUTIVE ? 1 : (sk->chunking == hs::CHUNK_RUNS ? 3 : 2); break;
        case HS_Q_PBUFS: *v = sk->chunked ? (sk->tp.pingpong ? 2 : 1) : 0; break;
        case HS_Q_SEQ_TILES: *v = sk->seq_ok ? sk->seq.KT : 0; break;
        case HS_Q_SEQ_TILE_JOINTS: *v = sk->seq_ok ? sk->seq.F : 0; break;
        case HS_Q_SEQ_EXPORTS: *v = sk->seq_ok ? sk->seq.n_exp : 0; break;
        case HS_Q_SEQ_SMEM_BYTES: *v = sk->seq_ok ? sk->seq_smem : 0; break;
        case HS_Q_SEQ_CHUNK: *v = sk->seq_ok ? sk->seq_K : 0; break;
        case HS_Q_SEQ_SBUFS: *v = sk->seq_ok ? sk->seq_sbufs : 0; break;
        default: return fail(HS_ERR_INVALID_ARG, "unknown query");
    }
    return HS_OK;
}

const char* hs_status_string(hs_status s) {
    switch (s) {
        case HS_OK: return "HS_OK";
        case HS_ERR_INVALID_ARG: return "HS_ERR_INVALID_ARG";
        case HS_ERR_EMPTY: return "HS_ERR_EMPTY";
        case HS_ERR_OUT_OF_RANGE: return "HS_ERR_OUT_OF_RANGE";
        case HS_ERR_CYCLE: return "HS_ERR_CYCLE";
        case HS_ERR_CUDA: return "HS_ERR_CUDA";
        case HS_ERR_OOM: return "HS_ERR_OOM";
        case HS_ERR_WRONG_DEVICE: return "HS_ERR_WRONG_DEVICE";
        case HS_ERR_UNSUPPORTED: return "HS_ERR_UNSUPPORTED";
        default: return "HS_ERR_UNKNOWN";
    }
}

const char* hs_last_error(void) { return g_err.c_str(); }

// ------------------------------------------------------------------ host-only plan
hs_status hs_plan_create_ex(const int32_t* parents, int32_t n_joints, const hs_create_opts* opts,
                            int32_t block_size, hs_plan** out) {
    if (!out) return fail(HS_ERR_INVALID_ARG, "out is null");
    hs_create_opts o;
    std::memset(&o, 0, sizeof(o));
    if (opts) o = *opts;
    try {
        hs_plan* p = new hs_plan();
        std::string err;
        int st = hs::build_plan(parents, n_joints, p->plan, err);
        if (st != 0) { delete p; return fail((hs_status)st, err); }
        p->K = o.chunk == 0 ? 5 : o.chunk;
        if (!is_valid_k(p->K)) { delete p; return fail(HS_ERR_INVALID_ARG, "chunk must be odd in 3..11"); }
        if (o.chunking < 0 || o.chunking > 3) { delete p; return fail(HS_ERR_INVALID_ARG, "bad chunking"); }
        const int mode = o.chunking == 1 ? hs::CHUNK_CONSECUTIVE
                                         : (o.chunking == 2 ? hs::CHUNK_HEAVY : hs::CHUNK_RUNS);
        p->block_size = block_size <= 0 ? 64 : block_size;
        std::vector<int32_t> pos(p->plan.order);
        p->decomp = hs::decompose(p->plan.ipar, p->K, mode, &pos, true);
        p->tile = hs::build_tile_program(p->plan, p->K, 1, true, mode);
        for (int F = o.tile_joints > 0 ? std::min(o.tile_joints, 1024) : 1024; F >= 64 && !p->seq_ok; F -= 64)
            p->seq_ok = hs::build_seq_program(p->plan, p->K, F - F % 32, mode, 224, p->seq);
        *out = p;
        return HS_OK;
    } catch (const std::bad_alloc&) {
        return fail(HS_ERR_OOM, "host allocation failed");
    }
}

hs_status hs_plan_create(const int32_t* parents, int32_t n_joints, int32_t chunk, int32_t block_size,
                         hs_plan** out) {
    hs_create_opts o;
    std::memset(&o, 0, sizeof(o));
    o.chunk = chunk;
    return hs_plan_create_ex(parents, n_joints, &o, block_size, out);
}

hs_status hs_plan_query(const hs_plan* p, int32_t what, int64_t* v) {
    if (!p || !v) return fail(HS_ERR_INVALID_ARG, "null argument");
    switch (what) {
        case HS_Q_N_JOINTS: *v = p->plan.n; break;
        case HS_Q_MAX_LEVEL: *v = p->plan.L; break;
        case HS_Q_ROUNDS: *v = p->plan.R; break;
        case HS_Q_CHUNK: *v = p->K; break;
        case HS_Q_ANCHORS: *v = (int64_t)p->decomp.slots.size(); break;
        case HS_Q_THREADS: *v = (int64_t)p->decomp.lists.size(); break;
        case HS_Q_TILE_SLOTS: *v = p->tile.nslots; break;
        case HS_Q_TILE_ROUNDS_ENTRIES: *v = (int64_t)p->tile.rounds.size(); break;
        case HS_Q_TILE_R2: *v = p->tile.R2; break;
        case HS_Q_IDENTITY_ORDER: *v = p->plan.identity ? 1 : 0; break;
        case HS_Q_SEQ_TILES: *v = p->seq_ok ? p->seq.KT : 0; break;
        case HS_Q_SEQ_TILE_JOINTS: *v = p->seq.F; break;
        case HS_Q_SEQ_EXPORTS: *v = p->seq.n_exp; break;
        case HS_Q_SEQ_THREADS: *v = p->seq.T; break;
        case HS_Q_SEQ_SLOTS: *v = p->seq.S; break;
        case HS_Q_SEQ_R2MAX: *v = p->seq.R2max; break;
        case HS_Q_SEQ_ENTRIES: *v = (int64_t)p->seq.rounds.size(); break;
        case HS_Q_SEQ_IMPORTS: *v = (int64_t)p->seq.exl.size() / 2; break;
        case HS_Q_SEQ_RUNS: *v = (int64_t)p->seq.runs.size() / 4; break;
        case HS_Q_SEQ_QSLOTS: *v = p->seq.nQ; break;
        case HS_Q_ANCHOR_ROUNDS: {
            hs::TileProgram tp = hs::build_tile_program(p->plan, p->K, 1, true, hs::CHUNK_HEAVY);
            *v = tp.R2;
            break;
        }
        default: return fail(HS_ERR_INVALID_ARG, "unknown plan query");
    }
    return HS_OK;
}

hs_status hs_plan_export(const hs_plan* p, int32_t what, void* buf, int64_t buf_bytes) {
    if (!p || !buf) return fail(HS_ERR_INVALID_ARG, "null argument");
    std::vector<int32_t> tmp;
    const hs::Plan& P = p->plan;
    const hs::TileProgram& tp = p->tile;
    auto raw = [&](const void* src, size_t bytes) -> hs_status {
        if ((int64_t)bytes > buf_bytes) return fail(HS_ERR_INVALID_ARG, "buffer too small");
        if (bytes) std::memcpy(buf, src, bytes);
        return HS_OK;
    };
    switch (what) {
        case HS_X_TILE_META: return raw(tp.meta.data(), tp.meta.size() * sizeof(uint64_t));
        case HS_X_TILE_P1LEN: return raw(tp.p1len.data(), tp.p1len.size() * sizeof(int32_t));
        case HS_X_TILE_ROUND_OFF: return raw(tp.round_off.data(), tp.round_off.size() * sizeof(int32_t));
        case HS_X_TILE_ROUNDS: return raw(tp.rounds.data(), tp.rounds.size() * sizeof(uint32_t));
        case HS_X_SEQ_TILES: return raw(p->seq.tiles.data(), p->seq.tiles.size() * sizeof(hs::SeqTile));
        case HS_X_SEQ_META: return raw(p->seq.meta.data(), p->seq.meta.size() * sizeof(uint64_t));
        case HS_X_SEQ_P1LEN: return raw(p->seq.p1len.data(), p->seq.p1len.size() * sizeof(int32_t));
        case HS_X_SEQ_ROUND_OFF: return raw(p->seq.round_off.data(), p->seq.round_off.size() * sizeof(int32_t));
        case HS_X_SEQ_ROUNDS: return raw(p->seq.rounds.data(), p->seq.rounds.size() * sizeof(uint32_t));
        case HS_X_SEQ_IMP: return raw(p->seq.exl.data(), p->seq.exl.size() * sizeof(int32_t));
        case HS_X_SEQ_RUNS: return raw(p->seq.runs.data(), p->seq.runs.size() * sizeof(int32_t));
        case HS_X_SEQ_IB_USER: return raw(p->seq.ib_user.data(), p->seq.ib_user.size() * sizeof(int32_t));
        case HS_X_LEVELS: tmp = P.level; break;
        case HS_X_ORDER: tmp = P.order; break;
        case HS_X_LIFT: tmp = P.lift; break;
        case HS_X_BLOCK_OF:
        case HS_X_MPOB: {
            std::vector<int32_t> b, m;
            hs::block_layout(P, p->block_size, b, m);
            tmp = what == HS_X_BLOCK_OF ? b : m;
            break;
        }
        case HS_X_CHUNK_SRC: tmp = p->decomp.src; break;
        case HS_X_ANCHOR_LINK: tmp = p->decomp.link0; break;
        case HS_X_CHUNK_LISTS:
            tmp.assign(p->decomp.lists.size() * (size_t)p->K, -1);
            for (size_t t = 0; t < p->decomp.lists.size(); ++t)
                for (size_t s = 0; s < p->decomp.lists[t].size(); ++s) tmp[t * p->K + s] = p->decomp.lists[t][s];
            break;
        default: return fail(HS_ERR_INVALID_ARG, "unknown export");
    }
    if ((int64_t)(tmp.size() * sizeof(int32_t)) > buf_bytes) return fail(HS_ERR_INVALID_ARG, "buffer too small");
    if (!tmp.empty()) std::memcpy(buf, tmp.data(), tmp.size() * sizeof(int32_t));
    return HS_OK;
}

hs_status hs_plan_destroy(hs_plan* p) {
    delete p;
    return HS_OK;
}

// ------------------------------------------------------------------ host pipeline
hs_status hs_pipeline_create(int64_t batch_bytes, hs_pipeline** out) {
    if (!out) return fail(HS_ERR_INVALID_ARG, "out is null");
    if (batch_bytes <= 0) batch_bytes = (int64_t)256 << 20;
    batch_bytes = (batch_bytes + 15) & ~(int64_t)15;
    hs_pipeline* pl = new (std::nothrow) hs_pipeline();
    if (!pl) return fail(HS_ERR_OOM, "host allocation failed");
    pl->batch_bytes = batch_bytes;
    cudaError_t e = cudaGetDevice(&pl->device);
    for (int i = 0; i < 3 && e == cudaSuccess; ++i) {
        e = cudaStreamCreateWithFlags(&pl->st[i], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&pl->d_in[i]), (size_t)batch_bytes);
        if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&pl->d_g[i]), (size_t)batch_bytes);
        if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&pl->d_s[i]), (size_t)batch_bytes);
    }
    if (e != cudaSuccess) {
        hs_pipeline_destroy(pl);
        return cuda_fail(e, "pipeline create");
    }
    *out = pl;
    return HS_OK;
}

// An error in the middle of a host pipeline returns only after the copies already
// queued on its streams have finished: they read and write the caller's host buffers.
static hs_status drain_fail(hs_pipeline* pl, hs_status s) {
    for (int i = 0; i < 3; ++i) cudaStreamSynchronize(pl->st[i]);
    return s;
}

hs_status hs_scan_host_batch(hs_pipeline* pl, const hs_batch_item* items, int32_t n_items) {
    if (!pl) return fail(HS_ERR_INVALID_ARG, "null handle");
    if (n_items < 0 || (n_items > 0 && !items)) return fail(HS_ERR_INVALID_ARG, "bad item list");
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != pl->device) return fail(HS_ERR_WRONG_DEVICE, "device mismatch");
    for (int32_t k = 0; k < n_items; ++k) {
        const hs_batch_item& it = items[k];
        if (!it.skeleton) return fail(HS_ERR_INVALID_ARG, "null skeleton");
        if (it.n_chars < 0) return fail(HS_ERR_INVALID_ARG, "n_chars < 0");
        if (it.n_chars && (!it.local || !it.global_out || !it.skin_out)) return fail(HS_ERR_INVALID_ARG, "null buffer");
        if (it.skeleton->device != dev) return fail(HS_ERR_WRONG_DEVICE, "device mismatch");
        if (pl->batch_bytes / ((int64_t)it.skeleton->plan.n * 48) < 1)
            return fail(HS_ERR_INVALID_ARG, "pipeline batch smaller than one character");
    }
    // one pipeline over every item's characters: the 3 streams rotate across items
    // without draining in between; batches ramp up geometrically from ~8 MB at the
    // start, so the read-back copy engine (the larger direction) idles only for the
    // first small upload
    int64_t b = 0, ramp = (int64_t)8 << 20;
    for (int32_t k = 0; k < n_items; ++k) {
        const hs_batch_item& it = items[k];
        const hs_skeleton* sk = it.skeleton;
        const int64_t per_char = (int64_t)sk->plan.n * 48;
        const int64_t batch = pl->batch_bytes / per_char;
        for (int64_t c0 = 0, nb = 0; c0 < it.n_chars; c0 += nb, ++b) {
            const int i = (int)(b % 3);
            const int64_t cur = std::max<int64_t>(1, std::min<int64_t>(batch, ramp / per_char));
            ramp = std::min<int64_t>(2 * ramp, pl->batch_bytes);
            nb = std::min(cur, it.n_chars - c0);
            const size_t bytes = (size_t)(nb * per_char);
            const int64_t foff = c0 * sk->plan.n * 12;
            cudaError_t e = cudaMemcpyAsync(pl->d_in[i], it.local + foff, bytes, cudaMemcpyHostToDevice, pl->st[i]);
            if (e != cudaSuccess) return drain_fail(pl, cuda_fail(e, "H2D"));
            hs_status s = scan_impl(sk, pl->d_in[i], nb, pl->d_g[i], pl->d_s[i], pl->st[i], HS_ALGO_AUTO, -1, 0);
            if (s != HS_OK) return drain_fail(pl, s);
            if ((e = cudaMemcpyAsync(it.global_out + foff, pl->d_g[i], bytes, cudaMemcpyDeviceToHost, pl->st[i])) !=
                    cudaSuccess ||
                (e = cudaMemcpyAsync(it.skin_out + foff, pl->d_s[i], bytes, cudaMemcpyDeviceToHost, pl->st[i])) !=
                    cudaSuccess)
                return drain_fail(pl, cuda_fail(e, "D2H"));
        }
    }
    for (int i = 0; i < 3; ++i) {
        cudaError_t e = cudaStreamSynchronize(pl->st[i]);
        if (e != cudaSuccess) return cuda_fail(e, "pipeline sync");
    }
    return HS_OK;
}

hs_status hs_scan_host(hs_pipeline* pl, const hs_skeleton* sk, const float* h_local, int64_t n_chars,
                       float* h_global, float* h_skin) {
    if (!pl || !sk) return fail(HS_ERR_INVALID_ARG, "null handle");
    if (n_chars < 0) return fail(HS_ERR_INVALID_ARG, "n_chars < 0");
    if (n_chars == 0) return HS_OK;
    if (!h_local || !h_global || !h_skin) return fail(HS_ERR_INVALID_ARG, "null buffer");
    const hs_batch_item it{sk, h_local, n_chars, h_global, h_skin};
    return hs_scan_host_batch(pl, &it, 1);
}

hs_status hs_animate_host(hs_pipeline* pl, const hs_skeleton* sk, const hs_clipset* cs, const void* h_layers,
                          int32_t n_layers, int64_t n_chars, float* h_global, float* h_skin) {
    if (!pl || !sk || !cs) return fail(HS_ERR_INVALID_ARG, "null handle");
    if (n_chars < 0) return fail(HS_ERR_INVALID_ARG, "n_chars < 0");
    if (n_chars == 0) return HS_OK;
    if (!h_layers || !h_global || !h_skin) return fail(HS_ERR_INVALID_ARG, "null buffer");
    if (n_layers < 1 || n_layers > 8) return fail(HS_ERR_INVALID_ARG, "n_layers must be in 1..8");
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != sk->device || dev != pl->device) return fail(HS_ERR_WRONG_DEVICE, "device mismatch");
    const int32_t J = sk->plan.n;
    const int64_t per_char = (int64_t)J * 48, lay_bytes = (int64_t)n_layers * 16;
    const int64_t batch = pl->batch_bytes / std::max(per_char, lay_bytes);
    if (batch < 1) return fail(HS_ERR_INVALID_ARG, "pipeline batch smaller than one character");
    hs_animate_opts o{};
    o.mode = HS_ANIMATE_TWO_PASS;
    o.workspace_bytes = batch * per_char;
    // layers up (16 B per layer), Stage 1 + scan + bind on the device, poses back; the
    // 3 streams rotate and the batches ramp up from ~8 MB as in hs_scan_host
    int64_t b = 0, ramp = (int64_t)8 << 20;
    for (int64_t c0 = 0, nb = 0; c0 < n_chars; c0 += nb, ++b) {
        const int i = (int)(b % 3);
        const int64_t cur = std::max<int64_t>(1, std::min<int64_t>(batch, ramp / per_char));
        ramp = std::min<int64_t>(2 * ramp, pl->batch_bytes);
        nb = std::min(cur, n_chars - c0);
        cudaError_t e = cudaMemcpyAsync(pl->d_in[i], static_cast<const char*>(h_layers) + c0 * lay_bytes,
                                        (size_t)(nb * lay_bytes), cudaMemcpyHostToDevice, pl->st[i]);
        if (e != cudaSuccess) return drain_fail(pl, cuda_fail(e, "H2D"));
        hs_status s = hs_animate_ex(sk, cs, pl->d_in[i], n_layers, nb, pl->d_g[i], pl->d_s[i], pl->st[i], &o);
        if (s != HS_OK) return drain_fail(pl, s);
        const size_t bytes = (size_t)(nb * per_char);
        const int64_t foff = c0 * J * 12;
        if ((e = cudaMemcpyAsync(h_global + foff, pl->d_g[i], bytes, cudaMemcpyDeviceToHost, pl->st[i])) !=
                cudaSuccess ||
            (e = cudaMemcpyAsync(h_skin + foff, pl->d_s[i], bytes, cudaMemcpyDeviceToHost, pl->st[i])) !=
                cudaSuccess)
            return drain_fail(pl, cuda_fail(e, "D2H"));
    }
    for (int i = 0; i < 3; ++i) {
        cudaError_t e = cudaStreamSynchronize(pl->st[i]);
        if (e != cudaSuccess) return cuda_fail(e, "pipeline sync");
    }
    return HS_OK;
}

hs_status hs_workspace_trim(int64_t* held_bytes) {
    if (held_bytes) *held_bytes = 0;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev < 0 || dev >= 64) return HS_OK;
    std::lock_guard<std::mutex> lock(g_pools_mu);
    cudaMemPool_t pool = g_pools[dev];
    if (!pool) return HS_OK;
    if ((e = cudaMemPoolTrimTo(pool, 0)) != cudaSuccess) return cuda_fail(e, "cudaMemPoolTrimTo");
    if (held_bytes) {
        uint64_t v = 0;
        if ((e = cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &v)) != cudaSuccess)
            return cuda_fail(e, "cudaMemPoolGetAttribute");
        *held_bytes = (int64_t)v;
    }
    return HS_OK;
}

hs_status hs_pipeline_destroy(hs_pipeline* pl) {
    if (!pl) return HS_OK;
    for (int i = 0; i < 3; ++i) {
        if (pl->st[i]) cudaStreamSynchronize(pl->st[i]);
        cudaFree(pl->d_in[i]);
        cudaFree(pl->d_g[i]);
        cudaFree(pl->d_s[i]);
        if (pl->st[i]) cudaStreamDestroy(pl->st[i]);
    }
    delete pl;
    return HS_OK;
}

}  // extern "C"
