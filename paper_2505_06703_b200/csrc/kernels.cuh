// kernels.cuh — launch interface of the sm_100a kernels (kernels.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

// Debug/tuning builds only (tools/prof_*.py build a libhs_prof.so variant): the
// HS_DEBUG_PROF phase profile.  The product build compiles it out, so the shipped
// library reads no environment variable on any call.
#ifndef HS_PROF_HOOKS
#define HS_PROF_HOOKS 0   // its per-phase checks cost ~3 % on tree1024
#endif
#ifndef HS_BULK_PIECE
#define HS_BULK_PIECE 4096   // bytes per TMA bulk copy (4 KB 10.63, 8 KB 10.67, whole tile 10.83 ms on C5)
#endif

namespace hs {

// Persistent TMA tile kernel (HS_ALGO_CHUNKED), DESIGN.md §5.1.  One launch runs
// up to kMaxSegs segments (a skeleton's crowd each, NEXT-3): their tiles form one
// global tile space, CTA b taking tiles b, b + grid, ...; a CTA switches programs
// when its tile crosses into the next segment.
constexpr int kMaxSegs = 8;

struct SegArgs {
    const float* local;        // [n_chars][J][12]
    float* gout;               // [n_chars][J][12]
    float* sout;               // [n_chars][J][12] or nullptr (no bind epilogue)
    const float* ib;           // [J][12] user order (used when sout != nullptr)
    const uint64_t* meta;      // [T][K]
    const int32_t* p1len;      // [T]: phase-1 length | run_back << 8 | (run anchor + 1) << 16
    const int32_t* round_off;  // [R2+1]
    const uint32_t* rounds;    // phase-2 descriptors (copied to smem by each CTA)
    int64_t n_chars;
    int64_t tile_base;         // first global tile of this segment
    int32_t J, C, F, T;        // joints, chars per tile, joints per tile, compute threads
    int32_t nslots, R2;
    int32_t n_rounds_entries;
    int32_t p_single;          // 1 = single P buffer, all reads of a round before its writes
};

struct ChunkedArgs {
    SegArgs seg[kMaxSegs];
    int32_t nseg;
    int64_t total_tiles;
    int32_t tile_f;            // floats per stage / S buffer: 12 x max F
    int32_t p_floats;          // floats of the P region (max over segments)
    int32_t r2_max;            // max R2 (table layout)
    int32_t stages, sbufs;
    int64_t smem_bytes;
    int32_t threads;           // consumer warps * 32 + 32 (producer warp)
    int32_t ctas_per_sm;       // 0 = occupancy maximum
    int32_t has_runs;          // some segment's lanes are joined by the warp-shuffle scan
    int32_t bulk_piece;        // bytes per TMA bulk copy (0 = one copy per tile and buffer)
    // Stage-1 prologue (hs_animate, one segment): layers != nullptr replaces the
    // local-pose input
    const void* layers;        // device [n_chars][n_layers] hs_layer (16 B)
    const float* keys;         // device [n_clips][n_keys] rows of 10 * Jp floats (planar keys)
    int32_t n_layers, n_keys, wrap;
    int32_t desc_off;          // smem byte offset of the layer-descriptor ring ([stages][C * n_layers] int4)
    float fps, duration;
    // LBS epilogue (hs_scan_skin, one segment): verts != nullptr adds vertex skinning
    const float4* mesh_a;      // [V] (px, py, pz, w0)
    const float4* mesh_b;      // [V] (w1, w2, w3, 0)
    const int2* mesh_j;        // [V] (j0 | j1 << 16, j2 | j3 << 16)
    float* verts;              // [n_chars][V][3]
    int32_t n_verts;
    unsigned long long* prof;  // debug: per-phase clock64 sums of consumer thread 0 (or nullptr)
};
// Multi-tile kernel (HS_ALGO_TILES): skeletons beyond one CTA.  A
// persistent CTA takes whole characters (b, b + grid, ...) and walks each one's KT
// tiles in topological order; cross-tile parents are final workspace values.
// Multi-tile kernel: barrier header bytes, and the helper warp's inbox loads in flight
// per lane (16-byte pieces)
constexpr int kSeqHeaderBytes = 256;
constexpr int kSeqExportUnroll = 4;   // export pieces in flight per thread
// inbox staging by the consumers: at most this many 16-byte pieces per thread
// (3 x inbox rows <= kSeqInboxPieces x threads; the plan checks)
constexpr int kSeqInboxPieces = 9;   // rows from tiles <= k - 2 (loaded at the top of tile k - 1)
constexpr int kSeqInboxLate = 4;     // rows from tile k - 1 (loaded after its phase-2 barrier)
struct SeqTileDev {               // = hs::SeqTile (plan.hpp)
    int32_t n_early, nj, R2, n_entries, rounds_off, n_imp, imp_off, n_runs, runs_off, T, n_exl, exl_off;
};
struct SeqArgs {
    const float* local;        // [n_chars][J][12]
    float* gout;               // [n_chars][J][12]
    float* sout;               // [n_chars][J][12] or nullptr
    float* ws;                 // [grid][n_exp][12]: the inboxes of the CTA's current character
    const float* ib;           // [KT][F][12] inverse bind by tile smem offset
    const SeqTileDev* tiles;   // [KT]
    const uint64_t* meta;      // [KT][T][K]
    const int32_t* p1len;      // [KT][T]
    const int32_t* round_off;  // [KT][R2max + 1]
    const uint32_t* rounds;    // concatenated descriptors
    const int2* exl;           // export lists: (smem offset in the tile, workspace row)
    const int4* runs;          // (user start, smem offset, length, 0)
    int64_t n_chars;
    int32_t J, KT, F, T, S, nQ, n_exp, r2max, max_imp, max_entries;
    int32_t r2p, entp;         // program record widths: round_off row, phase-2 entries (padded to 4)
    int32_t max_exl;           // export-list buffer (pairs, even)
    int32_t p_floats;          // (2S + 2 nQ) * 12: anchors (ping-pong) and two Q buffers
    int32_t stages, sbufs, threads, has_runs, bulk_piece;
    int64_t smem_bytes;
    int32_t ctas_per_sm;       // 0 = occupancy maximum (1)
    unsigned long long* prof;  // profiling builds: per-phase clock64 sums of consumer thread 0 (or nullptr)
};
cudaError_t launch_seq(int K, const SeqArgs& a, cudaStream_t st);
cudaError_t prepare_seq(int K);

int sm_count();   // SMs of the current device (cached)
cudaError_t launch_chunked(int K, const ChunkedArgs& a, cudaStream_t st);
// Linear blend skinning from skin poses in HBM (two-pass hs_scan_skin): S [n_chars][J][12].
cudaError_t launch_lbs(const float* S, int64_t n_chars, int32_t J, const float4* mesh_a, const float4* mesh_b,
                       const int2* mesh_j, int32_t V, float* verts, cudaStream_t st);
// Stage 1 alone (two-pass hs_animate): local poses of characters [c0, c0 + n_chars)
// of a.layers into local ([n_chars][J][12]).
cudaError_t launch_stage1(const ChunkedArgs& a, int64_t c0, int64_t n_chars, float* local, cudaStream_t st);
cudaError_t prepare_chunked(int K, int64_t smem_bytes);   // sets the dynamic smem attribute
int max_chunked_blocks_per_sm(int K, bool runs, int threads, int64_t smem_bytes);

// Alg. 2: radix-2 pointer jumping, one thread per joint.
cudaError_t launch_doubling(const float* local, float* gout, float* sout, const float* ib,
                            const int32_t* lift, int32_t J, int32_t R, int32_t rounds,
                            int64_t n_chars, cudaStream_t st);

// Alg. 3 literally: 64-joint blocks, clamped in-block doubling, then
// the MaxParentOutBlock walk (comparison kernel).
cudaError_t launch_blocked(const float* local, float* gout, float* sout, const float* ib, const int32_t* lb,
                           const int32_t* mpob, int32_t J, int32_t RB, int64_t n_chars, cudaStream_t st);

// Alg. 4 literally: 64-joint blocks, 7 serial in-block composes,
// 7 stride-8 composes on that snapshot, then the MaxParentOutBlock walk (comparison).
cudaError_t launch_compressed(const float* local, float* gout, float* sout, const float* ib, const int32_t* lp,
                              const int32_t* l8, const int32_t* mpob, int32_t J, int64_t n_chars, cudaStream_t st);

// Per-character topology (NEXT-3): parents [n_chars][J] (character-local labels),
// inverse binds [n_chars][J][12] or nullptr (skin = global); J <= 1024.
cudaError_t launch_varied(const int32_t* parents, const float* local, const float* ib, int32_t J,
                          int64_t n_chars, float* gout, float* sout, cudaStream_t st);

// Alg. 1: thread per joint walks all ancestors.
cudaError_t launch_gateau(const float* local, float* gout, float* sout, const float* ib,
                          const int32_t* parents, int32_t J, int64_t n_chars, cudaStream_t st);

// KIYA leaf walk: thread per leaf fills its root path top-down.
cudaError_t launch_leaf(const float* local, float* gout, float* sout, const float* ib,
                        const int32_t* path_off, const int32_t* path, int32_t n_leaves, int32_t J,
                        int64_t n_chars, cudaStream_t st);

// Multi-CTA (split) path: phase 1 and phase 3 over chunks.
cudaError_t launch_split_p1(int K, const float* local, float* pg, const int32_t* meta,
                            int32_t nchunks, int32_t J, int32_t nslots, int64_t n_chars,
                            cudaStream_t st);
cudaError_t launch_split_p3(int K, const float* local, float* gout, float* sout, const float* ib,
                            const float* pf, const int32_t* meta, int32_t nchunks, int32_t J,
                            int32_t nslots, int64_t n_chars, cudaStream_t st);

}  // namespace hs
