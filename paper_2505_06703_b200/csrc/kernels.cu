// kernels.cu — hand-written sm_100a kernels for the Hierarchy-Scan + fused
// Bind MeshPose (§1 steps 2-3, Eq. 1, Algs. 1-4).  DESIGN.md §5.
//
// Every pose is a 3x4 fp32 affine [R|t] (48 B).  compose(a, b) = a (x) b with
// the parent on the LEFT (Alg. 1's "M[jointID] = M[curParentID] * M[jointID]",
// PAPER.md:81).  No tensor cores: a chain of tiny 3x4 products is not a dense
// contraction (BASELINE.json north_star); the path is HBM-bound.
//
// This file: the chunked kernel (the hot path) and its launcher;
// the other kernels live in kernels_aux.cu, shared device helpers in device_util.cuh.
#include <atomic>
#include <mutex>

#include "device_util.cuh"

#ifndef HS_LBS_U
#define HS_LBS_U 2
#endif
#ifndef HS_STREAM_HINTS
#define HS_STREAM_HINTS 0   // L2 evict_first on the streaming TMA copies (A/B: tools/time_scan.py)
#endif

namespace hs {
namespace {
constexpr int kLbsU = HS_LBS_U;   // vertices per thread in flight in the fused LBS epilogue

// ================================================================== chunked kernel
// Persistent, warp-specialised.  Warps 0..nwc-1 compute; warp nwc is the TMA
// producer.  Per tile of C characters (F = C*J joints, user order in smem):
//   phase 1  each compute thread folds its chunk of K consecutive internal
//            positions left-to-right (in-chunk parent = previous position) and
//            publishes the running product at anchor joints into P;
//   phase 2  pointer jumping (Alg. 2) over the anchor forest, ping-pong P;
//   phase 3  each thread re-folds its chunk starting from the final P of each
//            segment head's parent, writes G in place over L, and S = G (x) IB
//            (IB held in registers) into the S buffer;
// then the producer bulk-stores G and S and refills the stage.
// Kernel modes: one segment (hs_scan), one segment with the Stage-1 prologue
// (hs_animate), several segments in one launch (hs_scan_batch, NEXT-3), or one
// segment with the linear-blend-skinning epilogue (hs_scan_skin, NEXT-4).
enum : int { kModeScan = 0, kModeStage1 = 1, kModeMulti = 2, kModeSkin = 3 };

// Producer-side view of the segment a tile belongs to; advanced only when the tile
// index crosses into the next segment (tiles of a CTA only move forward).
struct SegCursor {
    int s;
    int64_t next_base, base, n_chars;
    int J, C;
    const float* local;
    float* gout;
    float* sout;
    __device__ __forceinline__ void load(const ChunkedArgs& a, int i) {
        const SegArgs& S = a.seg[i];
        s = i;
        base = S.tile_base; n_chars = S.n_chars; J = S.J; C = S.C;
        local = S.local; gout = S.gout; sout = S.sout;
        next_base = i + 1 < a.nseg ? a.seg[i + 1].tile_base : INT64_MAX;
    }
    __device__ __forceinline__ void seek(const ChunkedArgs& a, int64_t g) {
        if (g >= next_base) {
            int i = s + 1;
            while (i + 1 < a.nseg && g >= a.seg[i + 1].tile_base) ++i;
            load(a, i);
        }
    }
};

template <int K, bool RUNS, int MODE>
__global__ void __launch_bounds__(256, 1) chunked_kernel(const __grid_constant__ ChunkedArgs a) {
    constexpr bool PRO = MODE == kModeStage1;
    constexpr bool MULTI = MODE == kModeMulti;
    constexpr bool LBS = MODE == kModeSkin;
    extern __shared__ __align__(128) unsigned char smem[];
    const int NS = a.stages, NSS = a.sbufs;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* done = full + 4;
    uint64_t* sfree = done + 4;
    float* LG = reinterpret_cast<float*>(smem + 128);
    const int64_t tile_f = a.tile_f;
    float* SB = LG + NS * tile_f;
    float* P = SB + NSS * tile_f;
    int32_t* s_round_off = reinterpret_cast<int32_t*>(P + a.p_floats);
    uint32_t* s_rounds = reinterpret_cast<uint32_t*>(s_round_off + a.r2_max + 1);
    int4* desc = reinterpret_cast<int4*>(smem + a.desc_off);   // Stage 1: [NS][C * n_layers]

    const int nwc = (int)(blockDim.x >> 5) - 1;
    const int NC = nwc * 32;
    const int warp = threadIdx.x >> 5;
    const int64_t ntiles = a.total_tiles;
    const int64_t my_tiles =
        blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&done[s], 1); }
        for (int s = 0; s < NSS; ++s) mbar_init(&sfree[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == nwc) {
        // ------------------------------------------------------------ producer
        // (Stage 1: the whole warp writes the next tiles' layer descriptors)
        const int lane = threadIdx.x & 31;
        if (!PRO && lane != 0) return;
        const uint32_t piece = a.bulk_piece > 0 ? (uint32_t)a.bulk_piece : 0xffffffffu;
#if HS_STREAM_HINTS
        const uint64_t stream_pol = policy_evict_first();   // tiles in, G and S out: touched once
#endif
        // stage / S-buffer indices and mbarrier parities advance incrementally: no
        // 64-bit division in the loop; segment cursors for the loads (run NS tiles
        // ahead) and for the stores
        SegCursor ld, st;
        ld.load(a, 0);
        st.load(a, 0);
        auto issue_load = [&](int64_t it, int stage) {
            const int64_t g = blockIdx.x + it * gridDim.x;
            if (MULTI) ld.seek(a, g);
            const int64_t c0 = (g - ld.base) * ld.C;
            const int64_t nc = min((int64_t)ld.C, ld.n_chars - c0);
            const uint32_t bytes = (uint32_t)(nc * ld.J * 48);
            HS_BOUND(nc > 0 && c0 >= 0 && (int64_t)bytes <= tile_f * 4);
            mbar_expect_tx(&full[stage], bytes);
            const char* src = reinterpret_cast<const char*>(ld.local + c0 * ld.J * 12);
            char* dst = reinterpret_cast<char*>(LG + stage * tile_f);
            for (uint32_t o = 0; o < bytes; o += piece) {
#if HS_STREAM_HINTS
                bulk_g2s_hint(dst + o, src + o, min(piece, bytes - o), &full[stage], stream_pol);
#else
                bulk_g2s(dst + o, src + o, min(piece, bytes - o), &full[stage]);
#endif
            }
        };
        // Stage 1 (one segment): descriptors of tile `it`'s (character, layer) pairs
        // into desc[stage], then full[stage] tells the consumers the stage is theirs
        auto fill_desc = [&](int64_t it, int stage) {
            const int64_t c0 = (blockIdx.x + it * gridDim.x) * st.C;
            const int nl = a.n_layers;
            const int n = (int)min((int64_t)st.C, st.n_chars - c0) * nl;
            const int4* lay = reinterpret_cast<const int4*>(a.layers) + c0 * nl;
            int4* d = desc + stage * st.C * nl;
            for (int i = lane; i < n; i += 32) d[i] = layer_desc(a, __ldg(lay + i));
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[stage]);
        };
        if (!PRO)
            for (int64_t it = 0; it < my_tiles && it < NS; ++it) issue_load(it, (int)it);
        else
            for (int64_t it = 0; it < my_tiles && it < NS; ++it) fill_desc(it, (int)it);
        int stage = 0, sb = 0;
        uint32_t phase = 0;
        for (int64_t it = 0; it < my_tiles; ++it) {
            HS_DELAY(1);
            mbar_wait(&done[stage], phase);
            HS_DELAY(2);
            if (PRO && lane != 0) {   // lanes 1..31: only the descriptor fill
                __syncwarp();
                if (it + NS < my_tiles) fill_desc(it + NS, stage);
                if (++stage == NS) { stage = 0; phase ^= 1u; }
                continue;
            }
            const int64_t g = blockIdx.x + it * gridDim.x;
            if (MULTI) st.seek(a, g);
            const bool do_skin = st.sout != nullptr;
            const int64_t c0 = (g - st.base) * st.C;
            const int64_t nc = min((int64_t)st.C, st.n_chars - c0);
            const uint32_t bytes = (uint32_t)(nc * st.J * 48);
            HS_BOUND(nc > 0 && c0 >= 0 && (int64_t)bytes <= tile_f * 4);
            {
                char* gp = reinterpret_cast<char*>(st.gout + c0 * st.J * 12);
                const char* sg = reinterpret_cast<const char*>(LG + stage * tile_f);
                char* sp = do_skin ? reinterpret_cast<char*>(st.sout + c0 * st.J * 12) : nullptr;
                const char* ss = reinterpret_cast<const char*>(SB + sb * tile_f);
                for (uint32_t o = 0; o < bytes; o += piece) {
                    const uint32_t nb = min(piece, bytes - o);
#if HS_STREAM_HINTS
                    bulk_s2g_hint(gp + o, sg + o, nb, stream_pol);
                    if (do_skin) bulk_s2g_hint(sp + o, ss + o, nb, stream_pol);
#else
                    bulk_s2g(gp + o, sg + o, nb);
                    if (do_skin) bulk_s2g(sp + o, ss + o, nb);
#endif
                }
            }
            bulk_commit();
            HS_DELAY(3);
            bulk_wait_read<0>();                  // smem of this tile has been read out
            HS_DELAY(4);
            mbar_arrive(&sfree[sb]);              // (also when this segment has no skin output)
            if (PRO) {   // Stage 1 computes tiles in place: the stage is free once read out
                __syncwarp();
                if (it + NS < my_tiles) fill_desc(it + NS, stage);
            } else if (it + NS < my_tiles) {
                issue_load(it + NS, stage);
            }
            if (++stage == NS) { stage = 0; phase ^= 1u; }
            if (++sb == NSS) sb = 0;
        }
        if (lane == 0) bulk_wait_all();
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int t = threadIdx.x;
    uint64_t m[K];
    float ibr[K][12];
    int p1 = 0, run_back = 0, run_anchor = -1;
    // the current segment's program (MULTI: reloaded when a tile crosses into the next
    // segment; otherwise loaded once)
    int cseg = 0;
    int64_t next_base = INT64_MAX;
    int J = 0, C = 0, S2 = 0, R2 = 0, p_single = 0;
    int64_t nch = 0, tbase = 0;
    bool do_skin = false;
    auto load_program = [&](int s) {
        const SegArgs& S = a.seg[s];
        J = S.J; C = S.C; S2 = S.nslots; R2 = S.R2; p_single = S.p_single;
        nch = S.n_chars; tbase = S.tile_base; do_skin = LBS || S.sout != nullptr;
        next_base = s + 1 < a.nseg ? a.seg[s + 1].tile_base : INT64_MAX;
        p1 = 0; run_back = 0; run_anchor = -1;
        if (t < S.T) {
            const int info = S.p1len[t];
            p1 = info & 0xff;
            run_back = (info >> 8) & 0xff;
            run_anchor = (int)((uint32_t)info >> 16) - 1;
#pragma unroll
            for (int s2 = 0; s2 < K; ++s2) m[s2] = S.meta[(int64_t)t * K + s2];
        } else {
#pragma unroll
            for (int s2 = 0; s2 < K; ++s2) m[s2] = (uint64_t)(uint16_t)(int16_t)kSrcNone << 32;
        }
        if (do_skin) {
#pragma unroll
            for (int s2 = 0; s2 < K; ++s2) {
                const int src = (int)(int16_t)(m[s2] >> 32);
                const int ibu = (int)((m[s2] >> 16) & 0xffff);
                if (src != kSrcNone) {
                    HS_BOUND(ibu >= 0 && ibu < S.J);
                    ldg3(S.ib + (int64_t)ibu * 12, ibr[s2]);
                }
            }
        }
        // phase-2 tables: identical for every tile of the segment, staged per CTA (the
        // previous tile ended with a consumer barrier, so nobody still reads them)
        for (int i = t; i <= S.R2; i += NC) s_round_off[i] = __ldg(S.round_off + i);
        for (int i = t; i < S.n_rounds_entries; i += NC) s_rounds[i] = __ldg(S.rounds + i);
        bar_consumers(NC);
    };
    if (my_tiles > 0) {
        if (MULTI) {
            int s0 = 0;
            while (s0 + 1 < a.nseg && (int64_t)blockIdx.x >= a.seg[s0 + 1].tile_base) ++s0;
            cseg = s0;
        }
        load_program(cseg);
    }

    // debug phase profile (HS_DEBUG_PROF): consumer thread 0 accumulates clock64 deltas
    long long prof_last = 0;
    auto prof_mark = [&](int slot) {
        if (HS_PROF_HOOKS && a.prof && t == 0) {
            const long long now = clock64();
            if (slot >= 0) atomicAdd(a.prof + slot, (unsigned long long)(now - prof_last));
            prof_last = now;
        }
    };
    // per-segment values in the tile loop, read from the kernel parameters with the
    // (CTA-uniform) segment index, so loop bounds and branches stay uniform
#define SEGV(field, var) (a.seg[MULTI ? cseg : 0].field)
#define SKIN (LBS || a.seg[MULTI ? cseg : 0].sout != nullptr)
    int stage = 0, sb = 0;
    uint32_t phase = 0, sphase = 0;   // full[] parity; sfree[] parity of the S buffer's last use
    // tiles of this CTA, grouped by segment: the program switch sits outside the hot
    // loop (MULTI only; one group otherwise)
    int64_t it = 0;
    while (it < my_tiles) {
        int64_t it_end = my_tiles;
        if (MULTI) {
            const int64_t g0 = blockIdx.x + it * gridDim.x;
            if (g0 >= next_base) {   // first tile in a later segment: switch programs
                int s = cseg + 1;
                while (s + 1 < a.nseg && g0 >= a.seg[s + 1].tile_base) ++s;
                cseg = s;
                load_program(s);
            }
            if (next_base != INT64_MAX)
                it_end = min(it_end, (next_base - (int64_t)blockIdx.x + gridDim.x - 1) / gridDim.x);
        }
        for (; it < it_end; ++it) {
            const int64_t g = blockIdx.x + it * gridDim.x;
            float* L = LG + stage * tile_f;
            prof_mark(-1);
            HS_DELAY(5);
            mbar_wait(&full[stage], phase);
            prof_mark(0);
            if (PRO) {
                // phase 0 (Stage 1): the tile's local poses, computed into the stage buffer
                // by all consumer threads, consecutive elements on consecutive lanes
                // (coalesced key reads)
                const int64_t c0 = (g - SEGV(tile_base, tbase_g)) * SEGV(C, C_g);
                const int nel = (int)min((int64_t)SEGV(C, C_g), SEGV(n_chars, nch_g) - c0) * SEGV(J, J_g);
                const int nl = a.n_layers;
                const int4* dsc_t = desc + stage * SEGV(C, C_g) * nl;
                stage1_tile<HS_S1_E, HS_S1_PIPE != 0>(a.keys, dsc_t, nel, SEGV(J, J_g), nl, t, NC, L);
                bar_consumers(NC);
                prof_mark(8);   // phase 0 (Stage 1)
            }

            // phase 1: in-chunk fold, publish anchors (buffer 0 of P)
            float acc[12];
            if (p1 > 0) {
#pragma unroll
                for (int s = 0; s < K; ++s) {
                    if (s < p1) {
                        const int off = (int)(m[s] & 0xffff);
                        const int src = (int)(int16_t)(m[s] >> 32);
                        const int own = (int)(int16_t)(m[s] >> 48);
                        float l[12];
                        HS_BOUND(off >= 0 && (off + 1) * 12 <= tile_f);
                        ld3(L + off * 12, l);
                        if (src == kSrcPrev) {
                            float tmp[12];
                            compose(acc, l, tmp);
#pragma unroll
                            for (int e = 0; e < 12; ++e) acc[e] = tmp[e];
                        } else {
#pragma unroll
                            for (int e = 0; e < 12; ++e) acc[e] = l[e];
                        }
                        HS_BOUND(own < a.p_floats / 12);
                        if (own >= 0) st3(P + own * 12, acc);
                    }
                }
            }
            prof_mark(6);   // phase-1 fold of thread 0 (before any barrier)
            // phase 2a: heavy paths longer than K sit on consecutive lanes (runs); a
            // segmented warp-shuffle scan joins their pieces (Hillis-Steele over lanes,
            // parent on the left), then each run lane lifts its anchors by its exclusive
            // prefix.  No CTA barrier: runs never cross a warp.
            float excl[12];
            // longest run prefix in this warp: the scan needs ceil(log2(max + 1)) steps
            // (reduced per tile so the compiler sees a warp-uniform bound: no divergence
            // guards around the shuffles)
            const int warp_maxrb = RUNS ? (int)__reduce_max_sync(0xffffffffu, (unsigned)run_back) : 0;
            if (RUNS && warp_maxrb > 0) {   // warp-uniform: this warp holds run lanes
                for (int d = 1; d <= warp_maxrb; d <<= 1) {
                    float u[12];
#pragma unroll
                    for (int e = 0; e < 12; ++e) u[e] = __shfl_up_sync(0xffffffffu, acc[e], d);
                    if (run_back >= d) {
                        float w[12];
                        compose(u, acc, w);
#pragma unroll
                        for (int e = 0; e < 12; ++e) acc[e] = w[e];
                    }
                }
#pragma unroll
                for (int e = 0; e < 12; ++e) excl[e] = __shfl_up_sync(0xffffffffu, acc[e], 1);
                if (run_back > 0) {
#pragma unroll
                    for (int s = 0; s < K; ++s) {
                        const int own = (int)(int16_t)(m[s] >> 48);
                        if (own >= 0) {
                            float x[12], y[12];
                            HS_BOUND(own < a.p_floats / 12);
                            ld3(P + own * 12, x);
                            compose(excl, x, y);
                            st3(P + own * 12, y);
                        }
                    }
                }
            }
            prof_mark(7);   // phase-2a scan + lift of thread 0's warp
            bar_consumers(NC);

            prof_mark(1);
            // phase 2: pointer jumping over anchors (Alg. 2 on the anchor forest) with
            // snapshot semantics: ping-pong P, or a single P with every read of a round
            // before any of its writes (entries held in registers, <= 4 per thread).
            // Descriptors (slot | dst buf | self buf | link location) come from smem.
            for (int r = 0, nr = SEGV(R2, R2_g); r < nr; ++r) {
                const int eb = s_round_off[r], e1 = s_round_off[r + 1];
                if (!SEGV(p_single, psingle_g)) {
                    for (int e = eb + t; e < e1; e += NC) {
                        const uint32_t w = s_rounds[e];
                        const int slot = (int)(w & 0x3fff);
                        const int dst = slot + ((w >> 14) & 1) * SEGV(nslots, S2_g),
                                  self = slot + ((w >> 15) & 1) * SEGV(nslots, S2_g),
                                  link = (int)(w >> 16);
                        float x[12], y[12], z[12];
                        HS_BOUND(link >= 0 && link < a.p_floats / 12 && self < a.p_floats / 12 &&
                                 dst < a.p_floats / 12);
                        ld3(P + link * 12, x);
                        ld3(P + self * 12, y);
                        compose(x, y, z);
                        st3(P + dst * 12, z);
                    }
                    bar_consumers(NC);
                } else {
                    float z[4][12];
                    int dst[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int e = eb + t + q * NC;
                        dst[q] = -1;
                        if (e < e1) {
                            const uint32_t w = s_rounds[e];
                            float x[12], y[12];
                            HS_BOUND((int)(w >> 16) < a.p_floats / 12 && (int)(w & 0x3fff) < a.p_floats / 12);
                            ld3(P + (int)(w >> 16) * 12, x);
                            ld3(P + (int)(w & 0x3fff) * 12, y);
                            compose(x, y, z[q]);
                            dst[q] = (int)(w & 0x3fff);
                        }
                    }
                    bar_consumers(NC);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (dst[q] >= 0) st3(P + dst[q] * 12, z[q]);
                    bar_consumers(NC);
                }
            }
            prof_mark(2);

            // phase 3: final fold, G in place, S into the S buffer
            float* S = SB + sb * tile_f;
            // The S buffer's previous use must have been read out by the producer's bulk
            // store.  sphase tracks the parity of use it / NSS - 1, which is only right if
            // every use is awaited: a multi-segment launch can mix segments with and
            // without skin output, so it waits on every tile (the producer arrives on
            // sfree after every tile, skin or not).
            HS_DELAY(6);
            if ((SKIN || MULTI) && it >= NSS) mbar_wait(&sfree[sb], sphase);
            prof_mark(3);
            {
                float acc[12];
#pragma unroll
                for (int s = 0; s < K; ++s) {
                    const int src = (int)(int16_t)(m[s] >> 32);
                    if (src == kSrcNone) continue;
                    const int off = (int)(m[s] & 0xffff);
                    float l[12];
                    HS_BOUND(off >= 0 && (off + 1) * 12 <= tile_f);
                    ld3(L + off * 12, l);
                    if (RUNS) {
                        // the parent's global pose as the left operand, then ONE compose
                        // for every lane (lanes of a runs program mix sources at the same
                        // slot; divergent compose paths cost tree1024 4 %): the previous
                        // joint of the chunk, the identity at a root (I (x) l == l
                        // exactly for finite l), an anchor's final, or a run lane's
                        // P[run anchor] (x) exclusive scan
                        float left[12];
                        if (src == kSrcPrev) {
#pragma unroll
                            for (int e = 0; e < 12; ++e) left[e] = acc[e];
                        } else if (src == kSrcRoot) {
#pragma unroll
                            for (int e = 0; e < 12; ++e) left[e] = (e == 0 || e == 5 || e == 10) ? 1.0f : 0.0f;
                        } else if (src == kSrcRun) {
                            if (run_anchor >= 0) {
                                float pa[12];
                                HS_BOUND(run_anchor < a.p_floats / 12);
                                ld3(P + run_anchor * 12, pa);
                                compose(pa, excl, left);
                            } else {
#pragma unroll
                                for (int e = 0; e < 12; ++e) left[e] = excl[e];
                            }
                        } else {
                            HS_BOUND(src >= 0 && src < a.p_floats / 12);
                            ld3(P + src * 12, left);
                        }
                        compose(left, l, acc);
                    } else if (src == kSrcPrev) {
                        float tmp[12];
                        compose(acc, l, tmp);
#pragma unroll
                        for (int e = 0; e < 12; ++e) acc[e] = tmp[e];
                    } else if (src == kSrcRoot) {
#pragma unroll
                        for (int e = 0; e < 12; ++e) acc[e] = l[e];
                    } else {
                        float pa[12];
                        HS_BOUND(src >= 0 && src < a.p_floats / 12);
                        ld3(P + src * 12, pa);
                        compose(pa, l, acc);
                    }
                    st3(L + off * 12, acc);
                    if (SKIN) {
                        float sk[12];
                        compose(acc, ibr[s], sk);
                        st3(S + off * 12, sk);
                    }
                }
            }
            fence_proxy_async();
            HS_DELAY(7);
            bar_consumers(NC);
            HS_DELAY(8);
            if (t == 0) mbar_arrive(&done[stage]);
            if (LBS) {
                // linear blend skinning (R24): the tile's skin palette is in
                // the S buffer; vertex v of character c = sum_k w_k S[c][j_k] (p_v, 1).
                // Consecutive vertices on consecutive lanes (planar mesh arrays, L2-
                // resident, coalesced stores); the producer's bulk store of S only reads
                // the buffer.
                const SegArgs& S0 = a.seg[0];
                const int64_t c0 = (g - S0.tile_base) * S0.C;
                const int V = a.n_verts, Jn = S0.J;
                const int nct = (int)min((int64_t)S0.C, S0.n_chars - c0);   // characters in the tile
                const float* Sb = SB + sb * tile_f;
                float* vout = a.verts + c0 * V * 3;
                // vertex-major: mesh records of two vertices per thread loaded up front,
                // then every character of the tile (independent palette reads and
                // stores: ILP, no division)
                for (int v0 = t; v0 < V; v0 += kLbsU * NC) {
                    float4 pa[kLbsU], pb[kLbsU];
                    int js[kLbsU][4];
#pragma unroll
                    for (int u = 0; u < kLbsU; ++u) {
                        const int v = min(v0 + u * NC, V - 1);
                        pa[u] = __ldg(a.mesh_a + v);
                        pb[u] = __ldg(a.mesh_b + v);
                        mesh_joints(__ldg(a.mesh_j + v), js[u]);
                    }
                    for (int cl = 0; cl < nct; ++cl) {
                        const float* Sc = Sb + cl * Jn * 12;
#pragma unroll
                        for (int u = 0; u < kLbsU; ++u) {
                            const int v = v0 + u * NC;
                            HS_BOUND((cl + 1) * Jn * 12 <= tile_f && js[u][0] < Jn * 12 && js[u][1] < Jn * 12 &&
                                     js[u][2] < Jn * 12 && js[u][3] < Jn * 12);
                            if (v < V) lbs_vertex(Sc, pa[u], pb[u], js[u], vout + ((int64_t)cl * V + v) * 3);
                        }
                    }
                }
            }
            prof_mark(4);
            if (HS_PROF_HOOKS && a.prof && t == 0) atomicAdd(a.prof + 5, 1ull);
            if (++stage == NS) { stage = 0; phase ^= 1u; }
            if (++sb == NSS) { sb = 0; if (it + 1 >= 2 * NSS) sphase ^= 1u; }   // parity of use q-1
        }
    }
}
#undef SEGV
#undef SKIN

template <int K, int MODE>
void* chunked_ptr_m(bool runs) {
    return runs ? reinterpret_cast<void*>(&chunked_kernel<K, true, MODE>)
                : reinterpret_cast<void*>(&chunked_kernel<K, false, MODE>);
}

template <int K>
void* chunked_ptr(bool runs, int mode) {
    switch (mode) {
        case kModeScan: return chunked_ptr_m<K, kModeScan>(runs);
        case kModeStage1: return chunked_ptr_m<K, kModeStage1>(runs);
        case kModeMulti: return chunked_ptr_m<K, kModeMulti>(runs);
        case kModeSkin: return chunked_ptr_m<K, kModeSkin>(runs);
        default: return nullptr;
    }
}

void* chunked_fn(int K, bool runs, int mode) {
    switch (K) {
        case 3: return chunked_ptr<3>(runs, mode);
        case 5: return chunked_ptr<5>(runs, mode);
        case 7: return chunked_ptr<7>(runs, mode);
        case 9: return chunked_ptr<9>(runs, mode);
        case 11: return chunked_ptr<11>(runs, mode);
        default: return nullptr;
    }
}

}  // namespace

int sm_count() {   // of the current device, queried once per device
    static std::atomic<int> sms[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int n = sms[dev].load(std::memory_order_relaxed);
    if (n <= 0) {
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        sms[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

cudaError_t prepare_chunked(int K, int64_t smem_bytes) {
    // The attribute is per function, shared by every skeleton handle: raise it to the
    // device's opt-in maximum once so handles with different smem needs coexist.
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    if (smem_bytes > optin) return cudaErrorInvalidValue;
    for (bool runs : {false, true})
        for (int mode : {(int)kModeScan, (int)kModeStage1, (int)kModeMulti, (int)kModeSkin}) {
            void* fn = chunked_fn(K, runs, mode);
            if (!fn) return cudaErrorInvalidValue;
            e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
            if (e != cudaSuccess) return e;
        }
    return cudaSuccess;
}

int max_chunked_blocks_per_sm(int K, bool runs, int threads, int64_t smem_bytes) {
    // the occupancy query costs a few microseconds of host time per launch: remember
    // each (device, kernel, block shape) answer (a handful of shapes per process)
    struct Entry {
        int dev;
        const void* fn;
        int threads;
        int64_t smem;
        int nb;
    };
    static Entry cache[64];
    static int n_cached = 0;
    static std::mutex mu;
    void* fn = chunked_fn(K, runs, kModeScan);
    if (!fn) return 1;
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lock(mu);
        for (int i = 0; i < n_cached; ++i)
            if (cache[i].dev == dev && cache[i].fn == fn && cache[i].threads == threads && cache[i].smem == smem_bytes)
                return cache[i].nb;
    }
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, (size_t)smem_bytes) != cudaSuccess)
        return 1;
    nb = nb > 0 ? nb : 1;
    std::lock_guard<std::mutex> lock(mu);
    if (n_cached < 64) cache[n_cached++] = Entry{dev, fn, threads, smem_bytes, nb};
    return nb;
}

cudaError_t launch_chunked(int K, const ChunkedArgs& a, cudaStream_t st) {
    const int mode = a.layers != nullptr ? kModeStage1
                     : a.verts != nullptr ? kModeSkin
                     : (a.nseg > 1 ? kModeMulti : kModeScan);
    if ((mode == kModeStage1 || mode == kModeSkin) && a.nseg != 1) return cudaErrorInvalidValue;
    if (a.layers != nullptr && a.verts != nullptr) return cudaErrorInvalidValue;
    void* fn = chunked_fn(K, a.has_runs != 0, mode);
    if (!fn) return cudaErrorInvalidValue;
    const int64_t ntiles = a.total_tiles;
    int per_sm = a.ctas_per_sm > 0 ? a.ctas_per_sm
                                   : max_chunked_blocks_per_sm(K, a.has_runs != 0, a.threads, a.smem_bytes);
    int64_t grid = (int64_t)sm_count() * per_sm;
    if (grid > ntiles) grid = ntiles;
    if (grid < 1) grid = 1;
    ChunkedArgs args = a;
    void* params[] = {&args};
    return cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(a.threads), params, (size_t)a.smem_bytes, st);
}

}  // namespace hs
