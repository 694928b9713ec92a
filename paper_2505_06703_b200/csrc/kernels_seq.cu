// kernels_seq.cu — the multi-tile kernel (HS_ALGO_TILES): skeletons
// larger than one CTA's shared memory (the cross-block carry of
// Alg. 3).
//
// The skeleton's internal (topological) order is cut into KT tiles of <= F joints
// (plan.cpp build_seq_program).  A persistent CTA takes whole characters b, b + grid,
// ... and runs each one's tiles in order 0..KT-1, so when a tile runs, every joint
// outside it that it depends on (an earlier tile's joint) already has its FINAL global
// pose — the cross-block carry is resolved before the block, not walked after it.
// Per tile, the same three phases as the single-CTA chunked kernel (kernels.cu) on
// the tile's sub-forest, whose external parents are Q locations (final roots):
//   phase 1  per-thread chunk folds, anchor prefixes published to P;
//   phase 2a warp-shuffle scan of runs (heavy paths longer than K);
//   phase 2  pointer jumping over the anchor forest, whose roots are true roots
//            and Q locations (already final);
//   phase 3  re-fold from the final anchors, G in place, S = G (x) IB in place over
//            the tile's inverse binds, and a joint with a child in the next tile
//            forwards its G into that tile's Q buffer.
// Parents two or more tiles back reach Q through the tile's inbox: after each tile the
// compute threads store its exported joints into later tiles' inboxes (a contiguous
// workspace range per consumer tile, coalesced, L2-resident), and during tile k - 1
// the threads stage tile k's inbox into its Q buffer through registers.
// The producer warp's lane 0 streams, by TMA bulk copies with mbarrier completion,
// the tiles in (one copy per run of consecutive user labels: one run per tile when
// the user order is already topological), G and S out, each tile's program (chunk
// metadata, phase-1 info, phase-2 descriptors; three tiles ahead), export list and
// inverse binds (into the tile's S buffer).  DESIGN.md §5.1e.
//
// HBM bytes per joint: 48 (L in) + 48 (G out) + 48 (S out), as the single-CTA path;
// the workspace (one character's inboxes per CTA), programs and inverse binds stay
// in L2.
#include <atomic>

#include "device_util.cuh"

namespace hs {
namespace {

template <int K, bool RUNS>
__global__ void __launch_bounds__(256, 1) seq_kernel(const __grid_constant__ SeqArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int NS = a.stages, NSS = a.sbufs;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* done = full + 4;
    uint64_t* ibfull = done + 4;   // S buffer holds the tile's inverse binds (TMA), S computed in place
    uint64_t* progfull = ibfull + 4;   // [3]: a tile program has landed (TMA by the producer)
    uint64_t* exlfull = progfull + 3;  // [1]: the export list of the current tile has landed
    const int tile_f = a.F * 12;
    float* LG = reinterpret_cast<float*>(smem + kSeqHeaderBytes);
    float* SB = LG + NS * tile_f;
    float* P = SB + NSS * tile_f;
    // three program buffers (tile counter mod 3), each: meta [T][K] | p1 [T] | round_off
    // [r2p] | rounds [entp] (16-byte multiples, TMA destinations)
    const int TK = a.T * K;
    const int PROGW = TK * 2 + a.T + a.r2p + a.entp;                        // 4-byte words
    int32_t* s_prog = reinterpret_cast<int32_t*>(P + a.p_floats);
    int2* s_exl = reinterpret_cast<int2*>(s_prog + 3 * PROGW);              // [max_exl]
    SeqTileDev* s_tiles = reinterpret_cast<SeqTileDev*>(s_exl + a.max_exl);  // [KT]
    auto prog_meta = [&](int b) { return reinterpret_cast<const uint64_t*>(s_prog + b * PROGW); };
    auto prog_p1 = [&](int b) { return s_prog + b * PROGW + 2 * TK; };
    auto prog_roff = [&](int b) { return s_prog + b * PROGW + 2 * TK + a.T; };
    auto prog_rounds = [&](int b) {
        return reinterpret_cast<const uint32_t*>(s_prog + b * PROGW + 2 * TK + a.T + a.r2p);
    };

    const int nwc = (int)(blockDim.x >> 5) - 1;   // consumer warps; then the TMA producer warp
    const int NC = nwc * 32;
    const int warp = threadIdx.x >> 5;
    const int KT = a.KT;
    const int J = a.J;
    const int64_t my_chars = blockIdx.x < a.n_chars ? (a.n_chars - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t my_tiles = my_chars * KT;

    for (int i = threadIdx.x; i < KT * (int)(sizeof(SeqTileDev) / 4); i += blockDim.x)
        reinterpret_cast<int32_t*>(s_tiles)[i] = __ldg(reinterpret_cast<const int32_t*>(a.tiles) + i);
    if (threadIdx.x == 0) {
        // done: every consumer thread arrives after its share of the tile's exports
        for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&done[s], NC); }
        for (int s = 0; s < NSS; ++s) mbar_init(&ibfull[s], 1);
        for (int s = 0; s < 3; ++s) mbar_init(&progfull[s], 1);
        mbar_init(exlfull, 1);
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == nwc) {
        // ------------------------------------------------------------ producer
        // lane 0 streams tiles, programs, inverse binds and export lists
        if ((threadIdx.x & 31) != 0) return;
        const uint32_t piece = a.bulk_piece > 0 ? (uint32_t)a.bulk_piece : 0xffffffffu;
        const uint64_t stream_pol = policy_evict_first(), keep_pol = policy_evict_last();
        // tile cursors (character, tile) for the loads (NS ahead) and the stores
        int64_t lc = blockIdx.x, sc = blockIdx.x;
        int lk = 0, sk = 0;
        auto issue_load = [&](int stage) {
            const SeqTileDev tl = s_tiles[lk];
            mbar_expect_tx(&full[stage], (uint32_t)tl.nj * 48u);
            const char* base = reinterpret_cast<const char*>(a.local + lc * J * 12);
            char* dst = reinterpret_cast<char*>(LG + stage * tile_f);
            for (int r = 0; r < tl.n_runs; ++r) {
                const int4 run = __ldg(a.runs + tl.runs_off + r);
                const uint32_t bytes = (uint32_t)run.z * 48u;
                HS_BOUND(run.y >= 0 && run.y + run.z <= tl.nj && run.x >= 0 && run.x + run.z <= J);
                const char* s0 = base + (int64_t)run.x * 48;
                char* d0 = dst + run.y * 48;
                for (uint32_t o = 0; o < bytes; o += piece)
                    bulk_g2s_hint(d0 + o, s0 + o, min(piece, bytes - o), &full[stage], stream_pol);
            }
            if (++lk == KT) { lk = 0; lc += gridDim.x; }
        };
        // tile programs: counter c's tile into program buffer c % 3, three tiles ahead (so a
        // tile's import list is in place when the tile before it stages the imports)
        int pk = 0;
        auto issue_prog = [&](int buf) {
            const SeqTileDev tl = s_tiles[pk];
            const uint32_t b_meta = (uint32_t)TK * 8u, b_p1 = (uint32_t)a.T * 4u, b_ro = (uint32_t)a.r2p * 4u;
            const uint32_t b_rd = (uint32_t)((tl.n_entries + 3) & ~3) * 4u;
            mbar_expect_tx(&progfull[buf], b_meta + b_p1 + b_ro + b_rd);
            int32_t* d = s_prog + buf * PROGW;
            bulk_g2s(d, a.meta + (int64_t)pk * TK, b_meta, &progfull[buf]);
            bulk_g2s(d + 2 * TK, a.p1len + (int64_t)pk * a.T, b_p1, &progfull[buf]);
            bulk_g2s(d + 2 * TK + a.T, a.round_off + (int64_t)pk * a.r2p, b_ro, &progfull[buf]);
            if (b_rd) bulk_g2s(d + 2 * TK + a.T + a.r2p, a.rounds + tl.rounds_off, b_rd, &progfull[buf]);
            if (++pk == KT) pk = 0;
        };
        const bool do_skin = a.sout != nullptr;
        // inverse binds of a tile, by smem offset, into its S buffer (phase 3 computes
        // S = G (x) IB in place: each slot is read and then written by one thread)
        int ibk = 0;
        auto issue_ib = [&](int buf) {
            const SeqTileDev tl = s_tiles[ibk];
            const uint32_t bytes = (uint32_t)tl.nj * 48u;
            mbar_expect_tx(&ibfull[buf], bytes);
            const char* src = reinterpret_cast<const char*>(a.ib + (int64_t)ibk * a.F * 12);
            char* dst = reinterpret_cast<char*>(SB + buf * tile_f);
            for (uint32_t o = 0; o < bytes; o += piece)
                bulk_g2s_hint(dst + o, src + o, min(piece, bytes - o), &ibfull[buf], keep_pol);
            if (++ibk == KT) ibk = 0;
        };
        // the export list of a tile into the (single) export-list buffer
        auto issue_exl = [&](int j) {
            const SeqTileDev tl = s_tiles[j];
            const uint32_t bytes = (uint32_t)((tl.n_exl + 1) & ~1) * 8u;
            mbar_expect_tx(exlfull, bytes);
            if (bytes) bulk_g2s(s_exl, a.exl + tl.exl_off, bytes, exlfull);
        };
        {
            if (my_tiles > 0) issue_exl(0);
            for (int64_t it = 0; it < my_tiles && it < 3; ++it) issue_prog((int)it);
            for (int64_t it = 0; it < my_tiles && it < NS; ++it) issue_load((int)it);
            if (do_skin)
                for (int64_t it = 0; it < my_tiles && it < NSS; ++it) issue_ib((int)it);
        }
        int stage = 0, sb = 0, pbuf = 0;
        uint32_t phase = 0;
        for (int64_t it = 0; it < my_tiles; ++it) {
            HS_DELAY(11);
            mbar_wait(&done[stage], phase);
            HS_DELAY(12);
            const SeqTileDev tl = s_tiles[sk];
            if (it + 1 < my_tiles) issue_exl(sk + 1 < KT ? sk + 1 : 0);   // read by tile it's exports: done
            if (it + 3 < my_tiles) issue_prog(pbuf);   // tile it no longer reads its program
            if (++pbuf == 3) pbuf = 0;
            {
                const int64_t cbase = sc * J * 12;
                const char* sg = reinterpret_cast<const char*>(LG + stage * tile_f);
                const char* ss = reinterpret_cast<const char*>(SB + sb * tile_f);
                for (int r = 0; r < tl.n_runs; ++r) {
                    const int4 run = __ldg(a.runs + tl.runs_off + r);
                    const uint32_t bytes = (uint32_t)run.z * 48u;
                    char* gp = reinterpret_cast<char*>(a.gout + cbase) + (int64_t)run.x * 48;
                    char* sp = do_skin ? reinterpret_cast<char*>(a.sout + cbase) + (int64_t)run.x * 48 : nullptr;
                    for (uint32_t o = 0; o < bytes; o += piece) {
                        const uint32_t nb = min(piece, bytes - o);
                        bulk_s2g_hint(gp + o, sg + run.y * 48 + o, nb, stream_pol);
                        if (do_skin) bulk_s2g_hint(sp + o, ss + run.y * 48 + o, nb, stream_pol);
                    }
                }
                bulk_commit();
            }
            HS_DELAY(13);
            {
                bulk_wait_read<0>();
                HS_DELAY(14);
                if (do_skin && it + NSS < my_tiles) issue_ib(sb);   // the S buffer has been read out
                if (it + NS < my_tiles) issue_load(stage);
            }
            if (++sk == KT) { sk = 0; sc += gridDim.x; }
            if (++stage == NS) { stage = 0; phase ^= 1u; }
            if (++sb == NSS) sb = 0;
        }
        bulk_wait_all();
        return;
    }

    // ---------------------------------------------------------------- consumers
    // A tile's program (chunk metadata, phase-1 info, phase-2 tables) and its export
    // list arrive by TMA ahead of it.  Its Q values: parents in tile k - 1 are
    // forwarded into Q by the threads that compute them in phase 3 of tile k - 1;
    // parents in tiles <= k - 2 form the tile's inbox, staged during tile k - 1 through
    // registers (coalesced 16-byte loads): the rows exported by tiles <= k - 3 at the
    // top of tile k - 1, the rows exported by tile k - 2 after its phase-2 barrier.
    // After phase 3 each tile stores its exports (the joints tiles two or more later
    // read) into their inboxes.  Q buffers alternate with the tile index k (the plan
    // bakes the locations in).
    const int t = threadIdx.x;
    const bool skin = a.sout != nullptr;
    float* wsb = a.ws + (int64_t)blockIdx.x * a.n_exp * 12;   // this CTA's workspace (inboxes)
    const uint64_t ws_pol = policy_evict_last();
    const int qb0 = 2 * a.S, nQ = a.nQ;
    // profiling builds (HS_PROF_HOOKS): consumer thread 0's cycles per phase, summed
    long long prof_last = 0;
    auto prof_mark = [&](int slot) {
        if (HS_PROF_HOOKS && a.prof && t == 0) {
            const long long now = clock64();
            if (slot >= 0) atomicAdd(a.prof + slot, (unsigned long long)(now - prof_last));
            prof_last = now;
        }
    };
    uint64_t m[K];
    int stage = 0, sb = 0, pb = 0, k = 0;     // pb: program buffer (tile counter mod 3)
    uint32_t phase = 0, sphase = 0, pphase = 0;
    for (int64_t it = 0; it < my_tiles; ++it) {
        const SeqTileDev tl = s_tiles[k];
        float* L = LG + stage * tile_f;
        prof_mark(-1);
        HS_DELAY(15);
        mbar_wait(&progfull[pb], pphase);
        prof_mark(0);
        int p1, run_back, run_anchor;
        {
            const int info = t < a.T ? prog_p1(pb)[t] : 0;
            p1 = info & 0xff;
            run_back = (info >> 8) & 0xff;
            run_anchor = (int)((uint32_t)info >> 16) - 1;
        }
#pragma unroll
        for (int s = 0; s < K; ++s) m[s] = t < a.T ? prog_meta(pb)[t * K + s] : kSeqMetaNone;
        // the next tile's inbox: the rows exported by tiles <= k - 2 (before the barriers
        // of tile k - 1) now, the rest after this tile's phase-2 barrier
        float4 inb[kSeqInboxPieces], inl[kSeqInboxLate];   // early / late pieces (distinct registers:
        int nin3 = 0, ine3 = 0, inq = 0;                    // a late load must not wait for an early one)
        const float* insrc = wsb;
        if (it + 1 < my_tiles) {
            const SeqTileDev tn = s_tiles[k + 1 < KT ? k + 1 : 0];
            nin3 = 3 * tn.n_imp;
            ine3 = 3 * tn.n_early;
            inq = (qb0 + ((k + 1) & 1) * nQ) * 12;
            insrc = wsb + (int64_t)tn.imp_off * 12;
#pragma unroll
            for (int u = 0; u < kSeqInboxPieces; ++u) {
                const int q = t + u * NC;
                if (q < ine3) inb[u] = ldg4_hint(insrc + 4 * q, ws_pol);
            }
        }
        prof_mark(1);
        HS_DELAY(16);
        mbar_wait(&full[stage], phase);
        prof_mark(2);

        // phase 1: in-chunk fold, publish anchors
        float acc[12];
        if (p1 > 0) {
#pragma unroll
            for (int s = 0; s < K; ++s) {
                if (s < p1) {
                    const int off = seq_off(m[s]);
                    const int src = seq_src(m[s]);
                    const int own = seq_own(m[s]);
                    float l[12];
                    HS_BOUND(off >= 0 && off < tl.nj);
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
                    HS_BOUND(own < 2 * a.S);
                    if (own >= 0) st3(P + own * 12, acc);
                }
            }
        }
        // phase 2a: runs (warp-shuffle segmented scan), as in kernels.cu
        float excl[12];
        const int warp_maxrb = RUNS ? (int)__reduce_max_sync(0xffffffffu, (unsigned)run_back) : 0;
        if (RUNS && warp_maxrb > 0) {
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
                    const int own = seq_own(m[s]);
                    if (own >= 0) {
                        float x[12], y[12];
                        ld3(P + own * 12, x);
                        compose(excl, x, y);
                        st3(P + own * 12, y);
                    }
                }
            }
        }
        prof_mark(3);
        bar_consumers(NC);   // anchors published; this tile's Q and tables visible to all
        prof_mark(4);

        // phase 2: pointer jumping over the anchor forest (ping-pong P; Q roots final)
        const int32_t* s_round_off = prog_roff(pb);
        const uint32_t* s_rounds = prog_rounds(pb);
        for (int r = 0; r < tl.R2; ++r) {
            const int eb = s_round_off[r], e1 = s_round_off[r + 1];
            for (int e = eb + t; e < e1; e += NC) {
                const uint32_t w = s_rounds[e];
                const int slot = (int)(w & 0x3fff);
                const int dst = slot + ((w >> 14) & 1) * a.S, self = slot + ((w >> 15) & 1) * a.S,
                          link = (int)(w >> 16);
                float x[12], y[12], z[12];
                HS_BOUND(link >= 0 && (link + 1) * 12 <= a.p_floats && self < 2 * a.S && dst < 2 * a.S);
                ld3(P + link * 12, x);
                ld3(P + self * 12, y);
                compose(x, y, z);
                st3(P + dst * 12, z);
            }
            bar_consumers(NC);
        }

        prof_mark(10);
        // the rest of the next tile's inbox: rows exported by the previous tile (its
        // exports preceded this tile's phase-2 barrier)
        if (ine3 < nin3) {
#pragma unroll
            for (int u = 0; u < kSeqInboxLate; ++u) {
                const int q = ine3 + t + u * NC;
                if (q < nin3) inl[u] = ldg4_hint(insrc + 4 * q, ws_pol);
            }
        }
        // phase 3: final fold, G in place, S into the S buffer, exports to the workspace
        float* S = SB + sb * tile_f;
        prof_mark(5);
        if (skin) mbar_wait(&ibfull[sb], sphase);   // this tile's inverse binds are in S
        prof_mark(6);
        {
            float acc3[12];
#pragma unroll
            for (int s = 0; s < K; ++s) {
                const int src = seq_src(m[s]);
                if (src == kSrcNone) continue;
                const int off = seq_off(m[s]);
                const int fw = seq_fwd(m[s]);
                float l[12];
                HS_BOUND(off >= 0 && off < tl.nj);
                ld3(L + off * 12, l);
                float ibv[12];   // loaded with L: the stores below could alias it for the compiler
                if (skin) ld3(S + off * 12, ibv);
                if (RUNS) {
                    float left[12];
                    if (src == kSrcPrev) {
#pragma unroll
                        for (int e = 0; e < 12; ++e) left[e] = acc3[e];
                    } else if (src == kSrcRoot) {
#pragma unroll
                        for (int e = 0; e < 12; ++e) left[e] = (e == 0 || e == 5 || e == 10) ? 1.0f : 0.0f;
                    } else if (src == kSrcRun) {
                        if (run_anchor >= 0) {
                            float pa[12];
                            HS_BOUND((run_anchor + 1) * 12 <= a.p_floats);
                            ld3(P + run_anchor * 12, pa);
                            compose(pa, excl, left);
                        } else {
#pragma unroll
                            for (int e = 0; e < 12; ++e) left[e] = excl[e];
                        }
                    } else {
                        HS_BOUND(src >= 0 && (src + 1) * 12 <= a.p_floats);
                        ld3(P + src * 12, left);
                    }
                    compose(left, l, acc3);
                } else if (src == kSrcPrev) {
                    float tmp[12];
                    compose(acc3, l, tmp);
#pragma unroll
                    for (int e = 0; e < 12; ++e) acc3[e] = tmp[e];
                } else if (src == kSrcRoot) {
#pragma unroll
                    for (int e = 0; e < 12; ++e) acc3[e] = l[e];
                } else {
                    float pa[12];
                    HS_BOUND(src >= 0 && (src + 1) * 12 <= a.p_floats);
                    ld3(P + src * 12, pa);
                    compose(pa, l, acc3);
                }
                st3(L + off * 12, acc3);
                if (fw) {   // a child in tile k + 1: forward into that tile's Q buffer
                    HS_BOUND(fw - 1 < nQ);
                    st3(P + (qb0 + ((k + 1) & 1) * nQ + fw - 1) * 12, acc3);
                }
                if (skin) {
                    float sk[12];
                    compose(acc3, ibv, sk);
                    st3(S + off * 12, sk);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kSeqInboxPieces; ++u) {
            const int q = t + u * NC;
            if (q < ine3) *reinterpret_cast<float4*>(P + inq + 4 * q) = inb[u];
        }
#pragma unroll
        for (int u = 0; u < kSeqInboxLate; ++u) {
            const int q = ine3 + t + u * NC;
            if (q < nin3) *reinterpret_cast<float4*>(P + inq + 4 * q) = inl[u];
        }
        prof_mark(7);
        fence_proxy_async();   // smem G/S for the bulk stores
        HS_DELAY(17);
        bar_consumers(NC);     // the whole tile's G is in shared memory
        prof_mark(8);
        if (HS_PROF_HOOKS && a.prof && t == 0) atomicAdd(a.prof + 9, 1ull);
        // the next tile's inbox has been read by every thread (its pieces are in Q): its
        // L2 lines are dead, so drop the ones lying wholly inside it without a write-back
        // (the workspace would otherwise reach DRAM as dirty evictions)
        if (nin3) {
            const uintptr_t b0 = reinterpret_cast<uintptr_t>(insrc), b1 = b0 + (uintptr_t)nin3 * 16;
            for (uintptr_t p = ((b0 + 127) & ~(uintptr_t)127) + (uintptr_t)t * 128; p + 128 <= b1;
                 p += (uintptr_t)NC * 128)
                discard_l2(reinterpret_cast<const void*>(p));
        }
        // exports: the tile's joints that later tiles read (two or more tiles on) into
        // their inboxes; consecutive threads store consecutive 16-byte pieces of each
        // contiguous inbox range (coalesced)
        {
            const int n3 = 3 * tl.n_exl;
            if (n3) {
                HS_DELAY(18);
                mbar_wait(exlfull, (uint32_t)(it & 1));
                for (int q0 = t; q0 < n3; q0 += kSeqExportUnroll * NC) {
                    float4 v[kSeqExportUnroll];
                    int dst[kSeqExportUnroll];
#pragma unroll
                    for (int u = 0; u < kSeqExportUnroll; ++u) {   // independent loads first (ILP)
                        const int q = q0 + u * NC;
                        dst[u] = -1;
                        if (q < n3) {
                            const int e = q / 3, c = q - 3 * e;
                            const int2 x = s_exl[e];
                            HS_BOUND(x.x >= 0 && x.x < tl.nj && x.y >= 0 && x.y < a.n_exp);
                            v[u] = *reinterpret_cast<const float4*>(L + x.x * 12 + 4 * c);
                            dst[u] = x.y * 12 + 4 * c;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kSeqExportUnroll; ++u)
                        if (dst[u] >= 0) st4_hint(wsb + dst[u], v[u], ws_pol);
                }
            }
        }
        prof_mark(11);
        HS_DELAY(19);
        mbar_arrive(&done[stage]);   // every consumer thread (count NC): its exports read the stage
        if (++stage == NS) { stage = 0; phase ^= 1u; }
        if (++sb == NSS) { sb = 0; sphase ^= 1u; }   // parity of use it / NSS of buffer sb
        if (++pb == 3) { pb = 0; pphase ^= 1u; }     // program buffer use (it / 3) parity

        if (++k == KT) k = 0;
    }
}

void* seq_fn(int K, bool runs) {
    switch (K) {
        case 3: return runs ? (void*)&seq_kernel<3, true> : (void*)&seq_kernel<3, false>;
        case 5: return runs ? (void*)&seq_kernel<5, true> : (void*)&seq_kernel<5, false>;
        case 7: return runs ? (void*)&seq_kernel<7, true> : (void*)&seq_kernel<7, false>;
        default: return nullptr;
    }
}

}  // namespace

cudaError_t prepare_seq(int K) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    for (bool runs : {false, true}) {
        void* fn = seq_fn(K, runs);
        if (!fn) return cudaErrorInvalidValue;
        if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin)) != cudaSuccess)
            return e;
    }
    return cudaSuccess;
}

cudaError_t launch_seq(int K, const SeqArgs& a, cudaStream_t st) {
    void* fn = seq_fn(K, a.has_runs != 0);
    if (!fn) return cudaErrorInvalidValue;
    int64_t grid = (int64_t)sm_count() * (a.ctas_per_sm > 0 ? a.ctas_per_sm : 1);
    if (grid > a.n_chars) grid = a.n_chars;
    if (grid < 1) grid = 1;
    SeqArgs args = a;
    void* params[] = {&args};
    return cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(a.threads), params, (size_t)a.smem_bytes, st);
}

}  // namespace hs
