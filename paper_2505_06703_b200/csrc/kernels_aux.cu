// kernels_aux.cu — the sm_100a kernels around the hot path: the streaming Stage-1
// kernel (two-pass hs_animate), the two-pass LBS kernel, the per-character-topology
// scan, the paper's comparison algorithms (Alg. 1 Gateau, Alg. 2 doubling, Alg. 3
// blocked, KIYA leaf walk) and the multi-CTA split path.  DESIGN.md §5.
#include <atomic>

#include "device_util.cuh"

namespace hs {
namespace {

// ================================================================== Stage 1, two-pass
// The same per-element Stage-1 arithmetic as the fused prologue (layer_desc +
// stage1_elems: bitwise the same local poses), as a high-occupancy streaming kernel
// that writes the local poses to a workspace for a plain chunked scan.  One thread
// per (character, joint) element, consecutive joints on consecutive lanes.
#ifndef HS_S1K_PER_THREAD
#define HS_S1K_PER_THREAD 8
#endif
#ifndef HS_S1K_UNROLL
#define HS_S1K_UNROLL 1
#endif
#ifndef HS_S1K_CTAS_PER_SM
#define HS_S1K_CTAS_PER_SM 16   // grid-stride cap (4 resident per SM; 16 measured ~1 % better than 8 on chain256)
#endif
#ifndef HS_S1K_TMA_STORE
#define HS_S1K_TMA_STORE 1
#endif
#ifndef HS_S1K_SPECIALISE
#define HS_S1K_SPECIALISE 1
#endif
constexpr int kStage1PerThread = HS_S1K_PER_THREAD;   // elements per thread between descriptor refreshes
constexpr int kStage1Unroll = HS_S1K_UNROLL;

template <int NLT>
__global__ void __launch_bounds__(256) stage1_kernel(const __grid_constant__ ChunkedArgs a, int64_t c0,
                                                     int64_t n_chars, float* __restrict__ local, int per) {
    extern __shared__ int4 sd[];   // layer descriptors of the block's characters
    __shared__ __align__(128) float stg[(HS_S1K_TMA_STORE ? 2 : 1) * 256 * 12];   // warps' local poses before the store
#if HS_S1K_TMA_STORE
    int it = 0;   // store-buffer parity
#endif
    const int J = a.seg[0].J, nl = NLT > 0 ? NLT : a.n_layers;
    const int lane = threadIdx.x & 31;
    const int64_t n = n_chars * J;
    const int4* lay = reinterpret_cast<const int4*>(a.layers);
    const int kTile = 256 * per;   // elements per block iteration (per <= kStage1PerThread)
    for (int64_t e0 = (int64_t)blockIdx.x * kTile; e0 < n; e0 += (int64_t)gridDim.x * kTile) {
        const int64_t cfirst = e0 / J;
        const int nc = (int)((min(n, e0 + (int64_t)kTile) - 1) / J - cfirst + 1);
        __syncthreads();   // the previous block-tile's readers are done
        for (int i = threadIdx.x; i < nc * nl; i += blockDim.x)
            sd[i] = layer_desc(a, __ldg(lay + (c0 + cfirst) * nl + i));
        __syncthreads();
        // element rel = cl * J + j of the block-tile, advanced by 256 without division
        int rel = (int)(e0 - cfirst * J) + threadIdx.x;
        int cl = rel / J, jj = rel - cl * J;
        const int sc = 256 / J, sj = 256 - sc * J;
#pragma unroll kStage1Unroll
        for (int q = 0; q < per; ++q) {
            const int64_t wbase = e0 + q * 256 + (threadIdx.x & ~31);   // the warp's first element
            if (wbase >= n) break;                                      // warp-uniform
            const bool ok = wbase + lane < n;
            HS_BOUND(!ok || (cl >= 0 && cl < nc && jj >= 0 && jj < J));
            const int j[1] = {ok ? jj : 0};
            const int4* dp[1] = {sd + (ok ? cl : 0) * nl};
            const bool valid[1] = {ok};
            const int off[1] = {0};
#if HS_S1K_TMA_STORE
            // the warp's 32 local poses are 1536 contiguous bytes: staged in smem (two
            // buffers per warp) and written by one TMA bulk store, so the LSU carries
            // only the key loads; the store of two iterations ago must have been read
            float* sbuf = stg + (it & 1) * 256 * 12;
            HS_DELAY(21);
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            stage1_elems<1, false, NLT>(a.keys, dp, j, valid, nl, J + (J & 1), sbuf + threadIdx.x * 12, off);
            fence_proxy_async();
            __syncwarp();
            HS_DELAY(22);
            if (lane == 0) {
                bulk_s2g(local + wbase * 12, sbuf + (threadIdx.x & ~31) * 12,
                         (uint32_t)(48 * min((int64_t)32, n - wbase)));
                bulk_commit();
            }
            ++it;
#else
            stage1_elems<1, false, NLT>(a.keys, dp, j, valid, nl, J + (J & 1), stg + threadIdx.x * 12, off);
            __syncwarp();
            // the warp's 32 local poses are 1536 contiguous bytes: write them as 96
            // lane-consecutive float4 (whole sectors) instead of 3 x 32 strided ones
            const int nv3 = 3 * (int)min((int64_t)32, n - wbase);
            const float4* src = reinterpret_cast<const float4*>(stg + (threadIdx.x & ~31) * 12);
            float4* dst = reinterpret_cast<float4*>(local + wbase * 12);
#pragma unroll
            for (int i = 0; i < 3; ++i)
                if (lane + 32 * i < nv3) dst[lane + 32 * i] = src[lane + 32 * i];
            __syncwarp();
#endif
            cl += sc;
            jj += sj;
            if (jj >= J) { jj -= J; ++cl; }
        }
    }
#if HS_S1K_TMA_STORE
    if (lane == 0) bulk_wait_all();   // smem stays valid until the last store has read it
#endif
}

// ================================================================== varied topology
#ifndef HS_VARIED_THREADS
#define HS_VARIED_THREADS 64
#endif
#ifndef HS_VARIED_M2_ABOVE
#define HS_VARIED_M2_ABOVE 128   // hs_scan_varied: two joints per thread above this size
#endif
// NEXT-3's per-character topology: every character brings its own parent array
// (4 B/joint more input), so nothing can be planned per skeleton.  One thread per
// (character, joint), C = max(1, 64 / J) characters per CTA — one character per CTA
// from J = 64 up, so each barrier spans one character's threads only (1024-thread
// CTAs of 16 hum64 characters were 1.7x slower); pointer jumping WITH the
// parent pointers (Alg. 2 with the Eq. 2 lift built on the fly): V[i] <- V[p[i]] (x)
// V[i], p[i] <- p[p[i]] on ping-pong snapshots until no pointer is left (at most
// ceil(log2 J) + 1 rounds, so a malformed array still terminates).
// M joints per thread (slots f, f + T, ... of the CTA's C characters, T = blockDim.x):
// M = 1 up to 128 joints; M = 2 above, so a 1024-joint character runs on 512 threads
// with at most 64 registers and two CTAs share an SM (one CTA's barrier waits overlap
// the other's rounds; a 1024-thread CTA per SM had nothing to overlap with), and each
// thread's two joints are independent work between barriers.  Measured
// (tools/time_varied.py): tree1024 1.71 -> 1.42 ms, chain256 0.74 -> 0.69 ms; M = 2
// from 32 joints or M = 4 above 128 / 512 were slower.
template <int M>
__global__ void __launch_bounds__(1024 / M, M == 1 ? 1 : 2)
    varied_kernel(const int32_t* __restrict__ parents, const float* __restrict__ local,
                  const float* __restrict__ ib, int J, int C, int64_t n_chars, int max_rounds,
                  float* __restrict__ gout, float* __restrict__ sout) {
    extern __shared__ __align__(16) float sm[];
    const int F = C * J;
    float* v0 = sm;
    float* v1 = sm + F * 12;
    int32_t* q0 = reinterpret_cast<int32_t*>(sm + 2 * F * 12);
    int32_t* q1 = q0 + F;
    const int64_t c0 = (int64_t)blockIdx.x * C;
    const int nc = (int)min((int64_t)C, n_chars - c0);
    const int T = blockDim.x;
    float v[M][12];
    int p[M];
    bool any_local = false;
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int f = threadIdx.x + m * T;
        const int cl = f / J;
        p[m] = -1;
        if (f < F && cl < nc) {
            ldg3(local + (c0 * J + f) * 12, v[m]);
            p[m] = __ldg(parents + c0 * J + f);
            if (p[m] < -1 || p[m] >= J) p[m] = -1;   // out of range: treated as a root (documented)
        }
        if (f < F) { st3(v0 + f * 12, v[m]); q0[f] = p[m]; }
        any_local |= p[m] >= 0;
    }
    float* vc = v0;
    float* vn = v1;
    int32_t* qc = q0;
    int32_t* qn = q1;
    // one barrier per round: the OR of "a pointer is left" rides on the barrier that
    // publishes the round's snapshot
    int any = __syncthreads_or(any_local);
    for (int r = 0; r < max_rounds && any; ++r) {
        any_local = false;
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const int f = threadIdx.x + m * T;
            if (f < F) {
                if (p[m] >= 0) {
                    const int base = (f / J) * J;
                    float x[12], y[12];
                    ld3(vc + (base + p[m]) * 12, x);
                    compose(x, v[m], y);
#pragma unroll
                    for (int e = 0; e < 12; ++e) v[m][e] = y[e];
                    p[m] = qc[base + p[m]];
                }
                st3(vn + f * 12, v[m]);
                qn[f] = p[m];
                any_local |= p[m] >= 0;
            }
        }
        any = __syncthreads_or(any_local);
        float* tv = vc; vc = vn; vn = tv;
        int32_t* tq = qc; qc = qn; qn = tq;
    }
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int f = threadIdx.x + m * T;
        if (f < F && f / J < nc) {
            st3(gout + (c0 * J + f) * 12, v[m]);
            if (sout) {
                float s[12];
                if (ib) {
                    float b[12];
                    ldg3(ib + (c0 * J + f) * 12, b);
                    compose(v[m], b, s);
                } else {
#pragma unroll
                    for (int e = 0; e < 12; ++e) s[e] = v[m][e];
                }
                st3(sout + (c0 * J + f) * 12, s);
            }
        }
    }
}

// ================================================================== blocked (Alg. 3)
// The paper's Alg. 3 literally, a comparison kernel: one thread
// per (character, joint) in USER order, B = 64-joint blocks over the internal
// topological order.  Stage A: pointer jumping along in-block parents only (ceil
// log2 B rounds on a ping-pong snapshot; reading R8 clamps the hops to the block).
// Stage B: walk MaxParentOutBlock, G = A[mpob] (x) G, on the stage-A snapshot
// (reading R9 walks the variable).  "6 + n/64" composes per thread.
__global__ void __launch_bounds__(1024) blocked_kernel(const float* __restrict__ local,
                                                       float* __restrict__ gout,
                                                       float* __restrict__ sout,
                                                       const float* __restrict__ ib,
                                                       const int32_t* __restrict__ lb,
                                                       const int32_t* __restrict__ mpob, int J, int C,
                                                       int RB, int64_t n_chars) {
    extern __shared__ __align__(16) float sm[];
    const int F = C * J;
    float* buf0 = sm;
    float* buf1 = sm + F * 12;
    const int64_t c0 = (int64_t)blockIdx.x * C;
    const int nc = (int)min((int64_t)C, n_chars - c0);
    const int f = threadIdx.x;
    const int cl = f / J, u = f - cl * J;
    const bool valid = f < F && cl < nc;
    float v[12];
    if (valid) ldg3(local + (c0 * J + f) * 12, v);
    if (f < F) st3(buf0 + f * 12, v);
    __syncthreads();
    float* cur = buf0;
    float* nxt = buf1;
    for (int r = 0; r < RB; ++r) {   // stage A
        if (f < F) {
            const int anc = __ldg(lb + (int64_t)r * J + u);
            if (anc >= 0) {
                float x[12], y[12];
                ld3(cur + (cl * J + anc) * 12, x);
                compose(x, v, y);
#pragma unroll
                for (int e = 0; e < 12; ++e) v[e] = y[e];
            }
            st3(nxt + f * 12, v);
        }
        __syncthreads();
        float* tmp = cur; cur = nxt; nxt = tmp;
    }
    if (valid) {   // stage B on the stage-A snapshot `cur`
        for (int m = __ldg(mpob + u); m >= 0; m = __ldg(mpob + m)) {
            float x[12], y[12];
            ld3(cur + (cl * J + m) * 12, x);
            compose(x, v, y);
#pragma unroll
            for (int e = 0; e < 12; ++e) v[e] = y[e];
        }
        st3(gout + (c0 * J + f) * 12, v);
        if (sout) {
            float b[12], s[12];
            ldg3(ib + (int64_t)u * 12, b);
            compose(v, b, s);
            st3(sout + (c0 * J + f) * 12, s);
        }
    }
}

// ================================================================== compressed (Alg. 4)
// The paper's final algorithm literally ("State compression"; reading
// R10), a comparison kernel: one thread per (character, joint) in USER order, 64-joint
// blocks over the internal topological order (as blocked_kernel).
//   stage A  7 serial composes with the LOCALS of the in-block ancestors at distance
//            1..7 (R5: Alg. 1-4's M[curParentID] read as the immutable locals;
//            R8: hops clamped to the block) -> A[j] covers distances 0..7;
//   barrier  ("groupbarrier")
//   stage B  7 composes with the stage-A SNAPSHOT of the in-block ancestors at distance
//            8, 16, ..., 56 (MultiParent(., 8)) -> B[j] covers the in-block root path;
//   barrier
//   stage C  the MaxParentOutBlock walk on the stage-B snapshot (R9: walk variable).
// "14 + n/64" composes per thread, two barriers per block.
__global__ void __launch_bounds__(1024) compressed_kernel(const float* __restrict__ local,
                                                          float* __restrict__ gout,
                                                          float* __restrict__ sout,
                                                          const float* __restrict__ ib,
                                                          const int32_t* __restrict__ lp,
                                                          const int32_t* __restrict__ l8,
                                                          const int32_t* __restrict__ mpob, int J, int C,
                                                          int64_t n_chars) {
    extern __shared__ __align__(16) float sm[];
    const int F = C * J;
    float* buf0 = sm;            // locals, then stage B
    float* buf1 = sm + F * 12;   // stage A
    const int64_t c0 = (int64_t)blockIdx.x * C;
    const int nc = (int)min((int64_t)C, n_chars - c0);
    const int f = threadIdx.x;
    const int cl = f / J, u = f - cl * J;
    const bool valid = f < F && cl < nc;
    float v[12];
    if (valid) ldg3(local + (c0 * J + f) * 12, v);
    if (f < F) st3(buf0 + f * 12, v);
    __syncthreads();
    if (f < F) {   // stage A: in-block ancestors at distance 1..7, their locals
        int cur = __ldg(lp + u);
        for (int d = 1; d <= 7 && cur >= 0; ++d) {
            float x[12], y[12];
            ld3(buf0 + (cl * J + cur) * 12, x);
            compose(x, v, y);
#pragma unroll
            for (int e = 0; e < 12; ++e) v[e] = y[e];
            cur = __ldg(lp + cur);
        }
        st3(buf1 + f * 12, v);
    }
    __syncthreads();
    if (f < F) {   // stage B: stride-8 ancestors' stage-A values
        int cur = __ldg(l8 + u);
        for (int d = 1; d <= 7 && cur >= 0; ++d) {
            float x[12], y[12];
            ld3(buf1 + (cl * J + cur) * 12, x);
            compose(x, v, y);
#pragma unroll
            for (int e = 0; e < 12; ++e) v[e] = y[e];
            cur = __ldg(l8 + cur);
        }
        st3(buf0 + f * 12, v);
    }
    __syncthreads();
    if (valid) {   // stage C: MaxParentOutBlock walk on the stage-B snapshot
        for (int m = __ldg(mpob + u); m >= 0; m = __ldg(mpob + m)) {
            float x[12], y[12];
            ld3(buf0 + (cl * J + m) * 12, x);
            compose(x, v, y);
#pragma unroll
            for (int e = 0; e < 12; ++e) v[e] = y[e];
        }
        st3(gout + (c0 * J + f) * 12, v);
        if (sout) {
            float b[12], s[12];
            ldg3(ib + (int64_t)u * 12, b);
            compose(v, b, s);
            st3(sout + (c0 * J + f) * 12, s);
        }
    }
}

// ================================================================== LBS, two-pass
// Skinning from skin poses in HBM: one CTA per character (grid-stride), its palette
// staged in shared memory (J x 48 B), then consecutive vertices on consecutive
// threads.  Several CTAs per SM (vs the scan kernel's one) hide the palette-read
// latency; costs one extra 48 B/joint read of S.
__global__ void __launch_bounds__(256) lbs_kernel(const float* __restrict__ S, int64_t n_chars, int J,
                                                  const float4* __restrict__ mesh_a,
                                                  const float4* __restrict__ mesh_b,
                                                  const int2* __restrict__ mesh_j, int V,
                                                  float* __restrict__ verts) {
    extern __shared__ float4 pal4[];
    const float* pal = reinterpret_cast<const float*>(pal4);
    float* vs = reinterpret_cast<float*>(pal4 + J * 3);   // the character's vertices, caller order
    for (int64_t c = blockIdx.x; c < n_chars; c += gridDim.x) {
        __syncthreads();   // the previous character's readers / writers are done
        const float4* src = reinterpret_cast<const float4*>(S + c * J * 12);
        for (int i = threadIdx.x; i < J * 3; i += blockDim.x) pal4[i] = __ldcs(src + i);
        __syncthreads();
        // mesh records in joint-sorted order (palette broadcasts), each written to its
        // caller-order slot in smem, then one coalesced copy out
        for (int v = threadIdx.x; v < V; v += blockDim.x) {
            int js[4];
            mesh_joints(__ldg(mesh_j + v), js);
            const float4 pb = __ldg(mesh_b + v);
            HS_BOUND(js[0] < J * 12 && js[1] < J * 12 && js[2] < J * 12 && js[3] < J * 12 &&
                     __float_as_int(pb.w) >= 0 && __float_as_int(pb.w) < V);
            lbs_vertex(pal, __ldg(mesh_a + v), pb, js, vs + (int64_t)__float_as_int(pb.w) * 3);
        }
        __syncthreads();
        float* vout = verts + c * V * 3;
        for (int i = threadIdx.x; i < V * 3; i += blockDim.x) __stcs(vout + i, vs[i]);
    }
}

// ================================================================== doubling (Alg. 2)
// One CTA per group of C characters, one thread per (character, joint) in USER
// order (pointer jumping is order-agnostic).  Round r: V[j] <- V[anc_r(j)] (x) V[j]
// on the previous round's snapshot (ping-pong smem), PAPER.md:113-124 with the
// "pow(2,n) layer parent" hop of PAPER.md:139 (reading R6).
__global__ void __launch_bounds__(1024) doubling_kernel(const float* __restrict__ local,
                                                        float* __restrict__ gout,
                                                        float* __restrict__ sout,
                                                        const float* __restrict__ ib,
                                                        const int32_t* __restrict__ lift, int J,
                                                        int C, int rounds, int64_t n_chars) {
    extern __shared__ __align__(16) float sm[];
    const int F = C * J;
    float* buf0 = sm;
    float* buf1 = sm + F * 12;
    const int64_t c0 = (int64_t)blockIdx.x * C;
    const int nc = (int)min((int64_t)C, n_chars - c0);
    const int f = threadIdx.x;
    const int cl = f / J, u = f - cl * J;
    const bool valid = f < F && cl < nc;
    float v[12];
    if (valid) ldg3(local + (c0 * J + f) * 12, v);
    if (f < F) st3(buf0 + f * 12, v);
    __syncthreads();
    float* cur = buf0;
    float* nxt = buf1;
    for (int r = 0; r < rounds; ++r) {
        if (f < F) {
            const int anc = __ldg(lift + (int64_t)r * J + u);
            if (anc >= 0) {
                float x[12], y[12];
                ld3(cur + (cl * J + anc) * 12, x);
                compose(x, v, y);
#pragma unroll
                for (int e = 0; e < 12; ++e) v[e] = y[e];
            }
            st3(nxt + f * 12, v);
        }
        __syncthreads();
        float* tmp = cur; cur = nxt; nxt = tmp;
    }
    if (valid) {
        st3(gout + (c0 * J + f) * 12, v);
        if (sout) {
            float b[12], s[12];
            ldg3(ib + (int64_t)u * 12, b);
            compose(v, b, s);
            st3(sout + (c0 * J + f) * 12, s);
        }
    }
}

// ================================================================== Gateau (Alg. 1)
__global__ void gateau_kernel(const float* __restrict__ local, float* __restrict__ gout,
                              float* __restrict__ sout, const float* __restrict__ ib,
                              const int32_t* __restrict__ parents, int J, int64_t n_chars) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n_chars * J) return;
    const int64_t c = idx / J;
    const int u = (int)(idx - c * J);
    const float* lc = local + c * J * 12;
    float acc[12];
    ldg3(lc + (int64_t)u * 12, acc);
    for (int p = __ldg(parents + u); p >= 0; p = __ldg(parents + p)) {  // reading R5
        float x[12], y[12];
        ldg3(lc + (int64_t)p * 12, x);
        compose(x, acc, y);
#pragma unroll
        for (int e = 0; e < 12; ++e) acc[e] = y[e];
    }
    st3(gout + idx * 12, acc);
    if (sout) {
        float b[12], s[12];
        ldg3(ib + (int64_t)u * 12, b);
        compose(acc, b, s);
        st3(sout + idx * 12, s);
    }
}

// ================================================================== KIYA leaf walk
__global__ void leaf_kernel(const float* __restrict__ local, float* __restrict__ gout,
                            float* __restrict__ sout, const float* __restrict__ ib,
                            const int32_t* __restrict__ path_off, const int32_t* __restrict__ path,
                            int n_leaves, int J, int64_t n_chars) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n_chars * n_leaves) return;
    const int64_t c = idx / n_leaves;
    const int leaf = (int)(idx - c * n_leaves);
    const float* lc = local + c * J * 12;
    float acc[12];
    const int e0 = __ldg(path_off + leaf), e1 = __ldg(path_off + leaf + 1);
    for (int e = e0; e < e1; ++e) {   // root ... leaf
        const int u = __ldg(path + e);
        float l[12];
        ldg3(lc + (int64_t)u * 12, l);
        if (e == e0) {
#pragma unroll
            for (int k = 0; k < 12; ++k) acc[k] = l[k];
        } else {
            float y[12];
            compose(acc, l, y);
#pragma unroll
            for (int k = 0; k < 12; ++k) acc[k] = y[k];
        }
        st3(gout + (c * J + u) * 12, acc);
        if (sout) {
            float b[12], s[12];
            ldg3(ib + (int64_t)u * 12, b);
            compose(acc, b, s);
            st3(sout + (c * J + u) * 12, s);
        }
    }
}

// ================================================================== split (multi-CTA)
// Thread per (character, chunk).  Global-memory fallback for skeletons that do
// not fit one CTA; the anchor scan between p1 and p3 is a recursive hs_scan on
// the anchor skeleton.
template <int K>
__global__ void split_p1_kernel(const float* __restrict__ local, float* __restrict__ pg,
                                const int4* __restrict__ meta, int nchunks, int J, int nslots,
                                int64_t n_chars) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n_chars * nchunks) return;
    const int64_t c = idx / nchunks;
    const int ch = (int)(idx - c * nchunks);
    const float* lc = local + c * J * 12;
    float* pc = pg + c * nslots * 12;
    float acc[12];
#pragma unroll
    for (int s = 0; s < K; ++s) {
        const int4 mm = __ldg(meta + (int64_t)ch * K + s);
        if (mm.y == kSrcNone) break;
        float l[12];
        ldg3(lc + (int64_t)mm.x * 12, l);
        if (mm.y == kSrcPrev) {
            float y[12];
            compose(acc, l, y);
#pragma unroll
            for (int e = 0; e < 12; ++e) acc[e] = y[e];
        } else {
#pragma unroll
            for (int e = 0; e < 12; ++e) acc[e] = l[e];
        }
        if (mm.z >= 0) st3(pc + (int64_t)mm.z * 12, acc);
    }
}

template <int K>
__global__ void split_p3_kernel(const float* __restrict__ local, float* __restrict__ gout,
                                float* __restrict__ sout, const float* __restrict__ ib,
                                const float* __restrict__ pf, const int4* __restrict__ meta,
                                int nchunks, int J, int nslots, int64_t n_chars) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n_chars * nchunks) return;
    const int64_t c = idx / nchunks;
    const int ch = (int)(idx - c * nchunks);
    const float* lc = local + c * J * 12;
    const float* pc = pf + c * nslots * 12;
    float acc[12];
#pragma unroll
    for (int s = 0; s < K; ++s) {
        const int4 mm = __ldg(meta + (int64_t)ch * K + s);
        if (mm.y == kSrcNone) break;
        float l[12];
        ldg3(lc + (int64_t)mm.x * 12, l);
        if (mm.y == kSrcPrev) {
            float y[12];
            compose(acc, l, y);
#pragma unroll
            for (int e = 0; e < 12; ++e) acc[e] = y[e];
        } else if (mm.y == kSrcRoot) {
#pragma unroll
            for (int e = 0; e < 12; ++e) acc[e] = l[e];
        } else {
            float pa[12];
            ldg3(pc + (int64_t)mm.y * 12, pa);
            compose(pa, l, acc);
        }
        st3(gout + (c * J + mm.x) * 12, acc);
        if (sout) {
            float b[12], sk[12];
            ldg3(ib + (int64_t)mm.x * 12, b);
            compose(acc, b, sk);
            st3(sout + (c * J + mm.x) * 12, sk);
        }
    }
}

// cudaFuncSetAttribute applies to the current device only: raise a kernel's dynamic
// shared-memory limit once per (kernel, device), remembered in a per-kernel bitmask.
cudaError_t raise_smem_once(const void* fn, int bytes, std::atomic<uint64_t>& done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = dev < 64 ? (1ull << dev) : 0;
    if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_release);
    return e;
}

}  // namespace

cudaError_t launch_stage1(const ChunkedArgs& a, int64_t c0, int64_t n_chars, float* local, cudaStream_t st) {
    const int64_t n = n_chars * a.seg[0].J;
    // elements per thread between descriptor refreshes: fewer when the block-tile's
    // layer descriptors would not fit shared memory beside the static staging buffer
    // (one-joint skeletons with many layers: 2048 characters x 8 layers x 16 B)
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) optin = 227 * 1024;
    const size_t stat = (HS_S1K_TMA_STORE ? 2 : 1) * 256 * 12 * sizeof(float);
    int per = kStage1PerThread;
    auto smem_of = [&](int q) { return (size_t)(256 * q / a.seg[0].J + 2) * a.n_layers * sizeof(int4); };
    while (per > 1 && smem_of(per) + stat > (size_t)optin) --per;
    const size_t smem = smem_of(per);
    if (smem + stat > (size_t)optin) return cudaErrorInvalidValue;
    int64_t blocks = (n + 256 * per - 1) / (256 * per);
    const int64_t cap = (int64_t)sm_count() * HS_S1K_CTAS_PER_SM;   // grid-stride CTAs of 256 per SM
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    ChunkedArgs args = a;
    void* params[] = {&args, &c0, &n_chars, &local, &per};
    // one, two and three layers (the common blends) get the unrolled layer loop
    const void* fn = !HS_S1K_SPECIALISE ? reinterpret_cast<const void*>(&stage1_kernel<0>)
                     : a.n_layers == 1   ? reinterpret_cast<const void*>(&stage1_kernel<1>)
                     : a.n_layers == 2 ? reinterpret_cast<const void*>(&stage1_kernel<2>)
                     : a.n_layers == 3 ? reinterpret_cast<const void*>(&stage1_kernel<3>)
                                       : reinterpret_cast<const void*>(&stage1_kernel<0>);
    if (smem + stat > 48 * 1024) {   // static + dynamic above the default 48 KB: opt in
        const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    return cudaLaunchKernel(fn, dim3((unsigned)blocks), dim3(256), params, smem, st);
}

cudaError_t launch_lbs(const float* S, int64_t n_chars, int32_t J, const float4* mesh_a, const float4* mesh_b,
                       const int2* mesh_j, int32_t V, float* verts, cudaStream_t st) {
    const size_t smem = (size_t)J * 48 + (size_t)V * 12;
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<void*>(&lbs_kernel),
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lbs_kernel, 256, smem);
    int64_t grid = (int64_t)sm_count() * std::max(per_sm, 1);
    if (grid > n_chars) grid = n_chars;
    if (grid < 1) grid = 1;
    lbs_kernel<<<(unsigned)grid, 256, smem, st>>>(S, n_chars, J, mesh_a, mesh_b, mesh_j, V, verts);
    return cudaGetLastError();
}

cudaError_t launch_doubling(const float* local, float* gout, float* sout, const float* ib,
                            const int32_t* lift, int32_t J, int32_t R, int32_t rounds,
                            int64_t n_chars, cudaStream_t st) {
    if (J > 1024) return cudaErrorInvalidValue;
    const int C = std::max(1, HS_VARIED_THREADS / J);   // one character per CTA from J = 64 up
    if (rounds < 0 || rounds > R) rounds = R;
    const size_t smem = (size_t)2 * C * J * 48;
    static std::atomic<uint64_t> attr{0};
    if (const cudaError_t e = raise_smem_once(reinterpret_cast<const void*>(&doubling_kernel), 2 * 1024 * 48, attr);
        e != cudaSuccess)
        return e;
    const int64_t blocks = (n_chars + C - 1) / C;
    doubling_kernel<<<(unsigned)blocks, C * J, smem, st>>>(local, gout, sout, ib, lift, J, C, rounds,
                                                           n_chars);
    return cudaGetLastError();
}

cudaError_t launch_varied(const int32_t* parents, const float* local, const float* ib, int32_t J,
                          int64_t n_chars, float* gout, float* sout, cudaStream_t st) {
    if (J < 1 || J > 1024) return cudaErrorInvalidValue;
    const int C = std::max(1, HS_VARIED_THREADS / J);   // characters per CTA
    int rounds = 1;
    while ((1 << (rounds - 1)) < J) ++rounds;   // ceil(log2 J) + 1: enough for any forest
    const size_t smem = (size_t)C * J * (2 * 48 + 2 * 4);
    static std::atomic<uint64_t> attr1{0}, attr2{0};
    const int64_t blocks = (n_chars + C - 1) / C;
    if (J <= HS_VARIED_M2_ABOVE) {
        if (const cudaError_t e = raise_smem_once(reinterpret_cast<const void*>(&varied_kernel<1>),
                                                  1024 * (2 * 48 + 2 * 4), attr1);
            e != cudaSuccess)
            return e;
        varied_kernel<1><<<(unsigned)blocks, C * J, smem, st>>>(parents, local, ib, J, C, n_chars, rounds, gout,
                                                               sout);
    } else {   // two joints per thread
        if (const cudaError_t e = raise_smem_once(reinterpret_cast<const void*>(&varied_kernel<2>),
                                                  1024 * (2 * 48 + 2 * 4), attr2);
            e != cudaSuccess)
            return e;
        varied_kernel<2><<<(unsigned)blocks, (C * J + 1) / 2, smem, st>>>(parents, local, ib, J, C, n_chars, rounds,
                                                                      gout, sout);
    }
    return cudaGetLastError();
}

cudaError_t launch_blocked(const float* local, float* gout, float* sout, const float* ib, const int32_t* lb,
                           const int32_t* mpob, int32_t J, int32_t RB, int64_t n_chars, cudaStream_t st) {
    if (J > 1024) return cudaErrorInvalidValue;
    const int C = std::max(1, HS_VARIED_THREADS / J);   // one character per CTA from J = 64 up
    const size_t smem = (size_t)2 * C * J * 48;
    static std::atomic<uint64_t> attr{0};
    if (const cudaError_t e = raise_smem_once(reinterpret_cast<const void*>(&blocked_kernel), 2 * 1024 * 48, attr);
        e != cudaSuccess)
        return e;
    const int64_t blocks = (n_chars + C - 1) / C;
    blocked_kernel<<<(unsigned)blocks, C * J, smem, st>>>(local, gout, sout, ib, lb, mpob, J, C, RB, n_chars);
    return cudaGetLastError();
}

cudaError_t launch_compressed(const float* local, float* gout, float* sout, const float* ib, const int32_t* lp,
                              const int32_t* l8, const int32_t* mpob, int32_t J, int64_t n_chars, cudaStream_t st) {
    if (J > 1024) return cudaErrorInvalidValue;
    const int C = std::max(1, HS_VARIED_THREADS / J);   // one character per CTA from J = 64 up
    const size_t smem = (size_t)2 * C * J * 48;
    static std::atomic<uint64_t> attr{0};
    if (const cudaError_t e = raise_smem_once(reinterpret_cast<const void*>(&compressed_kernel), 2 * 1024 * 48, attr);
        e != cudaSuccess)
        return e;
    const int64_t blocks = (n_chars + C - 1) / C;
    compressed_kernel<<<(unsigned)blocks, C * J, smem, st>>>(local, gout, sout, ib, lp, l8, mpob, J, C, n_chars);
    return cudaGetLastError();
}

cudaError_t launch_gateau(const float* local, float* gout, float* sout, const float* ib,
                          const int32_t* parents, int32_t J, int64_t n_chars, cudaStream_t st) {
    const int64_t n = n_chars * J;
    gateau_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(local, gout, sout, ib, parents, J, n_chars);
    return cudaGetLastError();
}

cudaError_t launch_leaf(const float* local, float* gout, float* sout, const float* ib,
                        const int32_t* path_off, const int32_t* path, int32_t n_leaves, int32_t J,
                        int64_t n_chars, cudaStream_t st) {
    const int64_t n = n_chars * n_leaves;
    leaf_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(local, gout, sout, ib, path_off, path,
                                                             n_leaves, J, n_chars);
    return cudaGetLastError();
}

#define HS_SPLIT_CASE(KK)                                                                        \
    case KK:                                                                                     \
        split_p1_kernel<KK><<<blocks, 128, 0, st>>>(local, pg, reinterpret_cast<const int4*>(meta), \
                                                    nchunks, J, nslots, n_chars);                 \
        break;

cudaError_t launch_split_p1(int K, const float* local, float* pg, const int32_t* meta,
                            int32_t nchunks, int32_t J, int32_t nslots, int64_t n_chars,
                            cudaStream_t st) {
    const int64_t n = n_chars * nchunks;
    const unsigned blocks = (unsigned)((n + 127) / 128);
    switch (K) {
        HS_SPLIT_CASE(3) HS_SPLIT_CASE(5) HS_SPLIT_CASE(7) HS_SPLIT_CASE(9) HS_SPLIT_CASE(11)
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}
#undef HS_SPLIT_CASE

#define HS_SPLIT_CASE(KK)                                                                         \
    case KK:                                                                                      \
        split_p3_kernel<KK><<<blocks, 128, 0, st>>>(local, gout, sout, ib, pf,                    \
                                                    reinterpret_cast<const int4*>(meta), nchunks, J, \
                                                    nslots, n_chars);                              \
        break;

cudaError_t launch_split_p3(int K, const float* local, float* gout, float* sout, const float* ib,
                            const float* pf, const int32_t* meta, int32_t nchunks, int32_t J,
                            int32_t nslots, int64_t n_chars, cudaStream_t st) {
    const int64_t n = n_chars * nchunks;
    const unsigned blocks = (unsigned)((n + 127) / 128);
    switch (K) {
        HS_SPLIT_CASE(3) HS_SPLIT_CASE(5) HS_SPLIT_CASE(7) HS_SPLIT_CASE(9) HS_SPLIT_CASE(11)
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace hs
