// kernels.cu — hand-written sm_100a kernels for the Hierarchy-Scan + fused
// Bind MeshPose (§1 steps 2-3, Eq. 1, Algs. 1-4).  DESIGN.md §5.
//
// Every pose is a 3x4 fp32 affine [R|t] (48 B).  compose(a, b) = a (x) b with
// the parent on the LEFT (Alg. 1's "M[jointID] = M[curParentID] * M[jointID]",
// PAPER.md:81).  No tensor cores: a chain of tiny 3x4 products is not a dense
// contraction (BASELINE.json north_star); the path is HBM-bound.
#include "kernels.cuh"

#include <algorithm>
#include <cstdint>

#ifndef HS_S1_E
#define HS_S1_E 1      // Stage-1 elements per thread per pass
#endif
#ifndef HS_S1_PIPE
#define HS_S1_PIPE 0   // issue layer l + 1's key loads before layer l's arithmetic
#endif

namespace hs {
namespace {

enum : int { kSrcRoot = -1, kSrcPrev = -2, kSrcNone = -3, kSrcRun = -4 };

// ------------------------------------------------------------------ 3x4 algebra
struct M34 {
    float v[12];
};

__device__ __forceinline__ void compose(const float* __restrict__ a, const float* __restrict__ b,
                                        float* __restrict__ c) {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            float x = a[4 * r + 0] * b[k];
            x = fmaf(a[4 * r + 1], b[4 + k], x);
            c[4 * r + k] = fmaf(a[4 * r + 2], b[8 + k], x);
        }
        float t = fmaf(a[4 * r + 0], b[3], a[4 * r + 3]);
        t = fmaf(a[4 * r + 1], b[7], t);
        c[4 * r + 3] = fmaf(a[4 * r + 2], b[11], t);
    }
}

__device__ __forceinline__ void ld3(const float* p, float* v) {
    const float4* q = reinterpret_cast<const float4*>(p);
    float4 a = q[0], b = q[1], c = q[2];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    v[8] = c.x; v[9] = c.y; v[10] = c.z; v[11] = c.w;
}

__device__ __forceinline__ void st3(float* p, const float* v) {
    float4* q = reinterpret_cast<float4*>(p);
    q[0] = make_float4(v[0], v[1], v[2], v[3]);
    q[1] = make_float4(v[4], v[5], v[6], v[7]);
    q[2] = make_float4(v[8], v[9], v[10], v[11]);
}

__device__ __forceinline__ void ldg3(const float* p, float* v) {
    const float4* q = reinterpret_cast<const float4*>(p);
    float4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    v[8] = c.x; v[9] = c.y; v[10] = c.z; v[11] = c.w;
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t a = smem_u32(bar);
    while (!mbar_try_wait(a, parity)) {
    }
}
// 1D bulk copy global -> shared, completion signalled on an mbarrier (TMA, UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// 1D bulk copy shared -> global (bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_consumers(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// ================================================================== Stage 1 (NEXT-1)
// Keyframe sampling, layer blending and TRS -> 3x4 (
// DESIGN.md readings R19-R23), fused ahead of the scan: the local pose is computed
// in shared memory instead of being read from HBM.  Keys on the device are packed
// per (clip, key) row as planar arrays over joints: float4 {tx,ty,tz,qw}, float4
// {qx,qy,qz,sx}, float2 {sy,sz} (40 B per key and joint, see load_keys).
// The time -> key decision uses the oracle's exact fp32 operation sequence.
__device__ __forceinline__ void key_index(float t, int n_keys, float fps, float duration, int wrap,
                                          int& k0, float& a) {
    if (n_keys <= 1) { k0 = 0; a = 0.0f; return; }
    float tt;
    if (wrap == 1) {
        const float q = floorf(__fdiv_rn(t, duration));
        tt = __fsub_rn(t, __fmul_rn(q, duration));
        if (tt < 0.0f) tt = 0.0f;
    } else {
        tt = t < 0.0f ? 0.0f : (t > duration ? duration : t);
    }
    const float u = __fmul_rn(tt, fps);
    const float kf = floorf(u);
    float frac = __fsub_rn(u, kf);
    int ki = (int)kf;
    if (ki >= n_keys - 1) { ki = n_keys - 1; frac = 0.0f; }
    if (ki < 0) { ki = 0; frac = 0.0f; }
    k0 = ki;
    a = frac;
}

// MUFU approximations (rel. error ~2^-22): a unit quaternion's norm and the weight
// sum are far from denormal, so the IEEE fix-up paths of rsqrtf / '/' buy nothing.
__device__ __forceinline__ float rsqrt_fast(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_fast(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Layer descriptor of one (character, layer) of a tile, written by the producer
// warp ahead of the consumers (smem ring, one slot per stage):
//   x = float4 index of key k0 of the layer's clip at joint 0,
//   y = float4 offset from key k0 to key k0 + 1 (0 when frac == 0: one key),
//   z = frac (fp32 bits), w = weight (fp32 bits).
__device__ __forceinline__ int4 layer_desc(const ChunkedArgs& a, int4 L) {
    int k0;
    float fr;
    key_index(__int_as_float(L.y), a.n_keys, a.fps, a.duration, a.wrap, k0, fr);
    const int Jp = a.seg[0].J + (a.seg[0].J & 1);   // joints padded to even (16-byte planes)
    const int row = (L.x * a.n_keys + k0) * Jp * 10;
    return make_int4(row, fr != 0.0f ? Jp * 10 : 0, __float_as_int(fr), L.z);
}

// Sample (keys x0..z0 at k0, x1..z1 at k0 + 1): trs = t(3), q(w,x,y,z)(4), s(3).
__device__ __forceinline__ void sample_trs(float4 x0, float4 y0, float2 z0, float4 x1, float4 y1,
                                           float2 z1, float a, float* trs) {
    if (a == 0.0f) {   // on a key: that key exactly (R21)
        trs[0] = x0.x; trs[1] = x0.y; trs[2] = x0.z; trs[3] = x0.w;
        trs[4] = y0.x; trs[5] = y0.y; trs[6] = y0.z;
        trs[7] = y0.w; trs[8] = z0.x; trs[9] = z0.y;
        return;
    }
    const float b = 1.0f - a;
    trs[0] = b * x0.x + a * x1.x; trs[1] = b * x0.y + a * x1.y; trs[2] = b * x0.z + a * x1.z;
    trs[7] = b * y0.w + a * y1.w; trs[8] = b * z0.x + a * z1.x; trs[9] = b * z0.y + a * z1.y;
    const float d = x0.w * x1.w + y0.x * y1.x + y0.y * y1.y + y0.z * y1.z;
    const float as = d < 0.0f ? -a : a;
    float qw = b * x0.w + as * x1.w, qx = b * y0.x + as * y1.x, qy = b * y0.y + as * y1.y,
          qz = b * y0.z + as * y1.z;
    const float inv = rsqrt_fast(qw * qw + qx * qx + qy * qy + qz * qz);
    trs[3] = qw * inv; trs[4] = qx * inv; trs[5] = qy * inv; trs[6] = qz * inv;
}

__device__ __forceinline__ void trs_to_m34(const float* trs, float* m) {
    const float w = trs[3], x = trs[4], y = trs[5], z = trs[6];
    const float sx = trs[7], sy = trs[8], sz = trs[9];
    m[0] = (1.0f - 2.0f * (y * y + z * z)) * sx; m[1] = 2.0f * (x * y - w * z) * sy;
    m[2] = 2.0f * (x * z + w * y) * sz;          m[3] = trs[0];
    m[4] = 2.0f * (x * y + w * z) * sx;          m[5] = (1.0f - 2.0f * (x * x + z * z)) * sy;
    m[6] = 2.0f * (y * z - w * x) * sz;          m[7] = trs[1];
    m[8] = 2.0f * (x * z - w * y) * sx;          m[9] = 2.0f * (y * z + w * x) * sy;
    m[10] = (1.0f - 2.0f * (x * x + y * y)) * sz; m[11] = trs[2];
}

// Local poses of E tile elements at once (E independent (character, joint) pairs,
// so each layer's 6 * E key loads are in flight together; PIPE also issues layer
// l + 1's loads before layer l's arithmetic): sample every layer, blend (DESIGN.md
// R22), TRS -> 3x4, store into the tile in smem.
struct KeyPair {
    float4 x0, y0, x1, y1;
    float2 z0, z1;
};

// Keys are planar, 40 bytes per (key, joint): per (clip, key) row of 10 * Jp floats
// (Jp = joints padded to even), plane 0 = float4 {t, qw}, plane 1 = float4 {q.xyz, sx},
// plane 2 = float2 {sy, sz}; a warp's loads of one plane over consecutive joints are
// contiguous.  d.x = the row's float offset, d.y = the step to key k0 + 1 (0: one key).
__device__ __forceinline__ KeyPair load_keys(const float* __restrict__ keys, int4 d, int j, int Jp) {
    const float* p0 = keys + d.x;
    const float* p1 = p0 + d.y;
    KeyPair k;
    k.x0 = __ldg(reinterpret_cast<const float4*>(p0) + j);
    k.y0 = __ldg(reinterpret_cast<const float4*>(p0 + 4 * Jp) + j);
    k.z0 = __ldg(reinterpret_cast<const float2*>(p0 + 8 * Jp) + j);
    k.x1 = __ldg(reinterpret_cast<const float4*>(p1) + j);
    k.y1 = __ldg(reinterpret_cast<const float4*>(p1 + 4 * Jp) + j);
    k.z1 = __ldg(reinterpret_cast<const float2*>(p1 + 8 * Jp) + j);
    return k;
}

template <int E, bool PIPE>
__device__ __forceinline__ void stage1_elems(const float* __restrict__ keys, const int4* const* dsc,
                                             const int* j, const bool* valid, int nl, int Jp, float* L,
                                             const int* off) {
    float acc[E][10], q0[E][4], wsum[E];
    KeyPair kp[E];
    int4 d[E];
    if (PIPE) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            d[e] = valid[e] ? dsc[e][0] : make_int4(0, 0, 0, 0);
            kp[e] = load_keys(keys, d[e], j[e], Jp);
        }
    }
    for (int l = 0; l < nl; ++l) {
        KeyPair cur[E];
        int4 dc[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (PIPE) {
                cur[e] = kp[e];
                dc[e] = d[e];
                if (l + 1 < nl) {
                    d[e] = valid[e] ? dsc[e][l + 1] : make_int4(0, 0, 0, 0);
                    kp[e] = load_keys(keys, d[e], j[e], Jp);
                }
            } else {
                dc[e] = valid[e] ? dsc[e][l] : make_int4(0, 0, 0, 0);
                cur[e] = load_keys(keys, dc[e], j[e], Jp);
            }
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            float s[10];
            sample_trs(cur[e].x0, cur[e].y0, cur[e].z0, cur[e].x1, cur[e].y1, cur[e].z1,
                       __int_as_float(dc[e].z), s);
            const float w = __int_as_float(dc[e].w);
            if (nl == 1) {   // one layer: the sample itself (R22)
#pragma unroll
                for (int c = 0; c < 10; ++c) acc[e][c] = s[c];
            } else if (l == 0) {
#pragma unroll
                for (int c = 0; c < 4; ++c) q0[e][c] = s[3 + c];
#pragma unroll
                for (int c = 0; c < 10; ++c) acc[e][c] = w * s[c];
                wsum[e] = w;
            } else {
                const float dq = s[3] * q0[e][0] + s[4] * q0[e][1] + s[5] * q0[e][2] + s[6] * q0[e][3];
                const float ws = dq < 0.0f ? -w : w;
#pragma unroll
                for (int c = 0; c < 3; ++c) acc[e][c] += w * s[c];
#pragma unroll
                for (int c = 3; c < 7; ++c) acc[e][c] += ws * s[c];
#pragma unroll
                for (int c = 7; c < 10; ++c) acc[e][c] += w * s[c];
                wsum[e] += w;
            }
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (!valid[e]) continue;
        if (nl > 1) {
            const float iw = rcp_fast(wsum[e]);
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[e][c] *= iw;
#pragma unroll
            for (int c = 7; c < 10; ++c) acc[e][c] *= iw;
            const float inv = rsqrt_fast(acc[e][3] * acc[e][3] + acc[e][4] * acc[e][4] +
                                     acc[e][5] * acc[e][5] + acc[e][6] * acc[e][6]);
#pragma unroll
            for (int c = 3; c < 7; ++c) acc[e][c] *= inv;
        }
        float m[12];
        trs_to_m34(acc[e], m);
        st3(L + off[e] * 12, m);
    }
}

// Phase 0 over one tile: element o = (character o / J, joint o % J) of the tile,
// consecutive elements on consecutive threads (coalesced key reads), E per thread
// per pass.
template <int E, bool PIPE>
__device__ __forceinline__ void stage1_tile(const float* __restrict__ keys, const int4* dsc_t, int nel,
                                            int J, int nl, int t, int NC, float* L) {
    // element o = cl * J + j, advanced by E * NC per pass without a division
    const int step = E * NC, step_c = step / J, step_j = step - step_c * J;
    int cl0 = t / J, j0 = t - (t / J) * J;
    for (int o = t; o < nel; o += step) {
        int off[E], j[E];
        bool valid[E];
        const int4* dsc[E];
        int cl = cl0, jj = j0;
#pragma unroll
        for (int q = 0; q < E; ++q) {
            off[q] = o + q * NC;
            valid[q] = off[q] < nel;
            j[q] = valid[q] ? jj : 0;
            dsc[q] = dsc_t + (valid[q] ? cl : 0) * nl;
            if (q + 1 < E) {
                jj += NC;
                while (jj >= J) { jj -= J; ++cl; }
            }
        }
        stage1_elems<E, PIPE>(keys, dsc, j, valid, nl, J + (J & 1), L, off);
        cl0 += step_c;
        j0 += step_j;
        if (j0 >= J) { j0 -= J; ++cl0; }
    }
}

// ================================================================== LBS (NEXT-4)
// One skinned vertex (R24): sum_k w_k S[j_k] (p, 1) with the character's
// skin palette `pal` ([J][12], shared memory); joints pre-multiplied by 12.  The
// fused epilogue and the two-pass kernel share it, so their vertices are bitwise equal.
__device__ __forceinline__ void lbs_vertex(const float* pal, float4 pa, float4 pb, const int* js, float* d) {
    const float ws[4] = {pa.w, pb.x, pb.y, pb.z};
    float x = 0.f, y = 0.f, z = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        float m[12];
        ld3(pal + js[q], m);
        const float px = fmaf(m[0], pa.x, fmaf(m[1], pa.y, fmaf(m[2], pa.z, m[3])));
        const float py = fmaf(m[4], pa.x, fmaf(m[5], pa.y, fmaf(m[6], pa.z, m[7])));
        const float pz = fmaf(m[8], pa.x, fmaf(m[9], pa.y, fmaf(m[10], pa.z, m[11])));
        x = fmaf(ws[q], px, x);
        y = fmaf(ws[q], py, y);
        z = fmaf(ws[q], pz, z);
    }
    d[0] = x; d[1] = y; d[2] = z;
}

__device__ __forceinline__ void mesh_joints(int2 jj, int* js) {
    js[0] = (jj.x & 0xffff) * 12; js[1] = (int)((uint32_t)jj.x >> 16) * 12;
    js[2] = (jj.y & 0xffff) * 12; js[3] = (int)((uint32_t)jj.y >> 16) * 12;
}

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
            mbar_expect_tx(&full[stage], bytes);
            const char* src = reinterpret_cast<const char*>(ld.local + c0 * ld.J * 12);
            char* dst = reinterpret_cast<char*>(LG + stage * tile_f);
            for (uint32_t o = 0; o < bytes; o += piece)
                bulk_g2s(dst + o, src + o, min(piece, bytes - o), &full[stage]);
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
            mbar_wait(&done[stage], phase);
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
            {
                char* gp = reinterpret_cast<char*>(st.gout + c0 * st.J * 12);
                const char* sg = reinterpret_cast<const char*>(LG + stage * tile_f);
                char* sp = do_skin ? reinterpret_cast<char*>(st.sout + c0 * st.J * 12) : nullptr;
                const char* ss = reinterpret_cast<const char*>(SB + sb * tile_f);
                for (uint32_t o = 0; o < bytes; o += piece) {
                    const uint32_t nb = min(piece, bytes - o);
                    bulk_s2g(gp + o, sg + o, nb);
                    if (do_skin) bulk_s2g(sp + o, ss + o, nb);
                }
            }
            bulk_commit();
            bulk_wait_read<0>();                  // smem of this tile has been read out
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
                if (src != kSrcNone) ldg3(S.ib + (int64_t)ibu * 12, ibr[s2]);
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
        if (a.prof && t == 0) {
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
            if (SKIN && it >= NSS) mbar_wait(&sfree[sb], sphase);
            prof_mark(3);
            {
                float acc[12];
#pragma unroll
                for (int s = 0; s < K; ++s) {
                    const int src = (int)(int16_t)(m[s] >> 32);
                    if (src == kSrcNone) continue;
                    const int off = (int)(m[s] & 0xffff);
                    float l[12];
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
                                ld3(P + run_anchor * 12, pa);
                                compose(pa, excl, left);
                            } else {
#pragma unroll
                                for (int e = 0; e < 12; ++e) left[e] = excl[e];
                            }
                        } else {
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
            bar_consumers(NC);
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
                for (int v0 = t; v0 < V; v0 += 2 * NC) {
                    float4 pa[2], pb[2];
                    int js[2][4];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int v = min(v0 + u * NC, V - 1);
                        pa[u] = __ldg(a.mesh_a + v);
                        pb[u] = __ldg(a.mesh_b + v);
                        mesh_joints(__ldg(a.mesh_j + v), js[u]);
                    }
                    for (int cl = 0; cl < nct; ++cl) {
                        const float* Sc = Sb + cl * Jn * 12;
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const int v = v0 + u * NC;
                            if (v < V) lbs_vertex(Sc, pa[u], pb[u], js[u], vout + ((int64_t)cl * V + v) * 3);
                        }
                    }
                }
            }
            prof_mark(4);
            if (a.prof && t == 0) atomicAdd(a.prof + 5, 1ull);
            if (++stage == NS) { stage = 0; phase ^= 1u; }
            if (++sb == NSS) { sb = 0; if (it + 1 >= 2 * NSS) sphase ^= 1u; }   // parity of use q-1
        }
    }
}
#undef SEGV
#undef SKIN

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
constexpr int kStage1PerThread = HS_S1K_PER_THREAD;   // elements per thread between descriptor refreshes
constexpr int kStage1Unroll = HS_S1K_UNROLL;

__global__ void __launch_bounds__(256) stage1_kernel(const __grid_constant__ ChunkedArgs a, int64_t c0,
                                                     int64_t n_chars, float* __restrict__ local) {
    extern __shared__ int4 sd[];   // layer descriptors of the block's characters
    const int J = a.seg[0].J, nl = a.n_layers;
    const int64_t n = n_chars * J;
    const int4* lay = reinterpret_cast<const int4*>(a.layers);
    constexpr int kTile = 256 * kStage1PerThread;   // elements per block iteration
    for (int64_t e0 = (int64_t)blockIdx.x * kTile; e0 < n; e0 += (int64_t)gridDim.x * kTile) {
        const int64_t cfirst = e0 / J;
        const int nc = (int)((min(n, e0 + kTile) - 1) / J - cfirst + 1);
        __syncthreads();   // the previous block-tile's readers are done
        for (int i = threadIdx.x; i < nc * nl; i += blockDim.x)
            sd[i] = layer_desc(a, __ldg(lay + (c0 + cfirst) * nl + i));
        __syncthreads();
        // element rel = cl * J + j of the block-tile, advanced by 256 without division
        int rel = (int)(e0 - cfirst * J) + threadIdx.x;
        int cl = rel / J, jj = rel - cl * J;
        const int sc = 256 / J, sj = 256 - sc * J;
#pragma unroll kStage1Unroll
        for (int q = 0; q < kStage1PerThread; ++q) {
            const int64_t e = e0 + q * 256 + threadIdx.x;
            if (e >= n) break;
            const int j[1] = {jj};
            const int4* dp[1] = {sd + cl * nl};
            const bool valid[1] = {true};
            const int off[1] = {0};
            stage1_elems<1, false>(a.keys, dp, j, valid, nl, J + (J & 1), local + e * 12, off);
            cl += sc;
            jj += sj;
            if (jj >= J) { jj -= J; ++cl; }
        }
    }
}

// ================================================================== varied topology
// NEXT-3's per-character topology: every character brings its own parent array
// (4 B/joint more input), so nothing can be planned per skeleton.  One thread per
// (character, joint), C = 1024 / J characters per CTA; pointer jumping WITH the
// parent pointers (Alg. 2 with the Eq. 2 lift built on the fly): V[i] <- V[p[i]] (x)
// V[i], p[i] <- p[p[i]] on ping-pong snapshots until no pointer is left (at most
// ceil(log2 J) + 1 rounds, so a malformed array still terminates).
__global__ void __launch_bounds__(1024) varied_kernel(const int32_t* __restrict__ parents,
                                                      const float* __restrict__ local,
                                                      const float* __restrict__ ib, int J, int C,
                                                      int64_t n_chars, int max_rounds,
                                                      float* __restrict__ gout, float* __restrict__ sout) {
    extern __shared__ __align__(16) float sm[];
    const int F = C * J;
    float* v0 = sm;
    float* v1 = sm + F * 12;
    int32_t* q0 = reinterpret_cast<int32_t*>(sm + 2 * F * 12);
    int32_t* q1 = q0 + F;
    const int64_t c0 = (int64_t)blockIdx.x * C;
    const int nc = (int)min((int64_t)C, n_chars - c0);
    const int f = threadIdx.x;
    const int cl = f / J;
    const bool valid = f < F && cl < nc;
    float v[12];
    int p = -1;
    if (valid) {
        ldg3(local + (c0 * J + f) * 12, v);
        p = __ldg(parents + c0 * J + f);
        if (p < -1 || p >= J) p = -1;   // out of range: treated as a root (documented)
    }
    if (f < F) { st3(v0 + f * 12, v); q0[f] = p; }
    float* vc = v0;
    float* vn = v1;
    int32_t* qc = q0;
    int32_t* qn = q1;
    __syncthreads();
    for (int r = 0; r < max_rounds; ++r) {
        if (!__syncthreads_or(p >= 0)) break;
        if (f < F) {
            if (p >= 0) {
                float x[12], y[12];
                ld3(vc + (cl * J + p) * 12, x);
                compose(x, v, y);
#pragma unroll
                for (int e = 0; e < 12; ++e) v[e] = y[e];
                p = qc[cl * J + p];
            }
            st3(vn + f * 12, v);
            qn[f] = p;
        }
        __syncthreads();
        float* tv = vc; vc = vn; vn = tv;
        int32_t* tq = qc; qc = qn; qn = tq;
    }
    if (valid) {
        st3(gout + (c0 * J + f) * 12, v);
        if (sout) {
            float s[12];
            if (ib) {
                float b[12];
                ldg3(ib + (c0 * J + f) * 12, b);
                compose(v, b, s);
            } else {
#pragma unroll
                for (int e = 0; e < 12; ++e) s[e] = v[e];
            }
            st3(sout + (c0 * J + f) * 12, s);
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

int g_sms = 0;
int sm_count() {
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_sms <= 0) g_sms = 148;
    }
    return g_sms;
}

}  // namespace

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
    void* fn = chunked_fn(K, runs, kModeScan);
    int nb = 0;
    if (!fn || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, (size_t)smem_bytes) !=
                   cudaSuccess)
        return 1;
    return nb > 0 ? nb : 1;
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

cudaError_t launch_stage1(const ChunkedArgs& a, int64_t c0, int64_t n_chars, float* local, cudaStream_t st) {
    const int64_t n = n_chars * a.seg[0].J;
    int64_t blocks = (n + 256 * kStage1PerThread - 1) / (256 * kStage1PerThread);
    const int64_t cap = (int64_t)sm_count() * 8;   // grid-stride, 8 CTAs of 256 per SM
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    ChunkedArgs args = a;
    void* params[] = {&args, &c0, &n_chars, &local};
    const size_t smem = (size_t)(256 * kStage1PerThread / a.seg[0].J + 2) * a.n_layers * sizeof(int4);
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<void*>(&stage1_kernel),
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    return cudaLaunchKernel(reinterpret_cast<void*>(&stage1_kernel), dim3((unsigned)blocks), dim3(256), params,
                            smem, st);
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
    int C = 1024 / J;
    if (C < 1) C = 1;
    if (rounds < 0 || rounds > R) rounds = R;
    const size_t smem = (size_t)2 * C * J * 48;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(doubling_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 1024 * 48);
        attr = true;
    }
    const int64_t blocks = (n_chars + C - 1) / C;
    doubling_kernel<<<(unsigned)blocks, C * J, smem, st>>>(local, gout, sout, ib, lift, J, C, rounds,
                                                           n_chars);
    return cudaGetLastError();
}

cudaError_t launch_varied(const int32_t* parents, const float* local, const float* ib, int32_t J,
                          int64_t n_chars, float* gout, float* sout, cudaStream_t st) {
    if (J < 1 || J > 1024) return cudaErrorInvalidValue;
    const int C = std::max(1, 1024 / J);
    int rounds = 1;
    while ((1 << (rounds - 1)) < J) ++rounds;   // ceil(log2 J) + 1: enough for any forest
    const size_t smem = (size_t)C * J * (2 * 48 + 2 * 4);
    static bool attr = false;
    if (!attr) {
        const cudaError_t e = cudaFuncSetAttribute(varied_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   1024 * (2 * 48 + 2 * 4));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int64_t blocks = (n_chars + C - 1) / C;
    varied_kernel<<<(unsigned)blocks, C * J, smem, st>>>(parents, local, ib, J, C, n_chars, rounds, gout, sout);
    return cudaGetLastError();
}

cudaError_t launch_blocked(const float* local, float* gout, float* sout, const float* ib, const int32_t* lb,
                           const int32_t* mpob, int32_t J, int32_t RB, int64_t n_chars, cudaStream_t st) {
    if (J > 1024) return cudaErrorInvalidValue;
    int C = 1024 / J;
    if (C < 1) C = 1;
    const size_t smem = (size_t)2 * C * J * 48;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(blocked_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 1024 * 48);
        attr = true;
    }
    const int64_t blocks = (n_chars + C - 1) / C;
    blocked_kernel<<<(unsigned)blocks, C * J, smem, st>>>(local, gout, sout, ib, lb, mpob, J, C, RB, n_chars);
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
#undef HS_SPLIT_CASE

}  // namespace hs
