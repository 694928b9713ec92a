// device_util.cuh — device helpers shared by the sm_100a kernels (kernels.cu,
// kernels_aux.cu): 3x4 algebra, shared-memory / TMA / mbarrier primitives, the
// Stage-1 sampling and blending functions (NEXT-1) and the LBS vertex (NEXT-4).
// Everything is __device__ __forceinline__ in an unnamed namespace (one copy per TU).
#pragma once

#include "kernels.cuh"

#include <algorithm>
#include <cstdint>

// HS_DEBUG_BOUNDS=1 (a debug build, tests/test_gpu_bounds.py): every shared-memory
// slot index and TMA byte count is checked against its buffer; a violation traps.
// compute-sanitizer is closed on this pool, so this build stands in for memcheck.
#ifndef HS_DEBUG_BOUNDS
#define HS_DEBUG_BOUNDS 0
#endif
#if HS_DEBUG_BOUNDS
#include <cstdio>
#define HS_BOUND(cond)                                                                       \
    do {                                                                                      \
        if (!(cond)) {                                                                        \
            printf("hs bounds violated: %s (%s:%d, block %d thread %d)\n", #cond, __FILE__, \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                             \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define HS_BOUND(cond) \
    do {               \
    } while (0)
#endif
// Protocol stress build (HS_DEBUG_DELAY=1, tests/test_gpu_stress.py): random sleeps of
// up to ~4 us at the producer / consumer hand-off points of the TMA + mbarrier kernels,
// so a missing wait, a parity slip or an early buffer reuse shows up as a wrong bit in
// the bitwise parity suites instead of hiding behind the usual timing.  Compiled out
// of the shipped library.
#ifndef HS_DEBUG_DELAY
#define HS_DEBUG_DELAY 0
#endif
#if HS_DEBUG_DELAY
#define HS_DELAY(site) hs_debug_delay(site)
#else
#define HS_DELAY(site) \
    do {               \
    } while (0)
#endif
#ifndef HS_S1_E
#define HS_S1_E 1      // Stage-1 elements per thread per pass
#endif
#ifndef HS_S1_PIPE
#define HS_S1_PIPE 0   // issue layer l + 1's key loads before layer l's arithmetic
#endif

namespace hs {
namespace {


enum : int { kSrcRoot = -1, kSrcPrev = -2, kSrcNone = -3, kSrcRun = -4 };

// Multi-tile program slot word (plan.cpp build_seq_program): smem offset (10 bits),
// src + 8 (13), own + 1 (13), workspace export slot + 1 (16), next-tile Q forward + 1 (12).
constexpr uint64_t kSeqMetaNone = (uint64_t)(kSrcNone + 8) << 10;   // src none, own -1, no export
__device__ __forceinline__ int seq_off(uint64_t m) { return (int)(m & 0x3ff); }
__device__ __forceinline__ int seq_src(uint64_t m) { return (int)((m >> 10) & 0x1fff) - 8; }
__device__ __forceinline__ int seq_own(uint64_t m) { return (int)((m >> 23) & 0x1fff) - 1; }
__device__ __forceinline__ int seq_ex(uint64_t m) { return (int)((m >> 36) & 0xffff); }
__device__ __forceinline__ int seq_fwd(uint64_t m) { return (int)((m >> 52) & 0xfff); }

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
#if HS_DEBUG_DELAY
__device__ __forceinline__ void hs_debug_delay(unsigned site) {
    unsigned x = (unsigned)clock() ^ (blockIdx.x * 0x9E3779B9u) ^ (threadIdx.x * 0x85EBCA6Bu) ^ (site * 0xC2B2AE35u);
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    if ((x & 3) == 0) __nanosleep((x >> 8) & 4095);
}
#endif
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
// generic-proxy writes (shared AND global) ordered before later async-proxy (TMA) accesses
__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// L2 cache policies (createpolicy): streaming data that is touched once (tiles in, G and S
// out) is marked evict_first, so data that is re-read within the kernel (the multi-tile
// path's workspace of exported poses, the per-skeleton tables) stays in L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* gdst, const void* ssrc, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void st3_hint(float* p, const float* v, uint64_t pol) {
#pragma unroll
    for (int k = 0; k < 3; ++k)
        asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p + 4 * k),
                     "f"(v[4 * k]), "f"(v[4 * k + 1]), "f"(v[4 * k + 2]), "f"(v[4 * k + 3]), "l"(pol)
                     : "memory");
}
// invalidate one 128-byte L2 line without writing it back (its data is dead)
__device__ __forceinline__ void discard_l2(const void* p) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void st4_hint(float* p, float4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ float4 ldg4_hint(const float* p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol)
                 : "memory");
    return v;
}
__device__ __forceinline__ void cp_async16_cg_hint(void* sdst, const void* gsrc, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc),
                 "l"(pol)
                 : "memory");
}

// cp.async (LDGSTS): 4/8-byte copies through L1 (read-only program tables), 16-byte
// copies at L2 (.cg: data written earlier in the same kernel by other threads).
__device__ __forceinline__ void cp_async4(void* sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16_cg(void* sdst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
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

// Normalisation of the blended quaternion and of the weight sum.  HS_S1_NORM = 0:
// MUFU approximations (rsqrt.approx / rcp.approx, rel. error up to ~2^-22);
// 1: correctly rounded (__frsqrt_rn / __frcp_rn), the product build (DESIGN.md §3:
// Stage-1 error budget, measured per variant).
#ifndef HS_S1_NORM
#define HS_S1_NORM 1
#endif
__device__ __forceinline__ float rsqrt_fast(float x) {
#if HS_S1_NORM == 0
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
#else
    return __frsqrt_rn(x);
#endif
}
__device__ __forceinline__ float rcp_fast(float x) {
#if HS_S1_NORM == 0
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
#else
    return __frcp_rn(x);
#endif
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

// Every product and sum below is an explicit mul_rn / add_rn / fma_rn: the
// compiler's FMA contraction otherwise depends on the surrounding code (an unrolled
// layer loop contracts differently from a rolled one), and the fused and two-pass
// placements must produce the same local poses bit for bit.
// The Stage-1 arithmetic type s1r: fp32 (HS_S1_F64 = 0) or fp64 (1: sampling, blending
// and TRS in double, the 3x4 rounded once to fp32; DESIGN.md §3 Stage-1 budget).
#ifndef HS_S1_F64
#define HS_S1_F64 1
#endif
#if HS_S1_F64
typedef double s1r;
#else
typedef float s1r;
#endif
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float rsqrt_rn(float x) { return rsqrt_fast(x); }
__device__ __forceinline__ float rcp_rn(float x) { return rcp_fast(x); }
// fp64: the MUFU approximation (rel. error < 2^-21) refined by one Newton step in fp64
// (error ~2^-42, far below the final fp32 rounding) instead of the IEEE double sqrt /
// reciprocal sequences, which cost several times more issue slots
__device__ __forceinline__ double rsqrt_rn(double x) {
    float yf;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"((float)x));
    const double y = yf;
    return y * fma(-0.5 * x * y, y, 1.5);
}
__device__ __forceinline__ double rcp_rn(double x) {
    float yf;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"((float)x));
    const double y = yf;
    return y * fma(-x, y, 2.0);
}

__device__ __forceinline__ s1r lerp_rn(s1r b, s1r x0, s1r a, s1r x1) {
    return fma_rn(a, x1, mul_rn(b, x0));
}
__device__ __forceinline__ s1r dot4_rn(s1r a0, s1r a1, s1r a2, s1r a3, s1r b0, s1r b1, s1r b2, s1r b3) {
    return fma_rn(a3, b3, fma_rn(a2, b2, fma_rn(a1, b1, mul_rn(a0, b0))));
}

// Sample (keys x0..z0 at k0, x1..z1 at k0 + 1): trs = t(3), q(w,x,y,z)(4), s(3).
// NORM: normalise the interpolated quaternion (needed before a weighted blend of
// several layers); a single layer's quaternion goes to trs_to_m34 unnormalised, which
// divides by |q|^2 itself.
template <bool NORM>
__device__ __forceinline__ void sample_trs(float4 x0, float4 y0, float2 z0, float4 x1, float4 y1,
                                           float2 z1, float af, s1r* trs) {
    if (af == 0.0f) {   // on a key: that key exactly (R21)
        trs[0] = x0.x; trs[1] = x0.y; trs[2] = x0.z; trs[3] = x0.w;
        trs[4] = y0.x; trs[5] = y0.y; trs[6] = y0.z;
        trs[7] = y0.w; trs[8] = z0.x; trs[9] = z0.y;
        return;
    }
    const s1r a = af, b = sub_rn((s1r)1, a);
    trs[0] = lerp_rn(b, x0.x, a, x1.x); trs[1] = lerp_rn(b, x0.y, a, x1.y); trs[2] = lerp_rn(b, x0.z, a, x1.z);
    trs[7] = lerp_rn(b, y0.w, a, y1.w); trs[8] = lerp_rn(b, z0.x, a, z1.x); trs[9] = lerp_rn(b, z0.y, a, z1.y);
    const s1r d = dot4_rn(x0.w, y0.x, y0.y, y0.z, x1.w, y1.x, y1.y, y1.z);
    const s1r as = d < (s1r)0 ? -a : a;
    const s1r qw = lerp_rn(b, x0.w, as, x1.w), qx = lerp_rn(b, y0.x, as, y1.x),
              qy = lerp_rn(b, y0.y, as, y1.y), qz = lerp_rn(b, y0.z, as, y1.z);
    if (NORM) {
        const s1r inv = rsqrt_rn(dot4_rn(qw, qx, qy, qz, qw, qx, qy, qz));
        trs[3] = mul_rn(qw, inv); trs[4] = mul_rn(qx, inv); trs[5] = mul_rn(qy, inv);
        trs[6] = mul_rn(qz, inv);
    } else {
        trs[3] = qw; trs[4] = qx; trs[5] = qy; trs[6] = qz;
    }
}

// R(q) for ANY non-zero q: with c = 2 / |q|^2, R = [1 - c (y^2 + z^2), c (x y - w z), ...]
// equals the unit-quaternion formula of q / |q| (the oracle normalises in
// fp64 and uses the unit formula).  Dividing by |q|^2 here keeps R orthonormal to a few
// ulps however far |q| is from 1 after fp32 interpolation and blending; the unit
// formula on a quaternion of norm^2 = 1 + d gives R' = (1 + d) R + (-d) I, an O(d)
// non-rigid error that compounds down the root path (Stage-1 budget).
__device__ __forceinline__ void trs_to_m34(const s1r* trs, float* m) {
    const s1r w = trs[3], x = trs[4], y = trs[5], z = trs[6];
    const s1r sx = trs[7], sy = trs[8], sz = trs[9];
    const s1r c = mul_rn((s1r)2, rcp_rn(dot4_rn(w, x, y, z, w, x, y, z)));
    // 1 - c (u^2 + v^2) and c (u v -/+ w t), each rounded in one fixed order
    auto diag = [c](s1r u, s1r v) { return fma_rn(-c, fma_rn(u, u, mul_rn(v, v)), (s1r)1); };
    auto offd = [c](s1r u, s1r v, s1r p, s1r q, s1r sgn) {
        return mul_rn(c, fma_rn(sgn * p, q, mul_rn(u, v)));
    };
    m[0] = (float)mul_rn(diag(y, z), sx);                  m[1] = (float)mul_rn(offd(x, y, w, z, -1), sy);
    m[2] = (float)mul_rn(offd(x, z, w, y, 1), sz);         m[3] = (float)trs[0];
    m[4] = (float)mul_rn(offd(x, y, w, z, 1), sx);         m[5] = (float)mul_rn(diag(x, z), sy);
    m[6] = (float)mul_rn(offd(y, z, w, x, -1), sz);        m[7] = (float)trs[1];
    m[8] = (float)mul_rn(offd(x, z, w, y, -1), sx);        m[9] = (float)mul_rn(offd(y, z, w, x, 1), sy);
    m[10] = (float)mul_rn(diag(x, y), sz);                 m[11] = (float)trs[2];
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

// NLT > 0: the layer count is a compile-time constant (the layer loop unrolls, so
// every layer's key loads can be issued before the first layer's arithmetic).
template <int E, bool PIPE, int NLT = 0>
__device__ __forceinline__ void stage1_elems(const float* __restrict__ keys, const int4* const* dsc,
                                             const int* j, const bool* valid, int nl_rt, int Jp, float* L,
                                             const int* off) {
    const int nl = NLT > 0 ? NLT : nl_rt;
    s1r acc[E][10], q0[E][4], wsum[E];
    KeyPair kp[E];
    int4 d[E];
    constexpr int kPre = NLT > 0 ? NLT : 1;
    KeyPair pre[kPre][E];
    int4 pd[kPre][E];
    if (NLT > 0) {   // every layer's descriptors and keys in flight at once
#pragma unroll
        for (int l = 0; l < kPre; ++l)
#pragma unroll
            for (int e = 0; e < E; ++e) {
                pd[l][e] = valid[e] ? dsc[e][l] : make_int4(0, 0, 0, 0);
                pre[l][e] = load_keys(keys, pd[l][e], j[e], Jp);
            }
    } else if (PIPE) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            d[e] = valid[e] ? dsc[e][0] : make_int4(0, 0, 0, 0);
            kp[e] = load_keys(keys, d[e], j[e], Jp);
        }
    }
#pragma unroll(kPre)
    for (int l = 0; l < nl; ++l) {
        KeyPair cur[E];
        int4 dc[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (NLT > 0) {
                cur[e] = pre[l][e];
                dc[e] = pd[l][e];
            } else if (PIPE) {
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
            s1r s[10];
            if (nl == 1)
                sample_trs<false>(cur[e].x0, cur[e].y0, cur[e].z0, cur[e].x1, cur[e].y1, cur[e].z1,
                                  __int_as_float(dc[e].z), s);
            else
                sample_trs<true>(cur[e].x0, cur[e].y0, cur[e].z0, cur[e].x1, cur[e].y1, cur[e].z1,
                                 __int_as_float(dc[e].z), s);
            const s1r w = __int_as_float(dc[e].w);
            if (nl == 1) {   // one layer: the sample itself (R22)
#pragma unroll
                for (int c = 0; c < 10; ++c) acc[e][c] = s[c];
            } else if (l == 0) {
#pragma unroll
                for (int c = 0; c < 4; ++c) q0[e][c] = s[3 + c];
#pragma unroll
                for (int c = 0; c < 10; ++c) acc[e][c] = mul_rn(w, s[c]);
                wsum[e] = w;
            } else {
                const s1r dq = dot4_rn(s[3], s[4], s[5], s[6], q0[e][0], q0[e][1], q0[e][2], q0[e][3]);
                const s1r ws = dq < (s1r)0 ? -w : w;
#pragma unroll
                for (int c = 0; c < 3; ++c) acc[e][c] = fma_rn(w, s[c], acc[e][c]);
#pragma unroll
                for (int c = 3; c < 7; ++c) acc[e][c] = fma_rn(ws, s[c], acc[e][c]);
#pragma unroll
                for (int c = 7; c < 10; ++c) acc[e][c] = fma_rn(w, s[c], acc[e][c]);
                wsum[e] = add_rn(wsum[e], w);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (!valid[e]) continue;
        if (nl > 1) {
            const s1r iw = rcp_rn(wsum[e]);
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[e][c] = mul_rn(acc[e][c], iw);
#pragma unroll
            for (int c = 7; c < 10; ++c) acc[e][c] = mul_rn(acc[e][c], iw);
            // the blended quaternion is normalised by trs_to_m34 (c = 2 / |q|^2)
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

}  // namespace
}  // namespace hs
