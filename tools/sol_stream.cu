// sol_stream.cu — measurement probe (not part of the library): the HBM speed of light
// of the hot path's traffic pattern with no arithmetic.  The scan + bind reads 48 B and
// writes 2 x 48 B per joint (L in; G and S out); these kernels move exactly that mix
// (and, for reference, a plain 1:1 copy) so the chunked kernel's roofline fraction can
// be read against what the memory system sustains for the same read:write ratio.
//
//   sol_tma   persistent CTAs, one per SM; one thread streams tiles HBM -> smem by TMA
//             bulk copies (4 KB pieces, mbarrier completion, `stages` deep) and writes
//             each tile back `n_out` times by TMA bulk stores — the chunked kernel's
//             producer warp without its consumers.
//   sol_simt  grid-stride float4 loads / stores (n_out stores per load).
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC
//        tools/sol_stream.cu -o build/libsol.so   (tools/sol_stream.py does it)
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(su32(b)), "r"(parity)
            : "memory");
}
__device__ __forceinline__ void g2s(void* s, const void* g, uint32_t bytes, uint64_t* b, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            su32(s)),
        "l"(g), "r"(bytes), "r"(su32(b)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void s2g(void* g, const void* s, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(g),
                 "r"(su32(s)), "r"(bytes), "l"(pol)
                 : "memory");
}

__global__ void __launch_bounds__(32, 1) sol_tma(const char* in, char* out0, char* out1, int64_t n_tiles,
                                                  int tile_bytes, int stages, int n_out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);
    unsigned char* buf = sm + 128;
    if (threadIdx.x != 0) return;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int s = 0; s < stages; ++s) mb_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int64_t my = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto tile_of = [&](int64_t i) { return (int64_t)blockIdx.x + i * gridDim.x; };
    auto load = [&](int64_t i, int s) {
        const char* src = in + tile_of(i) * tile_bytes;
        unsigned char* dst = buf + (size_t)s * tile_bytes;
        mb_expect(&full[s], (uint32_t)tile_bytes);
        for (int o = 0; o < tile_bytes; o += 4096) g2s(dst + o, src + o, min(4096, tile_bytes - o), &full[s], pol);
    };
    for (int64_t i = 0; i < my && i < stages; ++i) load(i, (int)i);
    uint32_t phase = 0;
    int s = 0;
    for (int64_t i = 0; i < my; ++i) {
        mb_wait(&full[s], phase);
        const unsigned char* src = buf + (size_t)s * tile_bytes;
        for (int r = 0; r < n_out; ++r) {
            char* dst = (r ? out1 : out0) + tile_of(i) * tile_bytes;
            for (int o = 0; o < tile_bytes; o += 4096) s2g(dst + o, src + o, min(4096, tile_bytes - o), pol);
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // stage s read out
        if (i + stages < my) load(i + stages, s);
        if (++s == stages) { s = 0; phase ^= 1u; }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void sol_simt(const float4* __restrict__ in, float4* __restrict__ out0, float4* __restrict__ out1,
                         int64_t n, int n_out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const float4 v = __ldcs(in + i);
        __stcs(out0 + i, v);
        if (n_out > 1) __stcs(out1 + i, v);
    }
}

}  // namespace

extern "C" int sol_tma_launch(const void* in, void* out0, void* out1, int64_t n_tiles, int tile_bytes, int stages,
                              int n_out, void* stream) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = 128 + (size_t)stages * tile_bytes;
    if (cudaFuncSetAttribute(sol_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 1;
    sol_tma<<<sms, 32, smem, (cudaStream_t)stream>>>((const char*)in, (char*)out0, (char*)out1, n_tiles, tile_bytes,
                                                    stages, n_out);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

extern "C" int sol_simt_launch(const void* in, void* out0, void* out1, int64_t n_float4, int blocks_per_sm,
                               int n_out, void* stream) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    sol_simt<<<sms * blocks_per_sm, 512, 0, (cudaStream_t)stream>>>((const float4*)in, (float4*)out0, (float4*)out1,
                                                                   n_float4, n_out);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
