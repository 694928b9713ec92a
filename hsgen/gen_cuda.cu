// hsgen/gen_cuda.cu — device twin of hsgen/gen.c (local-pose recipe only).
//
// TEST/BENCH INFRASTRUCTURE: fills the bench's full-size inputs (up to 21.5 GB
// of local poses for the 1M-character crowd) directly in HBM, so nothing that
// large crosses PCIe.  It implements the SAME counter-based recipe as gen.c
// (see that file's header); it contains none of the method's arithmetic.  The
// only known difference from the host generator is libm-vs-CUDA fp64 sin/cos/
// cbrt rounding (<= 2 ulp in fp64), which can flip the single fp32 rounding of
// a value that lands within ~1e-16 of an fp32 midpoint — measured and reported
// by tests/test_gen.py (gpu).  Parity tests take their inputs from gen.c.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t sm64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double ucounter(uint64_t key, uint64_t c, uint64_t J,
                                           uint64_t j, uint64_t k) {
    return (double)(sm64(((c * J + j) * 8 + k) ^ key) >> 11) * 0x1.0p-53;
}

__global__ void local_poses_kernel(uint64_t key_rot, uint64_t key_tr, uint64_t J,
                                   uint64_t char0, uint64_t n_chars, float* __restrict__ out) {
    const double kPi = 3.14159265358979323846;
    uint64_t total = n_chars * J;
    for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t c = char0 + idx / J, j = idx % J;
        double u0 = ucounter(key_rot, c, J, j, 0), u1 = ucounter(key_rot, c, J, j, 1),
               u2 = ucounter(key_rot, c, J, j, 2);
        double s1 = sqrt(1.0 - u0), s2 = sqrt(u0);
        double a1 = 2.0 * kPi * u1, a2 = 2.0 * kPi * u2;
        double x = s1 * sin(a1), y = s1 * cos(a1), z = s2 * sin(a2), w = s2 * cos(a2);
        double R[9];
        R[0] = 1.0 - 2.0 * (y * y + z * z); R[1] = 2.0 * (x * y - w * z); R[2] = 2.0 * (x * z + w * y);
        R[3] = 2.0 * (x * y + w * z); R[4] = 1.0 - 2.0 * (x * x + z * z); R[5] = 2.0 * (y * z - w * x);
        R[6] = 2.0 * (x * z - w * y); R[7] = 2.0 * (y * z + w * x); R[8] = 1.0 - 2.0 * (x * x + y * y);
        double v0 = ucounter(key_tr, c, J, j, 0), v1 = ucounter(key_tr, c, J, j, 1),
               v2 = ucounter(key_tr, c, J, j, 2);
        double zz = 2.0 * v0 - 1.0, phi = 2.0 * kPi * v1, r = cbrt(v2);
        double rho = sqrt(fmax(0.0, 1.0 - zz * zz));
        double t0 = r * rho * cos(phi), t1 = r * rho * sin(phi), t2 = r * zz;
        float4* o = reinterpret_cast<float4*>(out + idx * 12);
        o[0] = make_float4((float)R[0], (float)R[1], (float)R[2], (float)t0);
        o[1] = make_float4((float)R[3], (float)R[4], (float)R[5], (float)t1);
        o[2] = make_float4((float)R[6], (float)R[7], (float)R[8], (float)t2);
    }
}

uint64_t host_sm64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

}  // namespace

extern "C" int hsg_cuda_local_poses(uint64_t seed, uint64_t type, uint64_t J, uint64_t char0,
                                    uint64_t n_chars, float* d_out, void* stream) {
    if (n_chars == 0 || J == 0) return 0;
    uint64_t key_rot = host_sm64(seed * 16 + 8 * type + 0);
    uint64_t key_tr = host_sm64(seed * 16 + 8 * type + 1);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    local_poses_kernel<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(key_rot, key_tr, J, char0,
                                                                   n_chars, d_out);
    return (int)cudaGetLastError();
}
