// ts_synth.cu -- counter-based synthetic instances generated in place on the
// GPU (BASELINE configs 3 and 4 need 5.6-34.8 GB of rows; generating them on
// the host and copying would dominate the run).  Bit-identical to
// paper_1212_2287_b200.synth.hash_uniform on the host, so any sampled row can
// be re-created for oracle checks.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ts_internal.h"

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_synth_uniform(float *x, long long n, long long f, long long ld,
                                unsigned long long seed, long long row0, uint32_t zero_thresh) {
    const long long total = n * f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / f, c = i - r * f;
        const uint64_t e = (uint64_t)(row0 + r) * (uint64_t)f + (uint64_t)c + 1ull;
        float v = (float)(uint32_t)(mix64(seed + e * 0x9E3779B97F4A7C15ull) >> 40) *
                  5.9604644775390625e-08f;  // 2^-24
        if (zero_thresh &&
            (uint32_t)(mix64((seed ^ 0xD1B54A32D192ED03ull) + e * 0x9E3779B97F4A7C15ull) >> 40) <
                zero_thresh)
            v = 0.0f;
        x[r * ld + c] = v;
    }
}

}  // namespace

extern "C" int ts_synth_uniform(float *x, int64_t n, int64_t f, int64_t ld, uint64_t seed,
                                int64_t row0, double zero_prob, void *stream) {
    if (n < 0 || f < 1 || ld < f) return ts::fail(TS_ERR_SHAPE, "bad synth shape");
    if (n == 0) return TS_OK;
    const uint32_t thresh = zero_prob > 0 ? (uint32_t)(zero_prob * (double)(1u << 24)) : 0u;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    k_synth_uniform<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(x, n, f, ld, seed, row0, thresh);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TS_OK : ts::cuda_fail(e, "ts_synth_uniform launch");
}
