// mb_ldg_gather.cu -- cost of a per-lane (divergent) global gather on the
// L1TEX data pipe, against the shared-memory gather the walk uses.  Deep
// trees (d >= 10) are capacity-bound in shared memory; reading their bottom
// levels from L1/L2 instead only pays if a 32-address LDG is cheap.
//   lds_rand   : LDS.32, each lane a random word of a 4 KB table
//   ldg_l1     : LDG.32, each lane a random word of a 16 KB table (L1 hits)
//   ldg_l2     : LDG.32, each lane a random word of a 64 MB table (L2 hits)
// 8 independent loads per iteration, addresses from a per-lane LCG;
// clk per warp-load per SM at 16 warps/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_ldg_gather mb_ldg_gather.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

template <int MODE>
__global__ void __launch_bounds__(512) probe(const float *__restrict__ g, uint32_t mask, float *out) {
    __shared__ float t[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) t[i] = (float)i;
    __syncthreads();
    uint32_t s[8];
#pragma unroll
    for (int k = 0; k < 8; k++) s[k] = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + k * 40503u;
    float acc = 0.f;
    const uint32_t tb = (uint32_t)__cvta_generic_to_shared(t);
    for (int it = 0; it < ITERS; it++) {
        float v[8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
            s[k] = s[k] * 1664525u + 1013904223u;
            const uint32_t idx = (s[k] >> 8) & mask;
            if (MODE == 0) {
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[k]) : "r"(tb + 4u * (idx & 1023u)));
            } else {
                v[k] = __ldg(g + idx);
            }
        }
#pragma unroll
        for (int k = 0; k < 8; k++) acc += v[k];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
void run(const char *name, const float *g, uint32_t mask, int sms, float *out) {
    const int grid = sms, block = 512;
    probe<MODE><<<grid, block>>>(g, mask, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) probe<MODE><<<grid, block>>>(g, mask, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double loads = 5.0 * grid * (block / 32) * (double)ITERS * 8;
    const double clk = ms * 1e-3 * 1965e6;
    printf("%-44s %8.3f ms  %7.2f clk per warp-load per SM  err=%s\n", name, ms / 5,
           clk / (loads / sms), cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *g, *out;
    const size_t n = 16u << 20;  // 64 MB
    cudaMalloc(&g, n * 4);
    cudaMemset(g, 0, n * 4);
    cudaMalloc(&out, sms * 512 * 4);
    run<0>("lds  32 random words of 4 KB", g, 1023u, sms, out);
    run<1>("ldg  32 random words of 4 KB (L1)", g, 1023u, sms, out);
    run<1>("ldg  32 random words of 16 KB (L1)", g, 4095u, sms, out);
    run<1>("ldg  32 random words of 256 KB (L1/L2)", g, 65535u, sms, out);
    run<1>("ldg  32 random words of 64 MB (L2)", g, (uint32_t)(n - 1), sms, out);
    return 0;
}
