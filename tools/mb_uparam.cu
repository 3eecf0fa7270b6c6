// mb_uparam.cu -- can the top two heap levels of each tree come from the
// kernel's parameter bank (uniform datapath: ULDC into uniform registers, no
// shared-memory wavefront) instead of shared memory?
//
// Walk as tools/mb_walk_sol.cu (K = 8 chains, 8 levels, x tile xs[f * B + r],
// 2 CTAs x 128 threads per SM), node records:
//   mode 0 "smem":  level 0 a broadcast 8-byte record (1 wavefront), levels
//                   1..7 distinct 8-byte records (2 wavefronts) -- the
//                   k_stream pattern;
//   mode 1 "param": levels 0-1 from a per-launch table in the kernel
//                   parameters (three records per tree, uniform loads, level 1
//                   picked with SELs), levels 2..7 as mode 0.
// Reports node visits per clock per SM (SURVEY 8(d) issue roofline: 32).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_uparam mb_uparam.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int B = 128, K = 8, LEVELS = 8, TREES = 1024, F = 136;

struct Top {
    uint2 rec[3 * TREES];  // {x byte offset, theta} of heap nodes 0, 1, 2 per tree
};

template <int MODE>
__global__ void __launch_bounds__(B, 2) walk(float *out, int salt, const __grid_constant__ Top top) {
    extern __shared__ float sm[];
    float *xs = sm;                                         // F x B
    uint2 *nodes = reinterpret_cast<uint2 *>(sm + F * B);  // 256 records
    for (int i = threadIdx.x; i < F * B; i += B) xs[i] = (float)((i * 37 + salt) % 1000) * 1e-3f;
    for (int i = threadIdx.x; i < 256; i += B)
        nodes[i] = make_uint2((uint32_t)(((i * 13) % F) * B * 4), 0x3f000000u);
    __syncthreads();
    const uint32_t xr = (uint32_t)__cvta_generic_to_shared(xs) + 4u * threadIdx.x;
    const uint32_t nb = (uint32_t)__cvta_generic_to_shared(nodes);
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    for (int rep = 0; rep < 2; rep++) {
        for (int t = 0; t < TREES; t += K) {
            uint32_t j[K];
            int l0 = 0;
            if (MODE == 1) {
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const uint2 r0 = top.rec[3 * (t + k)];
                    float v;
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(r0.x + xr));
                    const bool c0 = v >= __uint_as_float(r0.y);
                    uint2 a1 = top.rec[3 * (t + k) + 1], a2 = top.rec[3 * (t + k) + 2];
                    // both records loaded (uniform), then picked per lane
                    asm("" : "+r"(a1.x), "+r"(a1.y), "+r"(a2.x), "+r"(a2.y));
                    const uint2 r1 = c0 ? a2 : a1;
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(r1.x + xr));
                    const bool c1 = v >= __uint_as_float(r1.y);
                    j[k] = 3u + (c0 ? 2u : 0u) + (c1 ? 1u : 0u);
                }
                l0 = 2;
            } else if (MODE == 3) {
                // levels 0-1 from the parameter bank, chains in two halves so
                // at most 4 chains' records are live in uniform registers
#pragma unroll
                for (int h = 0; h < 2; h++) {
#pragma unroll
                    for (int k = h * (K / 2); k < (h + 1) * (K / 2); k++) {
                        const uint2 r0 = top.rec[3 * (t + k)];
                        float v;
                        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(r0.x + xr));
                        const bool c0 = v >= __uint_as_float(r0.y);
                        const uint2 a1 = top.rec[3 * (t + k) + 1], a2 = top.rec[3 * (t + k) + 2];
                        const uint32_t fx = c0 ? a2.x : a1.x, th = c0 ? a2.y : a1.y;
                        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(fx + xr));
                        const bool c1 = v >= __uint_as_float(th);
                        j[k] = 3u + (c0 ? 2u : 0u) + (c1 ? 1u : 0u);
                    }
                    asm volatile("" ::: "memory");
                }
                l0 = 2;
            } else if (MODE == 2) {
                // level 0 only from the parameter bank (one record per chain
                // live in uniform registers), levels 1..7 from shared memory
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const uint2 r0 = top.rec[3 * (t + k)];
                    float v;
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(r0.x + xr));
                    j[k] = v >= __uint_as_float(r0.y) ? 2u : 1u;
                }
                l0 = 1;
            } else {
#pragma unroll
                for (int k = 0; k < K; k++) j[k] = 0;
            }
#pragma unroll
            for (int l = l0; l < LEVELS; l++) {
#pragma unroll
                for (int k = 0; k < K; k++) {
                    uint32_t a;
                    if (l == 0) a = nb + 8u * ((t + k) & 31u);                   // broadcast
                    else a = nb + 8u * ((j[k] + lane + (uint32_t)t) & 31u);       // distinct
                    uint2 q;
                    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(q.x), "=r"(q.y) : "r"(a));
                    float v;
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(q.x + xr));
                    j[k] = 2u * j[k] + (v >= __uint_as_float(q.y) ? 2u : 1u);
                }
            }
#pragma unroll
            for (int k = 0; k < K; k++) acc += (double)(j[k] & 7u);
        }
    }
    out[blockIdx.x * B + threadIdx.x] = (float)acc;
}

template <int MODE>
void run(const char *name, int sms, int mhz, const Top &top) {
    constexpr int CTAS = 2;
    const int grid = sms * CTAS;
    const size_t smem = F * B * 4 + 256 * 8;
    float *out;
    cudaMalloc(&out, grid * B * sizeof(float));
    cudaFuncSetAttribute(walk<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    walk<MODE><<<grid, B, smem>>>(out, 1, top);
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    cudaEventRecord(s);
    for (int r = 0; r < 5; r++) walk<MODE><<<grid, B, smem>>>(out, r, top);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms;
    cudaEventElapsedTime(&ms, s, e);
    const double visits = 5.0 * grid * B * 2.0 * TREES * LEVELS;
    const double per_clk_sm = visits / (ms * 1e-3) / sms / (mhz * 1e6);
    printf("%-8s %8.3f ms  %6.2f visits/clk/SM  (%.1f %% of 32/clk)  err=%s\n", name, ms / 5,
           per_clk_sm, 100.0 * per_clk_sm / 32.0, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int mhz = 1965;
    static Top top;
    for (int i = 0; i < 3 * TREES; i++)
        top.rec[i] = make_uint2((uint32_t)(((i * 29) % F) * B * 4), 0x3f000000u);
    run<0>("smem", sms, mhz, top);
    run<1>("param", sms, mhz, top);
    run<2>("param-l0", sms, mhz, top);
    run<3>("param-h", sms, mhz, top);
    run<0>("smem", sms, mhz, top);
    run<1>("param", sms, mhz, top);
    run<2>("param-l0", sms, mhz, top);
    run<3>("param-h", sms, mhz, top);
    return 0;
}
