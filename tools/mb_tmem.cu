// mb_tmem.cu -- is tensor memory a second on-chip path for the walk's x reads?
// The shared-memory walk is bound by the L1TEX/shared data pipe (~1
// wavefront/clk/SM, profiles/r1_microbench_smem_pipes.txt).  A warp-uniform
// column read of TMEM (tcgen05.ld.32x32b.x1: lane r gets column c of TMEM
// lane r) is exactly x[fid] for the 32 rows when the fid is uniform -- which
// it is at a tree's root.  This probe measures
//   lds     : 8 conflict-free LDS.32 per iteration (the x read of a walk)
//   ldtm    : 8 tcgen05.ld.32x32b.x1 (uniform column) + one wait::ld
//   ldtm4   : 8 tcgen05.ld.32x32b.x4
//   lds+ldtm: both, interleaved (do the times add, or overlap?)
// per warp-op clocks per SM at 2 CTAs x 4 warps and 1 CTA x 16 warps.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_tmem mb_tmem.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ uint32_t ldtm1(uint32_t a) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(a) : "memory");
    return r;
}
__device__ __forceinline__ void ldtm4(uint32_t a, uint32_t &r0, uint32_t &r1, uint32_t &r2,
                                      uint32_t &r3) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(a)
                 : "memory");
}
__device__ __forceinline__ void tm_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int MODE, int WARPS, int F>
__global__ void __launch_bounds__(WARPS * 32) probe(float *out, int salt) {
    extern __shared__ float xs[];  // 136 x (32 * WARPS)
    __shared__ uint32_t tbase;
    constexpr int B = WARPS * 32;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < F * B; i += B) xs[i] = (float)((i * 37 + salt) % 1000) * 1e-3f;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
    // each lane writes its row's 136 features (8 columns per store)
    for (int c = 0; c + 8 <= F; c += 8) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = __float_as_uint(xs[(c + k) * B + threadIdx.x]);
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
                tm + c),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
            "r"(v[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    __syncthreads();
    const uint32_t xr = (uint32_t)__cvta_generic_to_shared(xs) + 4u * threadIdx.x;
    float acc[8];
    uint32_t la[8], ta[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        acc[k] = 0.f;
        la[k] = xr + 4u * B * (((uint32_t)salt + 17u * k) % F);
        ta[k] = tm + (((uint32_t)salt + 17u * k) % F);
    }
    for (int it = 0; it < ITERS; it++) {
        float v[8];
        if (MODE == 0 || MODE == 3) {
#pragma unroll
            for (int k = 0; k < 8; k++) {
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[k]) : "r"(la[k]) : "memory");
                la[k] ^= __float_as_uint(v[k]) & 4u;
            }
        }
        if (MODE == 1 || MODE == 3) {
            uint32_t r[8];
#pragma unroll
            for (int k = 0; k < 8; k++) r[k] = ldtm1(ta[k] + (uint32_t)(it & 1));
            tm_wait();
#pragma unroll
            for (int k = 0; k < 8; k++) {
                if (MODE == 3) v[k] += __uint_as_float(r[k]);
                else v[k] = __uint_as_float(r[k]);
            }
        }
        if (MODE == 2) {
#pragma unroll
            for (int k = 0; k < 8; k += 2) {
                uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
                ldtm4((ta[k] & ~3u) + 4u * (uint32_t)(it & 1), a0, a1, a2, a3);
                ldtm4((ta[k + 1] & ~3u) + 4u * (uint32_t)(it & 1), b0, b1, b2, b3);
                tm_wait();
                v[k] = __uint_as_float(a0) + __uint_as_float(a1) + __uint_as_float(a2) +
                       __uint_as_float(a3);
                v[k + 1] = __uint_as_float(b0) + __uint_as_float(b1) + __uint_as_float(b2) +
                           __uint_as_float(b3);
            }
        }
#pragma unroll
        for (int k = 0; k < 8; k++) acc[k] += v[k];
    }
    float accs = 0.f;
#pragma unroll
    for (int k = 0; k < 8; k++) accs += acc[k];
    out[blockIdx.x * B + threadIdx.x] = accs;
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

template <int MODE, int WARPS, int F = 136>
void run(const char *name, int sms, int ctas_per_sm, int mhz) {
    const int grid = sms * ctas_per_sm;
    const size_t smem = F * 32 * WARPS * 4;
    float *out;
    cudaMalloc(&out, grid * WARPS * 32 * sizeof(float));
    cudaFuncSetAttribute(probe<MODE, WARPS, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<MODE, WARPS, F><<<grid, WARPS * 32, smem>>>(out, 1);
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    cudaEventRecord(s);
    for (int r = 0; r < 5; r++) probe<MODE, WARPS, F><<<grid, WARPS * 32, smem>>>(out, r);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms;
    cudaEventElapsedTime(&ms, s, e);
    const double warp_ops = 5.0 * grid * WARPS * (double)ITERS * 8;  // per op kind
    const double clk = ms * 1e-3 * mhz * 1e6;
    printf("%-34s %8.3f ms  %6.3f clk per warp-op (of each kind) per SM   err=%s\n", name, ms / 5,
           clk / (warp_ops / sms), cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int mhz = 1965;
    printf("%d SMs, clock %d MHz\n", sms, mhz);
    run<0, 4>("lds        2 CTAs x 4 warps", sms, 2, mhz);
    run<1, 4>("ldtm.x1    2 CTAs x 4 warps", sms, 2, mhz);
    run<2, 4>("ldtm.x4    2 CTAs x 4 warps", sms, 2, mhz);
    run<3, 4>("lds+ldtm   2 CTAs x 4 warps", sms, 2, mhz);
    run<0, 8>("lds        1 CTA x 8 warps", sms, 1, mhz);
    run<1, 8>("ldtm.x1    1 CTA x 8 warps", sms, 1, mhz);
    run<3, 8>("lds+ldtm   1 CTA x 8 warps", sms, 1, mhz);
    run<0, 16, 48>("lds        1 CTA x 16 warps", sms, 1, mhz);
    run<1, 16, 48>("ldtm.x1    1 CTA x 16 warps", sms, 1, mhz);
    run<2, 16, 48>("ldtm.x4    1 CTA x 16 warps", sms, 1, mhz);
    run<3, 16, 48>("lds+ldtm   1 CTA x 16 warps", sms, 1, mhz);
    return 0;
}
