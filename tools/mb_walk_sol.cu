// mb_walk_sol.cu -- speed-of-light probe for a shared-memory predicated walk.
// Each visit does the two dependent shared loads every table walk needs (a
// node record, then x[fid] for the thread's own row) plus compare and index
// update, with the node loads made as cheap as the hardware allows:
//   mode 0 "ideal": every lane reads the SAME 8-byte record (broadcast, 1
//           wavefront) -- no real walk can do better;
//   mode 1 "4-byte": lanes read distinct 4-byte records within 128 bytes
//           (1 wavefront, conflict-free);
//   mode 2 "8-byte": lanes read distinct 8-byte records within 256 bytes
//           (2 wavefronts, the half-warp rule).
// x reads are conflict-free (xs[f * B + r]), K = 8 independent chains per
// thread, 2 CTAs x 160 threads per SM like k_stream.  Reports node visits per
// clock per SM against the SURVEY 8(d) issue roofline of 32.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_walk_sol mb_walk_sol.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int B = 128, K = 8, LEVELS = 8, TREES = 2048;

template <int MODE, int F, int CTAS>
__global__ void __launch_bounds__(B, CTAS) walk(float *out, int salt) {
    extern __shared__ float sm[];
    float *xs = sm;                                   // F x B
    uint2 *nodes = reinterpret_cast<uint2 *>(sm + F * B);  // 256 records
    for (int i = threadIdx.x; i < F * B; i += B) xs[i] = (float)((i * 37 + salt) % 1000) * 1e-3f;
    for (int i = threadIdx.x; i < 256; i += B)
        nodes[i] = make_uint2((uint32_t)(((i * 13) % F) * B * 4), __float_as_uint(0.5f));
    __syncthreads();
    const uint32_t xr = (uint32_t)__cvta_generic_to_shared(xs) + 4u * threadIdx.x;
    const uint32_t nb = (uint32_t)__cvta_generic_to_shared(nodes);
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    for (int t = 0; t < TREES; t += K) {
        uint32_t j[K];
#pragma unroll
        for (int k = 0; k < K; k++) j[k] = (uint32_t)(t + k) & 15u;
#pragma unroll
        for (int l = 0; l < LEVELS; l++) {
#pragma unroll
            for (int k = 0; k < K; k++) {
                uint32_t a;
                if (MODE == 0) a = nb + 8u * (j[k] & 31u);                  // same for all lanes
                else if (MODE == 1) a = nb + 4u * ((j[k] + lane) & 31u);    // 32 distinct words
                else a = nb + 8u * ((j[k] + lane) & 31u);                   // 32 distinct records
                uint2 q;
                if (MODE == 1) {
                    uint32_t w;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(a));
                    q = make_uint2(w & 0xffff00u, 0x3f000000u);
                } else {
                    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(q.x), "=r"(q.y) : "r"(a));
                }
                float v;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(q.x + xr));
                j[k] = 2u * j[k] + (v >= __uint_as_float(q.y) ? 2u : 1u);
            }
        }
#pragma unroll
        for (int k = 0; k < K; k++) acc += (double)(j[k] & 7u);
    }
    out[blockIdx.x * B + threadIdx.x] = (float)acc;
}

template <int MODE, int F, int CTAS>
void run(const char *name, int sms, int mhz) {
    const int grid = sms * CTAS;
    const size_t smem = F * B * 4 + 256 * 8;
    float *out;
    cudaMalloc(&out, grid * B * sizeof(float));
    cudaFuncSetAttribute(walk<MODE, F, CTAS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    walk<MODE, F, CTAS><<<grid, B, smem>>>(out, 1);
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    cudaEventRecord(s);
    for (int r = 0; r < 5; r++) walk<MODE, F, CTAS><<<grid, B, smem>>>(out, r);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms;
    cudaEventElapsedTime(&ms, s, e);
    const double visits = 5.0 * grid * B * (double)TREES * LEVELS;
    const double per_clk_sm = visits / (ms * 1e-3) / sms / (mhz * 1e6);
    printf("%-28s %8.3f ms  %6.2f visits/clk/SM  (%.1f %% of the 32/clk issue roofline)  err=%s\n",
           name, ms / 5, per_clk_sm, 100.0 * per_clk_sm / 32.0,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    int sms, khz;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const int mhz = 1965;  // MEASURED_PEAKS sm_max_mhz (the roofline's clock)
    printf("%d SMs, reported clock %d MHz, roofline clock %d MHz\n", sms, khz / 1000, mhz);
    run<0, 136, 2>("ideal    F=136 8 warps/SM", sms, mhz);
    run<1, 136, 2>("4-byte   F=136 8 warps/SM", sms, mhz);
    run<2, 136, 2>("8-byte   F=136 8 warps/SM", sms, mhz);
    run<0, 64, 4>("ideal    F=64 16 warps/SM", sms, mhz);
    run<0, 32, 8>("ideal    F=32 32 warps/SM", sms, mhz);
    return 0;
}
