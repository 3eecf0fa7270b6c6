// mb_lds.cu -- shared-memory wavefront cost of the access patterns the
// traversal issues (broadcast / few-distinct / conflict-free 64- and 128-bit).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_lds mb_lds.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITER = 4096;

// MODE: lane -> element index pattern (in units of the access width)
template <typename T, int DISTINCT>
__global__ void k(float *out, int salt) {
    __shared__ __align__(16) float s[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i * 0.5f;
    __syncthreads();
    const T *st = reinterpret_cast<const T *>(s);
    constexpr int N = 8192 * 4 / sizeof(T);
    float acc = 0;
    unsigned lane = threadIdx.x & 31;
    unsigned a = DISTINCT == 0 ? lane * 37 : (lane % DISTINCT);  // 0 => random-ish
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
            T v = st[(a + u * 64 + it * 512 + salt) & (N - 1)];
            if constexpr (sizeof(T) == 4) acc += v;
            else if constexpr (sizeof(T) == 8) acc += v.x + v.y;
            else acc += v.x + v.y + v.z + v.w;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 4, threads = 256;
    float *out;
    cudaMalloc(&out, (size_t)blocks * threads * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double warp_loads = (double)blocks * threads / 32 * ITER * 8;
    auto run = [&](const char *name, auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 5; r++) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 5;
        double cycles = ms * 1e-3 * clk * 1e3;
        printf("%-22s %7.3f ms  %6.3f clk per warp-load per SM\n", name, ms,
               cycles * sms / warp_loads);
    };
    run("f32 broadcast", [&] { k<float, 1><<<blocks, threads>>>(out, 1); });
    run("f32 32 distinct", [&] { k<float, 32><<<blocks, threads>>>(out, 1); });
    run("f64 broadcast", [&] { k<float2, 1><<<blocks, threads>>>(out, 1); });
    run("f64 2 distinct", [&] { k<float2, 2><<<blocks, threads>>>(out, 1); });
    run("f64 8 distinct", [&] { k<float2, 8><<<blocks, threads>>>(out, 1); });
    run("f64 16 distinct", [&] { k<float2, 16><<<blocks, threads>>>(out, 1); });
    run("f64 32 distinct", [&] { k<float2, 32><<<blocks, threads>>>(out, 1); });
    run("f128 broadcast", [&] { k<float4, 1><<<blocks, threads>>>(out, 1); });
    run("f128 8 distinct", [&] { k<float4, 8><<<blocks, threads>>>(out, 1); });
    run("f128 32 distinct", [&] { k<float4, 32><<<blocks, threads>>>(out, 1); });
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
