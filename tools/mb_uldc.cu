// mb_uldc.cu -- do uniform constant loads (ULDC, uniform datapath) overlap
// with the shared-memory data pipe?  8 LDS per iteration, plus N warp-uniform
// __constant__ loads whose address depends only on the loop counter.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_uldc mb_uldc.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITER = 4096;
__constant__ uint2 cnodes[8192];

template <int NC>
__global__ void k(float *out, int salt) {
    __shared__ float s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5f;
    __syncthreads();
    float acc = 0;
    unsigned a = threadIdx.x & 31, u2 = 0;
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) acc += s[(a + u * 32 + it * 256 + salt) & 4095];
#pragma unroll
        for (int c = 0; c < NC; c++) {
            uint2 q = cnodes[(it * NC + c + salt) & 8191];
            u2 += q.x ^ q.y;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + u2;
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
    auto run = [&](const char *name, auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 5; r++) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-14s %7.3f ms\n", name, ms / 5);
    };
    run("lds8", [&] { k<0><<<blocks, threads>>>(out, 1); });
    run("lds8+uldc2", [&] { k<2><<<blocks, threads>>>(out, 1); });
    run("lds8+uldc4", [&] { k<4><<<blocks, threads>>>(out, 1); });
    run("lds8+uldc8", [&] { k<8><<<blocks, threads>>>(out, 1); });
    run("lds8+uldc16", [&] { k<16><<<blocks, threads>>>(out, 1); });
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
