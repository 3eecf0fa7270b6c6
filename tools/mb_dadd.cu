// Dependent-chain latency of the f64 add (DADD), f32->f64 convert (F2F) and
// shared load, one warp, clock64 (tools/mb_dadd.cu; nvcc -arch=sm_100a).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double *out, const float *in, long long *cyc, int iters) {
    __shared__ float sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = in[i];
    __syncthreads();
    double acc = out[threadIdx.x];
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) acc = __dadd_rn(acc, 1.0000001);
    long long t1 = clock64();
    float f = in[threadIdx.x];
    for (int i = 0; i < iters; i++) { double d = (double)f; f = (float)(d * 0.5); }
    long long t2 = clock64();
    unsigned idx = threadIdx.x;
    for (int i = 0; i < iters; i++) idx = __float_as_uint(sm[idx & 1023]) & 1023;
    long long t3 = clock64();
    out[threadIdx.x] = acc + f + idx;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}

int main() {
    double *out; float *in; long long *cyc;
    cudaMalloc(&out, 1024 * 8); cudaMalloc(&in, 1024 * 4); cudaMalloc(&cyc, 64);
    cudaMemset(out, 0, 1024 * 8); cudaMemset(in, 0, 1024 * 4);
    const int iters = 100000;
    k<<<1, 32>>>(out, in, cyc, iters);
    long long h[3];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    printf("DADD chain: %.1f clk/op\nF2F.F64+DMUL+F2F.F32 chain: %.1f clk/iter\nLDS chain: %.1f clk/op\n",
           (double)h[0] / iters, (double)h[1] / iters, (double)h[2] / iters);
    return 0;
}
