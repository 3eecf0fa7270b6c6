// mb_pipes.cu -- which on-chip load paths share the L1TEX/shared-memory data
// pipe on B200?  Each kernel issues the same number of loads per thread; if
// "A+B" takes ~max(A,B) the paths are independent, if ~A+B they share.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_pipes mb_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 4096;
__constant__ float cbuf[4096];

__global__ void k_lds(float *out, int salt) {
    __shared__ float s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5f;
    __syncthreads();
    float acc = 0;
    unsigned a = threadIdx.x & 31;
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) acc += s[(a + u * 32 + it * 256 + salt) & 4095];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_ldg(const float *__restrict__ g, float *out, int salt) {
    float acc = 0;
    unsigned a = threadIdx.x & 31;
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) acc += __ldg(g + ((a + u * 32 + it * 256 + salt) & 4095));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_lds_ldg(const float *__restrict__ g, float *out, int salt) {
    __shared__ float s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5f;
    __syncthreads();
    float acc = 0, acc2 = 0;
    unsigned a = threadIdx.x & 31;
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
            acc += s[(a + u * 32 + it * 256 + salt) & 4095];
            acc2 += __ldg(g + ((a + u * 32 + it * 256 + salt + 7) & 4095));
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + acc2;
}

__global__ void k_tex(cudaTextureObject_t t, float *out, int salt) {
    float acc = 0;
    unsigned a = threadIdx.x & 31;
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) acc += tex1Dfetch<float>(t, (a + u * 32 + it * 256 + salt) & 4095);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_lds_tex(cudaTextureObject_t t, float *out, int salt) {
    __shared__ float s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5f;
    __syncthreads();
    float acc = 0, acc2 = 0;
    unsigned a = threadIdx.x & 31;
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
            acc += s[(a + u * 32 + it * 256 + salt) & 4095];
            acc2 += tex1Dfetch<float>(t, (a + u * 32 + it * 256 + salt + 7) & 4095);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + acc2;
}

// constant loads with D distinct addresses per warp
template <int DIV>
__global__ void k_ldc(float *out, int salt) {
    float acc = 0;
    unsigned a = threadIdx.x & (DIV - 1);
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) acc += cbuf[(a + u * 64 + it * 8 + salt) & 4095];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int DIV>
__global__ void k_lds_ldc(float *out, int salt) {
    __shared__ float s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5f;
    __syncthreads();
    float acc = 0, acc2 = 0;
    unsigned a = threadIdx.x & 31;
    unsigned b = threadIdx.x & (DIV - 1);
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
            acc += s[(a + u * 32 + it * 256 + salt) & 4095];
            acc2 += cbuf[(b + u * 64 + it * 8 + salt) & 4095];
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + acc2;
}

__global__ void k_shfl(float *out, int salt) {
    float v = threadIdx.x * 0.25f, acc = 0;
    unsigned a = threadIdx.x & 31;
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) acc += __shfl_sync(0xffffffffu, v + u, (a * 7 + u + it + salt) & 31);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_lds_shfl(float *out, int salt) {
    __shared__ float s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5f;
    __syncthreads();
    float v = threadIdx.x * 0.25f, acc = 0, acc2 = 0;
    unsigned a = threadIdx.x & 31;
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
            acc += s[(a + u * 32 + it * 256 + salt) & 4095];
            acc2 += __shfl_sync(0xffffffffu, v + u, (a * 7 + u + it + salt) & 31);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + acc2;
}

// 64-bit LDS with all lanes on distinct consecutive 8B (256B/warp)
__global__ void k_lds64(float *out, int salt) {
    __shared__ float2 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float2(i, i + 1);
    __syncthreads();
    float acc = 0;
    unsigned a = threadIdx.x & 31;
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
            float2 v = s[(a + u * 32 + it * 256 + salt) & 2047];
            acc += v.x + v.y;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int NT, typename TT>
__global__ void k_lds_texr(cudaTextureObject_t t, float *out, int salt) {
    __shared__ float s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5f;
    __syncthreads();
    float acc = 0, acc2 = 0;
    unsigned a = threadIdx.x & 31;
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) acc += s[(a + u * 32 + it * 256 + salt) & 4095];
#pragma unroll
        for (int u = 0; u < NT; u++) {
            TT v = tex1Dfetch<TT>(t, (a * 5 + u * 32 + it * 256 + salt + 7) & 2047);
            if constexpr (sizeof(TT) == 8) acc2 += v.x + v.y; else acc2 += v;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + acc2;
}

template <int NT>
__global__ void k_lds_ldgr(const float *__restrict__ g, float *out, int salt) {
    __shared__ float s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5f;
    __syncthreads();
    float acc = 0, acc2 = 0;
    unsigned a = threadIdx.x & 31;
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) acc += s[(a + u * 32 + it * 256 + salt) & 4095];
#pragma unroll
        for (int u = 0; u < NT; u++) acc2 += __ldg(g + ((a * 5 + u * 32 + it * 256 + salt + 7) & 2047));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + acc2;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float *g, *out;
    cudaMalloc(&g, 4096 * 4);
    cudaMemset(g, 0, 4096 * 4);
    const int blocks = sms * 4, threads = 256;
    cudaMalloc(&out, (size_t)blocks * threads * 4);
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = g;
    rd.res.linear.desc = cudaCreateChannelDesc<float>();
    rd.res.linear.sizeInBytes = 4096 * 4;
    cudaTextureDesc td{};
    cudaTextureObject_t tex;
    cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double warp_loads = (double)blocks * threads / 32 * ITER * 8;  // per load stream
    auto run = [&](const char *name, auto launch, double streams) {
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
        printf("%-14s %8.3f ms  %6.3f warp-loads/clk/SM (per stream %6.3f)\n", name, ms,
               warp_loads * streams / cycles / sms, warp_loads / cycles / sms);
    };
    run("lds", [&] { k_lds<<<blocks, threads>>>(out, 1); }, 1);
    run("lds64", [&] { k_lds64<<<blocks, threads>>>(out, 1); }, 1);
    run("ldg_l1", [&] { k_ldg<<<blocks, threads>>>(g, out, 1); }, 1);
    run("lds+ldg", [&] { k_lds_ldg<<<blocks, threads>>>(g, out, 1); }, 2);
    run("tex", [&] { k_tex<<<blocks, threads>>>(tex, out, 1); }, 1);
    run("lds+tex", [&] { k_lds_tex<<<blocks, threads>>>(tex, out, 1); }, 2);
    run("ldc_div1", [&] { k_ldc<1><<<blocks, threads>>>(out, 1); }, 1);
    run("ldc_div2", [&] { k_ldc<2><<<blocks, threads>>>(out, 1); }, 1);
    run("ldc_div4", [&] { k_ldc<4><<<blocks, threads>>>(out, 1); }, 1);
    run("lds+ldc1", [&] { k_lds_ldc<1><<<blocks, threads>>>(out, 1); }, 2);
    run("lds+ldc2", [&] { k_lds_ldc<2><<<blocks, threads>>>(out, 1); }, 2);
    run("lds+ldc4", [&] { k_lds_ldc<4><<<blocks, threads>>>(out, 1); }, 2);
    cudaResourceDesc rd2 = rd;
    rd2.res.linear.desc = cudaCreateChannelDesc<float2>();
    cudaTextureObject_t tex2;
    cudaCreateTextureObject(&tex2, &rd2, &td, nullptr);
    run("lds8+tex1", [&] { k_lds_texr<1, float><<<blocks, threads>>>(tex, out, 1); }, 1);
    run("lds8+tex2", [&] { k_lds_texr<2, float><<<blocks, threads>>>(tex, out, 1); }, 1);
    run("lds8+tex4", [&] { k_lds_texr<4, float><<<blocks, threads>>>(tex, out, 1); }, 1);
    run("lds8+tex2x64", [&] { k_lds_texr<2, float2><<<blocks, threads>>>(tex2, out, 1); }, 1);
    run("lds8+ldg1", [&] { k_lds_ldgr<1><<<blocks, threads>>>(g, out, 1); }, 1);
    run("lds8+ldg2", [&] { k_lds_ldgr<2><<<blocks, threads>>>(g, out, 1); }, 1);
    run("shfl", [&] { k_shfl<<<blocks, threads>>>(out, 1); }, 1);
    run("lds+shfl", [&] { k_lds_shfl<<<blocks, threads>>>(out, 1); }, 2);
    printf("clock %d kHz, %d SMs, err=%s\n", clk, sms, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
