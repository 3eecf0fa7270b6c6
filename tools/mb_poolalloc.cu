// Cost of stream-ordered pool allocations inside a CUDA graph of small
// kernels: N x [alloc, kernel, kernel, free] against N x [kernel, kernel]
// and N x [kernel] (device time per iteration, graph replays).
//   nvcc -arch=sm_100a -O3 -o /tmp/mb_poolalloc tools/mb_poolalloc.cu && /tmp/mb_poolalloc
#include <cuda_runtime.h>
#include <stdio.h>
__global__ void k_small(double *p, int n) {
    if (p && threadIdx.x < n) p[threadIdx.x] = 1.0;
}
static float run(int mode, int iters, cudaMemPool_t pool) {
    cudaStream_t st;
    cudaStreamCreate(&st);
    static double *fixed = nullptr;
    if (!fixed) cudaMalloc(&fixed, 1 << 20);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < iters; i++) {
        double *p = fixed;
        if (mode == 2) cudaMallocFromPoolAsync((void **)&p, 1 << 20, pool, st);
        k_small<<<56, 160, 0, st>>>(p, 32);
        if (mode >= 1) k_small<<<1, 256, 0, st>>>(p, 32);
        if (mode == 2) cudaFreeAsync(p, st);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; w++) cudaGraphLaunch(ge, st);
    cudaEventRecord(a, st);
    const int reps = 20;
    for (int r = 0; r < reps; r++) cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st);
    cudaStreamSynchronize(st);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1000.f / reps / iters;
}
int main() {
    cudaMemPool_t pool;
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = 0;
    cudaMemPoolCreate(&pool, &props);
    unsigned long long keep = 2048ull << 20;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    const char *names[] = {"1 kernel", "2 kernels", "alloc + 2 kernels + free"};
    for (int mode = 0; mode < 3; mode++)
        printf("%-28s %.2f us / iteration\n", names[mode], run(mode, 20, pool));
    return 0;
}
