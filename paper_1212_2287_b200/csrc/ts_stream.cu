// ts_stream.cu -- the main sm_100a traversal kernel: complete trees whose
// node tables are STREAMED through shared memory by the TMA bulk-copy engine.
//
// Per CTA (one per SM, persistent over instance tiles):
//   * 8 consumer warps own a tile of B = 256 instances, staged from HBM and
//     transposed to xs[f * B + r] (feature-major: lane r's x[fid] reads are
//     bank-conflict-free for any mix of fids);
//   * 1 producer warp streams the segment's packed trees, chunk by chunk, into
//     an S-stage shared-memory ring with cp.async.bulk (TMA, UBLKCP in SASS);
//     full/empty mbarriers hand stages between producer and consumers, so the
//     next chunk (and the next tile's first chunks) land while the current
//     one is walked;
//   * each consumer thread walks K trees of the chunk at once (K independent
//     index chains for latency hiding): per level
//         rec = node[j] (LDS.64 {fid, theta});  v = xs[fid*B + r] (LDS);
//         j = 2j + 1 + (v >= theta)
//     -- the reference's update i = (i<<1)+1+(x[fid[i]] >= theta[i])
//     (ref evaluators.py:90-99) -- then adds w*leaf in f64, tree order
//     (ref evaluators.py:529-535; __dmul_rn/__dadd_rn, never an FMA).
//
// Chunk = `tpc` consecutive trees of one complete segment (all of depth D,
// so every tree record has the same size and chunk c starts at
// c * tpc * tree_bytes).  Tree record: (2^D - 1) uint2 {fid, theta bits} in
// heap order, then 2^D fp32 leaves, padded to 16 bytes.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "ts_internal.h"

namespace ts {
namespace {

constexpr int kConsumerWarps = 8;
constexpr int kB = kConsumerWarps * 32;  // instances per tile
constexpr int kThreads = kB + 32;        // + producer warp
constexpr int kStages = 2;

__device__ __forceinline__ uint32_t su32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kB) : "memory");
}
__device__ __forceinline__ bool finite_f(float v) { return fabsf(v) <= 3.402823466e38f; }

// Transposing stage of B rows into xs[f * kB + r] (consumer threads only).
__device__ __forceinline__ void stage_rows(const StreamArgs &a, float *xs, long long row0) {
    const int r = threadIdx.x;
    const long long row = row0 + r;
    const bool valid = row < a.n;
    const float *xrow = a.x + (valid ? row : 0) * a.ld;
    const int F = a.F;
    bool bad = false;
    if (((F & 3) == 0) && ((a.ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0)) {
        const float4 *x4 = reinterpret_cast<const float4 *>(xrow);
        int c = 0;
        for (; c + 16 <= F; c += 16) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; u++)
                v[u] = valid ? __ldg(x4 + (c >> 2) + u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < 4; u++) {
                bad |= !(finite_f(v[u].x) && finite_f(v[u].y) && finite_f(v[u].z) &&
                         finite_f(v[u].w));
                float *dst = xs + (c + 4 * u) * kB + r;
                dst[0] = v[u].x;
                dst[kB] = v[u].y;
                dst[2 * kB] = v[u].z;
                dst[3 * kB] = v[u].w;
            }
        }
        for (; c < F; c += 4) {
            float4 v = valid ? __ldg(x4 + (c >> 2)) : make_float4(0.f, 0.f, 0.f, 0.f);
            bad |= !(finite_f(v.x) && finite_f(v.y) && finite_f(v.z) && finite_f(v.w));
            float *dst = xs + c * kB + r;
            dst[0] = v.x;
            dst[kB] = v.y;
            dst[2 * kB] = v.z;
            dst[3 * kB] = v.w;
        }
    } else {
        for (int c = 0; c < F; c++) {
            float v = valid ? __ldg(xrow + c) : 0.f;
            bad |= !finite_f(v);
            xs[c * kB + r] = v;
        }
    }
    if (bad && a.status) atomicOr(a.status, 1);
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ float ldsf(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

// Walk NK trees of one chunk in lockstep (NK independent chains).
// Node records hold fid pre-scaled to the byte offset of its x-tile row
// (fid * kB * 4), so the x address is one add.  The chain state is the
// absolute shared address `p` of the current record; the heap step
// j -> 2j + 1 + c becomes p -> 2p + (c ? 16 - base : 8 - base).
template <int D, int NK>
__device__ __forceinline__ void walk_group(uint32_t tree0, uint32_t tree_bytes, uint32_t xr,
                                           double &acc, const StreamArgs &a, int t,
                                           long long row, bool valid) {
    constexpr uint32_t kInt = (1u << D) - 1u;
    uint32_t p[NK], s0[NK], s1[NK];
#pragma unroll
    for (int k = 0; k < NK; k++) {
        const uint32_t base = tree0 + k * tree_bytes;
        p[k] = base;
        s0[k] = 8u - base;
        s1[k] = 16u - base;
    }
#pragma unroll
    for (int l = 0; l < D; l++) {
#pragma unroll
        for (int k = 0; k < NK; k++) {
            const uint2 q = lds64(p[k]);
            const float v = ldsf(q.x + xr);
            p[k] = 2u * p[k] + (v >= __uint_as_float(q.y) ? s1[k] : s0[k]);
        }
    }
#pragma unroll
    for (int k = 0; k < NK; k++) {
        const uint32_t base = tree0 + k * tree_bytes;
        const uint32_t ord = ((p[k] - base) >> 3) - kInt;
        const float lv = ldsf(base + kInt * 8u + ord * 4u);
        acc = a.unit_w ? __dadd_rn(acc, (double)lv)
                       : __dadd_rn(acc, __dmul_rn(__ldg(a.weight + t + k), (double)lv));
        if (a.ord && valid) a.ord[(long long)(t + k) * a.ld_ord + row] = (uint16_t)ord;
    }
}

template <int D, int K>
__global__ void __launch_bounds__(kThreads, 1) k_stream(StreamArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *xs = reinterpret_cast<float *>(smem);
    unsigned char *ring = smem + a.xs_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + kStages * a.chunk_cap);
    uint64_t *empty = full + kStages;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; s++) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long ntiles = (a.n + kB - 1) / kB;
    const int nchunks = (a.t1 - a.t0 + a.tpc - 1) / a.tpc;

    if (warp == kConsumerWarps) {  // ---- producer warp: TMA bulk copies
        if (lane == 0) {
            uint32_t it = 0;
            for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int c = 0; c < nchunks; c++, it++) {
                    const int s = it % kStages;
                    if (it >= kStages) mbar_wait(empty + s, ((it / kStages) - 1) & 1);
                    const int trees = min(a.tpc, a.t1 - a.t0 - c * a.tpc);
                    const uint32_t bytes = (uint32_t)trees * a.tree_bytes;
                    mbar_expect_tx(full + s, bytes);
                    bulk_g2s(ring + s * a.chunk_cap,
                             a.blob + a.seg_byte0 + (size_t)c * a.tpc * a.tree_bytes, bytes,
                             full + s);
                }
            }
        }
        return;
    }

    // ---- consumer warps
    const int r = threadIdx.x;
    const uint32_t xr = su32(xs) + 4u * r;
    uint32_t it = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long row = tile * kB + r;
        const bool valid = row < a.n;
        consumer_sync();  // previous tile's walks are done with xs
        stage_rows(a, xs, tile * kB);
        consumer_sync();
        double acc = (a.accumulate && valid) ? a.out[row] : 0.0;
        for (int c = 0; c < nchunks; c++, it++) {
            const int s = it % kStages;
            mbar_wait(full + s, (it / kStages) & 1);
            const uint32_t buf = su32(ring + s * a.chunk_cap);
            const int t0 = a.t0 + c * a.tpc;
            const int trees = min(a.tpc, a.t1 - t0);
            int k = 0;
            for (; k + K <= trees; k += K)
                walk_group<D, K>(buf + k * a.tree_bytes, a.tree_bytes, xr, acc, a, t0 + k, row,
                                 valid);
            for (; k < trees; k++)
                walk_group<D, 1>(buf + k * a.tree_bytes, a.tree_bytes, xr, acc, a, t0 + k, row,
                                 valid);
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
        if (valid) a.out[row] = acc;
    }
}

template <int D>
cudaError_t launch_d(const StreamArgs &a, int device, cudaStream_t stream) {
    auto kern = k_stream<D, 8>;
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    const size_t smem = a.xs_bytes + (size_t)kStages * a.chunk_cap + 2 * kStages * 8;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long tiles = (a.n + kB - 1) / kB;
    const int grid = (int)(tiles < sms ? tiles : sms);
    kern<<<grid, kThreads, smem, stream>>>(a);
    count_launch();
    return cudaGetLastError();
}

using StreamFn = cudaError_t (*)(const StreamArgs &, int, cudaStream_t);
const StreamFn kStreamTable[kStreamMaxDepth + 1] = {
    launch_d<0>, launch_d<1>, launch_d<2>, launch_d<3>, launch_d<4>, launch_d<5>,
    launch_d<6>, launch_d<7>, launch_d<8>, launch_d<9>, launch_d<10>, launch_d<11>};

}  // namespace

int stream_instances_per_tile() { return kB; }

// Shared-memory plan for a segment of depth D over F features; returns false
// when the tile + two stages of at least K trees do not fit (the caller then
// uses the L1 kernel).
bool plan_stream(int F, int D, int device, StreamArgs *a) {
    if (D > kStreamMaxDepth) return false;
    int optin = 0;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) !=
        cudaSuccess)
        return false;
    const size_t xs = ((size_t)F * kB * sizeof(float) + 127) & ~(size_t)127;
    const uint32_t tb = a->tree_bytes;
    const size_t bars = 2 * kStages * 8;
    if (xs + bars + (size_t)kStages * tb > (size_t)optin) return false;
    size_t cap = ((size_t)optin - xs - bars) / kStages;
    cap = std::min<size_t>(cap, 48 * 1024);
    uint32_t tpc = (uint32_t)(cap / tb);
    if (tpc >= 8) tpc &= ~7u;  // whole K-groups per chunk
    if (tpc < 1) return false;
    a->xs_bytes = (uint32_t)xs;
    a->tpc = (int)tpc;
    a->chunk_cap = (tpc * tb + 127) & ~127u;
    return true;
}

cudaError_t launch_stream(int D, const StreamArgs &a, int device, cudaStream_t stream) {
    if (a.n <= 0) return cudaSuccess;
    return kStreamTable[D](a, device, stream);
}

}  // namespace ts
