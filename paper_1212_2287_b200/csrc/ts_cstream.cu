// ts_cstream.cu -- streaming kernel for IRREGULAR trees (BASELINE config 3:
// LambdaMART-shaped trees of <= 64 leaves and depth <= 16 over F = 700
// features).  Complete expansion would cost 2^16 slots per tree, so these
// trees keep their own nodes (kCStream records, ts_internal.h) and are
// streamed through shared memory by TMA exactly like ts_stream_kernel.cuh.
//
// What differs from the complete-tree kernel:
//  * wide feature rows leave room for only B = 32*G instances (G instance
//    groups of 32), so the 8 consumer warps split the TREES of each chunk as
//    well: warp w walks instance group w % G over the chunk's tree slots
//    (w / G), (w / G) + S, ... with S = 8 / G;
//  * inside a chunk the packer orders tree slots by depth, so the K trees a
//    thread walks in lockstep have nearly equal depth (a K-group steps
//    max(depth) times; a leaf is a self-loop whose x row is the -inf sentinel
//    row F, so shorter trees idle on their leaf);
//  * each walk writes its leaf value to a shared leaf buffer lb[slot][inst];
//    after the chunk, thread `inst` folds the chunk's leaves into its f64
//    accumulator in TREE order (acc = acc + w * leaf, __dmul_rn/__dadd_rn),
//    so the result stays bit-identical to the reference's sequential sum
//    (ref evaluators.py:529-535) whatever order the walks ran in.
// The per-level step is the reference predicate (ref evaluators.py:90-99)
// on child-index records: rec = {fid | left8 << 16, theta}, next record at
// tree_base + left8 + 8 * (x[fid] >= theta).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "ts_internal.h"
#include "ts_stream_kernel.cuh"

namespace ts {
namespace cstream_detail {

using namespace stream_detail;

constexpr int kWarps = 8;
constexpr int kConsumers = kWarps * 32;
constexpr int kThreadsC = kConsumers + 32;
constexpr int kK = 4;  // lockstep chains per thread
constexpr int kStagesC = 2;

// Stage B rows x F features into xs[f * B + r] (+ sentinel row F = -inf),
// all 256 consumer threads cooperating.
__device__ __forceinline__ void stage_rows_c(const CStreamArgs &a, float *xs, long long row0) {
    const int B = a.B;
    const int F = a.F;
    const int tid = threadIdx.x;
    bool bad = false;
    const bool vec = ((F & 3) == 0) && ((a.ld & 3) == 0) &&
                     ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
    if (vec) {
        const int F4 = F >> 2;
        for (int e = tid; e < B * F4; e += kConsumers) {
            const int r = e % B, c4 = e / B;
            const long long row = row0 + r;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (row < a.n) v = __ldg(reinterpret_cast<const float4 *>(a.x + row * a.ld) + c4);
            bad |= !(finite_f(v.x) && finite_f(v.y) && finite_f(v.z) && finite_f(v.w));
            float *dst = xs + (4 * c4) * B + r;
            dst[0] = v.x;
            dst[B] = v.y;
            dst[2 * B] = v.z;
            dst[3 * B] = v.w;
        }
    } else {
        for (int e = tid; e < B * F; e += kConsumers) {
            const int r = e % B, c = e / B;
            const long long row = row0 + r;
            float v = row < a.n ? __ldg(a.x + row * a.ld + c) : 0.f;
            bad |= !finite_f(v);
            xs[c * B + r] = v;
        }
    }
    for (int r = tid; r < B; r += kConsumers) xs[F * B + r] = -INFINITY;
    if (bad && a.status) atomicOr(a.status, 1);
}

template <bool UNIT_W, bool ORD>
__global__ void __launch_bounds__(kThreadsC, 1) k_cstream(CStreamArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *xs = reinterpret_cast<float *>(smem);
    float *lb = reinterpret_cast<float *>(smem + a.xs_bytes);
    unsigned char *ring = smem + a.xs_bytes + a.lb_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + kStagesC * a.chunk_cap);
    uint64_t *empty = full + kStagesC;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStagesC; s++) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int B = a.B;
    const long long ntiles = (a.n + B - 1) / B;

    if (warp == kWarps) {  // ---- producer: one TMA bulk copy per chunk
        if (lane == 0) {
            uint32_t it = 0;
            for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int c = 0; c < a.nchunks; c++, it++) {
                    const int s = it % kStagesC;
                    if (it >= kStagesC) mbar_wait(empty + s, ((it / kStagesC) - 1) & 1);
                    const uint4 ci = __ldg(a.chunk_info + a.chunk0 + c);
                    mbar_expect_tx(full + s, ci.y);
                    bulk_g2s(ring + s * a.chunk_cap, a.blob + 16ull * ci.x, ci.y, full + s);
                }
            }
        }
        return;
    }

    // ---- consumers
    const int tid = threadIdx.x;
    const int G = B >> 5;
    const int grp = warp % G;
    const int S = kWarps / G;
    const int sub = warp / G;
    const int inst = grp * 32 + lane;
    const uint32_t xr = su32(xs) + 4u * inst;
    const uint32_t B4 = 4u * B;
    const uint32_t lbase = su32(lb);
    uint32_t it = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long row0 = tile * B;
        consumer_sync();
        stage_rows_c(a, xs, row0);
        consumer_sync();
        const long long my_row = row0 + tid;  // accumulator owner (tid < B)
        double acc = (tid < B && my_row < a.n && a.accumulate) ? a.out[my_row] : 0.0;
        const long long walk_row = row0 + inst;
        const bool walk_valid = walk_row < a.n;
        for (int c = 0; c < a.nchunks; c++, it++) {
            const int s = it % kStagesC;
            const uint4 ci = __ldg(a.chunk_info + a.chunk0 + c);
            const int nt = (int)ci.z;
            const uint32_t *meta = a.slot_meta + (size_t)(a.chunk0 + c) * kCStreamMaxT;
            mbar_wait(full + s, (it / kStagesC) & 1);
            const uint32_t buf = su32(ring + s * a.chunk_cap);
            for (int s0 = sub; s0 < nt; s0 += S * kK) {
                uint32_t p[kK], tb[kK], ob[kK];
                int dk[kK];
                int dmax = 0;
#pragma unroll
                for (int k = 0; k < kK; k++) {
                    const int slot = s0 + k * S;
                    const uint32_t m = slot < nt ? __ldg(meta + slot) : __ldg(meta + s0);
                    tb[k] = buf + 8u * (m & 0xffffu);
                    p[k] = tb[k];
                    dk[k] = (m >> 16) & 31;
                    dmax = max(dmax, dk[k]);
                    ob[k] = 0;
                }
#pragma unroll 1
                for (int l = 0; l < dmax; l++) {
#pragma unroll
                    for (int k = 0; k < kK; k++) {
                        const uint2 q = lds64(p[k]);
                        const float v = ldsf((q.x & 0xffffu) * B4 + xr);
                        const bool c = v >= __uint_as_float(q.y);
                        p[k] = tb[k] + (q.x >> 16) + (c ? 8u : 0u);
                        if constexpr (ORD) ob[k] = 2u * ob[k] + (c ? 1u : 0u);
                    }
                }
#pragma unroll
                for (int k = 0; k < kK; k++) {
                    const int slot = s0 + k * S;
                    if (slot < nt) {
                        const float lv = ldsf(p[k] + 4u);
                        asm volatile("st.shared.f32 [%0], %1;" ::"r"(lbase + 4u * (slot * B + inst)),
                                     "f"(lv));
                        if constexpr (ORD) {
                            if (walk_valid) {
                                const uint32_t rel = __ldg(meta + slot) >> 21;
                                a.ord[(long long)(ci.w + rel) * a.ld_ord + walk_row] =
                                    (uint16_t)(ob[k] >> (dmax - dk[k]));
                            }
                        }
                    }
                }
            }
            consumer_sync();  // leaf buffer complete; ring stage fully read
            if (tid == 0) mbar_arrive(empty + s);
            if (tid < B) {
                const unsigned char *inv = a.slot_inv + (size_t)(a.chunk0 + c) * kCStreamMaxT;
                for (int i = 0; i < nt; i++) {
                    const float lv = lb[__ldg(inv + i) * B + tid];
                    if constexpr (UNIT_W) acc = __dadd_rn(acc, (double)lv);
                    else acc = __dadd_rn(acc, __dmul_rn(__ldg(a.weight + ci.w + i), (double)lv));
                }
            }
            consumer_sync();  // leaf buffer free for the next chunk
        }
        if (tid < B && my_row < a.n) a.out[my_row] = acc;
    }
}

}  // namespace cstream_detail

bool plan_cstream(int F, int device, CStreamArgs *a) {
    using namespace cstream_detail;
    int optin = 0;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) !=
        cudaSuccess)
        return false;
    for (int G = 8; G >= 1; G >>= 1) {
        const int B = 32 * G;
        const size_t xs = ((size_t)(F + 1) * B * 4 + 127) & ~(size_t)127;
        const size_t lb = (size_t)kCStreamMaxT * B * 4;
        const size_t bars = 4 * 8;
        if (xs + lb + bars >= (size_t)optin) continue;
        const size_t cap = (((size_t)optin - xs - lb - bars) / kStagesC) & ~(size_t)127;
        if (cap < 8 * 1024) continue;
        a->B = B;
        a->xs_bytes = (uint32_t)xs;
        a->lb_bytes = (uint32_t)lb;
        a->chunk_cap = (uint32_t)std::min<size_t>(cap, 64 * 1024);
        // trees per chunk: whole rounds of (S subsets x K chains), <= kCStreamMaxT
        const int S = kWarps / G;
        int tpc = S * kK;
        while (tpc * 2 <= kCStreamMaxT) tpc *= 2;
        a->tpc = tpc;
        return true;
    }
    return false;
}

cudaError_t launch_cstream(const CStreamArgs &a, int device, cudaStream_t stream) {
    using namespace cstream_detail;
    if (a.n <= 0) return cudaSuccess;
    auto kern = a.ord ? (a.unit_w ? k_cstream<true, true> : k_cstream<false, true>)
                      : (a.unit_w ? k_cstream<true, false> : k_cstream<false, false>);
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    const size_t smem = (size_t)a.xs_bytes + a.lb_bytes + (size_t)kStagesC * a.chunk_cap + 4 * 8;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long tiles = (a.n + a.B - 1) / a.B;
    const int grid = (int)(tiles < sms ? tiles : sms);
    kern<<<grid, kThreadsC, smem, stream>>>(a);
    count_launch();
    return cudaGetLastError();
}

}  // namespace ts
