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
//  * each walk writes its leaf value to a shared leaf buffer lb[tree][inst]
//    (tree = the slot's position in evaluation order within the chunk);
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
#include <type_traits>

#include "ts_internal.h"
#include "ts_stream_kernel.cuh"

namespace ts {
namespace cstream_detail {

using namespace stream_detail;

constexpr int kWarps = 8;
constexpr int kConsumers = kWarps * 32;
constexpr int kThreadsC = kConsumers + 64;  // + accumulator warp + producer warp
constexpr int kStagesC = 2;
constexpr uint32_t kMetaBytes = kCStreamMaxT * 4;  // slot table at the head of a stage
constexpr uint32_t kHeadBytes = kMetaBytes + 16;   // + the chunk's chunk_info entry

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
        constexpr int U = 8;  // independent loads in flight per thread
        for (int e0 = tid; e0 < B * F4; e0 += U * kConsumers) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int e = e0 + u * kConsumers;
                const int r = e % B, c4 = e / B;
                const long long row = row0 + r;
                v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (e < B * F4 && row < a.n)
                    v[u] = __ldg(reinterpret_cast<const float4 *>(a.x + row * a.ld) + c4);
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int e = e0 + u * kConsumers;
                if (e >= B * F4) break;
                const int r = e % B, c4 = e / B;
                bad |= !(finite_f(v[u].x) && finite_f(v[u].y) && finite_f(v[u].z) &&
                         finite_f(v[u].w));
                float *dst = xs + (4 * c4) * B + r;
                dst[0] = v[u].x;
                dst[B] = v[u].y;
                dst[2 * B] = v[u].z;
                dst[3 * B] = v[u].w;
            }
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

template <int kK, int G, bool UNIT_W, bool ORD>
__global__ void __launch_bounds__(kThreadsC, 1) k_cstream(CStreamArgs a) {
    // G instance groups of 32 (B = 32 * G) is a template parameter so the
    // accumulator's per-lane instance loop is fully unrolled with exactly G
    // independent f64 chains and the walkers' x-tile stride is an immediate.
    extern __shared__ __align__(128) unsigned char smem[];
    float *xs = reinterpret_cast<float *>(smem);
    float *lb0 = reinterpret_cast<float *>(smem + a.xs_bytes);  // two leaf buffers
    unsigned char *ring = smem + a.xs_bytes + a.lb_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + kStagesC * a.stage_bytes);
    uint64_t *empty = full + kStagesC;  // ring stage consumed (8 walker warps)
    uint64_t *lbf = empty + kStagesC;   // leaf buffer written (8 walker warps)
    uint64_t *lbe = lbf + 2;            // leaf buffer folded (accumulator warp)
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStagesC; s++) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kWarps);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(lbf + b, kWarps);
            mbar_init(lbe + b, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    constexpr int B = 32 * G;
    const long long ntiles = (a.n + B - 1) / B;
    const uint32_t lb_half = a.lb_bytes / 2;

    if (warp == kWarps + 1) {  // ---- producer: TMA bulk copies per chunk
        if (lane == 0) {
            uint32_t it = 0;
            for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int c = 0; c < a.nchunks; c++, it++) {
                    const int s = it % kStagesC;
                    if (it >= kStagesC) mbar_wait(empty + s, ((it / kStagesC) - 1) & 1);
                    const uint4 ci = __ldg(a.chunk_info + a.chunk0 + c);
                    unsigned char *stage = ring + s * a.stage_bytes;
                    mbar_expect_tx(full + s, ci.y + kMetaBytes + 16);
                    bulk_g2s(stage, a.slot_meta + (size_t)(a.chunk0 + c) * kCStreamMaxT,
                             kMetaBytes, full + s);
                    bulk_g2s(stage + kMetaBytes, a.chunk_info + a.chunk0 + c, 16, full + s);
                    bulk_g2s(stage + kHeadBytes, a.blob + 16ull * ci.x, ci.y, full + s);
                }
            }
        }
        return;
    }

    if (warp == kWarps) {  // ---- accumulator: folds leaves in TREE order
        uint32_t it = 0;
        for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const long long row0 = tile * B;
            double acc[G];
#pragma unroll
            for (int g = 0; g < G; g++) {
                const long long row = row0 + g * 32 + lane;
                acc[g] = (a.accumulate && row < a.n) ? a.out[row] : 0.0;
            }
            for (int c = 0; c < a.nchunks; c++, it++) {
                const uint4 ci = __ldg(a.chunk_info + a.chunk0 + c);
                const int nt = (int)ci.z;
                const int b = it & 1;
                mbar_wait(lbf + b, (it >> 1) & 1);
                const float *lbc = reinterpret_cast<const float *>(
                    reinterpret_cast<const unsigned char *>(lb0) + b * lb_half);
                for (int i = 0; i < nt; i++) {
                    double w = 1.0;
                    if constexpr (!UNIT_W) w = __ldg(a.weight + ci.w + i);
#pragma unroll
                    for (int g = 0; g < G; g++) {
                        const double lv = (double)lbc[i * B + g * 32 + lane];
                        acc[g] = UNIT_W ? __dadd_rn(acc[g], lv) : __dadd_rn(acc[g], __dmul_rn(w, lv));
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(lbe + b);
            }
#pragma unroll
            for (int g = 0; g < G; g++) {
                const long long row = row0 + g * 32 + lane;
                if (row < a.n) a.out[row] = acc[g];
            }
        }
        return;
    }

    // ---- walkers (8 warps)
    const int grp = warp % G;
    const int S = kWarps / G;
    const int sub = warp / G;
    const int inst = grp * 32 + lane;
    const uint32_t xr = su32(xs) + 4u * inst;
    constexpr uint32_t B4 = 4u * B;
    const uint32_t lbase0 = su32(lb0);
    uint32_t it = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long row0 = tile * B;
        consumer_sync<kConsumers>();  // all walks of the previous tile are done
        stage_rows_c(a, xs, row0);
        consumer_sync<kConsumers>();
        const long long walk_row = row0 + inst;
        const bool walk_valid = walk_row < a.n;
        for (int c = 0; c < a.nchunks; c++, it++) {
            const int s = it % kStagesC;
            const int b = it & 1;
            const uint32_t lbase = lbase0 + b * lb_half;
            mbar_wait(full + s, (it / kStagesC) & 1);
            const uint32_t meta = su32(ring + s * a.stage_bytes);
            uint32_t nt, tree0;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(nt), "=r"(tree0)
                         : "r"(meta + kMetaBytes + 8));  // chunk_info .z/.w
            const uint32_t buf = meta + kHeadBytes;
            bool waited = it < 2;  // this leaf buffer's previous fold must be done
            for (int s0 = sub; s0 < (int)nt; s0 += S * kK) {
                uint32_t p[kK], tb[kK], ob[kK], rel[kK];
                int dk[kK];
                int dmax = 0;
#pragma unroll
                for (int k = 0; k < kK; k++) {
                    const int slot = s0 + k * S;
                    uint32_t m;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(m)
                                 : "r"(meta + 4u * (slot < (int)nt ? slot : s0)));
                    rel[k] = m >> 21;
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
                if (!waited) {
                    mbar_wait(lbe + b, ((it >> 1) - 1) & 1);
                    waited = true;
                }
#pragma unroll
                for (int k = 0; k < kK; k++) {
                    const int slot = s0 + k * S;
                    if (slot < (int)nt) {
                        const float lv = ldsf(p[k] + 4u);
                        asm volatile("st.shared.f32 [%0], %1;" ::"r"(lbase + 4u * (rel[k] * B + inst)),
                                     "f"(lv));
                        if constexpr (ORD) {
                            if (walk_valid)
                                a.ord[(long long)(tree0 + rel[k]) * a.ld_ord + walk_row] =
                                    (uint16_t)(ob[k] >> (dmax - dk[k]));
                        }
                    }
                }
            }
            if (!waited) mbar_wait(lbe + b, ((it >> 1) - 1) & 1);
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(empty + s);  // ring stage read
                mbar_arrive(lbf + b);    // leaves published (release orders the stores)
            }
        }
    }
}

}  // namespace cstream_detail

bool plan_cstream(int F, int device, CStreamArgs *a) {
    using namespace cstream_detail;
    const int optin = dev_attrs(device).smem_optin;
    if (!optin) return false;
    // Largest instance tile first; then the chain count K whose full round of
    // S * K trees (one K-group per warp) fits a ring stage at ~1.2 KB/tree.
    for (int G = 8; G >= 1; G >>= 1) {
        const int B = 32 * G;
        const int S = kWarps / G;
        const size_t xs = ((size_t)(F + 1) * B * 4 + 127) & ~(size_t)127;
        for (int K = 8; K >= 4; K >>= 1) {
            const int tpc = std::min(S * K, kCStreamMaxT);
            const size_t lb = 2 * (size_t)tpc * B * 4;  // double-buffered
            const size_t bars = 8 * 8;
            if (xs + lb + bars >= (size_t)optin) continue;
            const size_t stage = ((((size_t)optin - xs - lb - bars) / kStagesC) & ~(size_t)127);
            if (stage < kHeadBytes + (size_t)tpc * 1200) continue;
            a->B = B;
            a->k = K;
            a->tpc = tpc;
            a->xs_bytes = (uint32_t)xs;
            a->lb_bytes = (uint32_t)lb;
            a->stage_bytes = (uint32_t)std::min<size_t>(stage, 64 * 1024 + kHeadBytes);
            a->chunk_cap = a->stage_bytes - kHeadBytes;  // tree bytes per stage
            return true;
        }
    }
    return false;
}

cudaError_t launch_cstream(const CStreamArgs &a, int device, cudaStream_t stream) {
    using namespace cstream_detail;
    if (a.n <= 0) return cudaSuccess;
    auto pick = [&](auto kk, auto gg) {
        constexpr int K = decltype(kk)::value, G = decltype(gg)::value;
        return a.ord ? (a.unit_w ? k_cstream<K, G, true, true> : k_cstream<K, G, false, true>)
                     : (a.unit_w ? k_cstream<K, G, true, false> : k_cstream<K, G, false, false>);
    };
    auto pick_g = [&](auto kk) {
        switch (a.B) {
            case 256: return pick(kk, std::integral_constant<int, 8>{});
            case 128: return pick(kk, std::integral_constant<int, 4>{});
            case 64: return pick(kk, std::integral_constant<int, 2>{});
            default: return pick(kk, std::integral_constant<int, 1>{});
        }
    };
    auto kern = a.k == 8 ? pick_g(std::integral_constant<int, 8>{})
                         : pick_g(std::integral_constant<int, 4>{});
    const int sms = dev_attrs(device).sms;
    cudaError_t e;
    const size_t smem = (size_t)a.xs_bytes + a.lb_bytes + (size_t)kStagesC * a.stage_bytes + 8 * 8;
    e = ensure_smem((const void *)kern, smem);
    if (e != cudaSuccess) return e;
    const long long tiles = (a.n + a.B - 1) / a.B;
    const int grid = (int)(tiles < sms ? tiles : sms);
    kern<<<grid, kThreadsC, smem, stream>>>(a);
    count_launch();
    return cudaGetLastError();
}

}  // namespace ts
