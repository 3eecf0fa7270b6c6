#pragma once
// ts_rank_kernel.cuh -- the rank form of the complete-tree walk (kRank layout,
// ts_internal.h; planning and launch: ts_rank.cu).
//
// Why: a deep complete tree is shared-memory-capacity-bound in k_stream.  A
// d = 12 tree's node part is 20.6 KB (8-byte top records, fp32 thresholds +
// 1-byte fids below) and a 256-row fp32 instance tile 139 KB, which leaves
// room for two lockstep chains per thread (16 per SM); with four the same
// walk runs 1.43x faster (profiles/r2_rank_design.txt).  Replacing every
// threshold by its rank among the ensemble's distinct thresholds of that
// feature makes a node ONE 4-byte record and an instance value a 2-byte rank:
// the tile halves, the records shrink by a fifth, and a node visit is one
// LDS.32 (one wavefront at the top levels) instead of LDS.64 / LDS + LDS.U8.
// Exactness: rank(v) = #{distinct thresholds u of the feature : u <= v}; for
// a threshold theta of that feature rank(theta) is its own 1-based position,
// and v >= theta <=> rank(v) >= rank(theta) for every float v (the order is
// IEEE's, -0.0 == +0.0; dummy +inf nodes get kRankInf, above every rank) --
// the reference's predicate x >= theta (ref evaluators.py:90-99), bit for bit.
//
//  * k_rank (pre-pass): R[tile][f][r] = rank(x[tile * 256 + r][f]) as u16 in
//    tile-transposed layout, so the walk stages a tile with plain 16-byte
//    copies; each CTA holds one group of features' threshold lists in shared
//    memory (one bulk copy) and binary-searches four rows per thread at once.
//  * k_rstream<D, K>: k_stream's structure (persistent 256-row tiles, one
//    producer warp streaming the segment's trees through a TMA ring, eight
//    consumer warps walking K trees in lockstep) on kRank records:
//        rec = LDS.32 [p];  v = LDS.U16 [xr + (rec >> 15)]   (= fid * 512;
//                                                      xr: rank_slot(row))
//        c = (v | rec & 0xff000000) >= rec                    (= rank(x) >= rank)
//        p = 2p + (c ? 8 - base : 4 - base)                   (heap step)
//    then w * leaf added in f64 in tree order (__dmul_rn / __dadd_rn).
#include "ts_stream_kernel.cuh"

namespace ts {
namespace rank_detail {

using namespace stream_detail;

constexpr int kCW = 8;                  // consumer warps: 256-row tiles
// (rank_slot: ts_internal.h)
constexpr int kThreads = kCW * 32 + 32;
constexpr int kRankMaxStages = 4;

struct RankArgs {
    const uint16_t *R;                  // [tiles][F][256] u16 instance ranks
    long long n;
    int F;
    const unsigned char *blob;
    unsigned long long seg_byte0;
    uint32_t tree_bytes, ring_tree_bytes, leaf0;
    int tpc;
    uint32_t chunk_cap;
    int stages;
    uint32_t xs_bytes;
    const double *weight;
    int t0, t1;
    int unit_w, accumulate;
    double *out;
    uint16_t *ord;
    long long ld_ord;
    // Balanced tree split (ts_stream.cu launch_balanced, same scheme): sk_ctas
    // CTAs take equal runs of the tile-major (tile, chunk) items; a tile
    // shared by several CTAs gets one partial per CTA ([tile][slice][row]).
    int sk_ctas, sk_slices;
    double *part_sum;
    uint32_t *part_key;
};

// ---------------------------------------------------------------------------
// Walk.
template <int KP>
struct RankPend {
    float lv[KP];
    int t = 0, n = 0;
    // balanced split (StreamArgs::part_key): high word of the largest |running
    // sum|, smallest nonzero |leaf| bit pattern minus 1
    uint32_t amax = 0u, kmin1 = 0xffffffffu;
};

template <bool UNIT_W, int KP, bool TRACK = false>
__device__ __forceinline__ void rank_flush(RankPend<KP> &pend, double &acc, const RankArgs &a) {
#pragma unroll
    for (int j = 0; j < KP; j++) {
        if (j < pend.n) {
            const double term = UNIT_W ? (double)pend.lv[j]
                                       : __dmul_rn(__ldg(a.weight + pend.t + j), (double)pend.lv[j]);
            acc = __dadd_rn(acc, term);
            if constexpr (TRACK)
                pend.amax = max(pend.amax, (uint32_t)__double2hiint(acc) & 0x7fffffffu);
        }
    }
    pend.n = 0;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    TS_DBG(addr, 4);
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t addr) {
    TS_DBG(addr, 2);
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// NK trees of one ring stage in lockstep, tree k's records at tree0 + k * TB.
// ORD: 0 scores, 1 also ordinals, 2 balanced split (unit weights, no
// ordinals: partial-sum bookkeeping).
template <int D, int NK, bool UNIT_W, int ORD, int KP>
__device__ __forceinline__ void rank_group(uint32_t tree0, uint32_t TB, uint32_t xr, double &acc,
                                           const RankArgs &a, int t, long long row, bool valid,
                                           RankPend<KP> &pend) {
    constexpr bool kGLeaf = D >= 11;
    uint32_t p[NK], lo[NK], hi[NK];
#pragma unroll
    for (int k = 0; k < NK; k++) {
        const uint32_t base = tree0 + k * TB;
        p[k] = base;
        lo[k] = 4u - base;
        hi[k] = 8u - base;
    }
#pragma unroll
    for (int l = 0; l < D; l++) {
#pragma unroll
        for (int k = 0; k < NK; k++) {
            const uint32_t rec = lds32(p[k]);
            const uint32_t v = lds16(xr + (rec >> 15));  // fid * 512: rank < 2^15
            const bool c = (v | (rec & 0xff000000u)) >= rec;
            p[k] = p[k] + p[k] + (c ? hi[k] : lo[k]);
        }
    }
    if constexpr (kGLeaf) rank_flush<UNIT_W, KP, ORD == 2>(pend, acc, a);  // the previous group's leaves
#pragma unroll
    for (int k = 0; k < NK; k++) {
        const uint32_t base = tree0 + k * TB;
        const uint32_t leaf = ((p[k] - base) >> 2) - ((1u << D) - 1u);  // 0 .. 2^D - 1
        float lv;
        if constexpr (kGLeaf)
            lv = __ldg(reinterpret_cast<const float *>(a.blob + a.seg_byte0 +
                                                       (size_t)(t + k - a.t0) * a.tree_bytes +
                                                       a.leaf0) +
                       leaf);
        else
            lv = ldsf(base + a.leaf0 + 4u * leaf);
        if constexpr (kGLeaf) {  // added after the next group's walk (L2 latency hidden)
            pend.lv[k] = lv;
            if (k == NK - 1) {
                pend.t = t;
                pend.n = NK;
            }
        } else {
            const double term =
                UNIT_W ? (double)lv : __dmul_rn(__ldg(a.weight + t + k), (double)lv);
            acc = __dadd_rn(acc, term);
            if constexpr (ORD == 2)
                pend.amax = max(pend.amax, (uint32_t)__double2hiint(acc) & 0x7fffffffu);
        }
        if constexpr (ORD == 2)
            pend.kmin1 = min(pend.kmin1, (__float_as_uint(lv) & 0x7fffffffu) - 1u);  // zero wraps: ignored
        if constexpr (ORD == 1)
            if (a.ord && valid) a.ord[(long long)(t + k) * a.ld_ord + row] = (uint16_t)leaf;
    }
}

template <int D>
__device__ __forceinline__ void produce_rank_chunk(const RankArgs &a, unsigned char *stage,
                                                   uint64_t *bar, int c, int trees) {
    const unsigned char *src = a.blob + a.seg_byte0 + (size_t)c * a.tpc * a.tree_bytes;
    mbar_expect_tx(bar, (uint32_t)trees * a.ring_tree_bytes);
    if (a.ring_tree_bytes != a.tree_bytes) {
        for (int i = 0; i < trees; i++)
            bulk_g2s(stage + (size_t)i * a.ring_tree_bytes, src + (size_t)i * a.tree_bytes,
                     a.ring_tree_bytes, bar);
    } else {
        bulk_g2s(stage, src, (uint32_t)trees * a.tree_bytes, bar);
    }
}

template <int D, int K, bool UNIT_W, int ORD>
__global__ void __launch_bounds__(kThreads, 1) k_rstream(RankArgs a) {
    constexpr int kB = kCW * 32;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *xs = smem;                      // [F][256] u16 ranks
    unsigned char *ring = smem + a.xs_bytes;
    const int kStages = a.stages;
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + kStages * a.chunk_cap);
    uint64_t *empty = full + kRankMaxStages;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kRankMaxStages; s++) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long ntiles = (a.n + kB - 1) / kB;
    const int nchunks = (a.t1 - a.t0 + a.tpc - 1) / a.tpc;
    // balanced split (ORD == 2): this CTA's run of tile-major (tile, chunk) items
    long long it_lo = 0, it_hi = 0;
    if constexpr (ORD == 2) {
        const long long W = ntiles * nchunks;
        it_lo = (long long)blockIdx.x * W / a.sk_ctas;
        it_hi = (long long)(blockIdx.x + 1) * W / a.sk_ctas;
    }

    if (warp == kCW) {  // ---- producer warp
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0, used = 0;
            auto produce = [&](int cb, int ce) {
                for (int c = cb; c < ce; c++) {
                    if (used) mbar_wait(empty + s, ph);
                    const int trees = min(a.tpc, a.t1 - a.t0 - c * a.tpc);
                    produce_rank_chunk<D>(a, ring + s * a.chunk_cap, full + s, c, trees);
                    if (++s == kStages) {
                        s = 0;
                        ph ^= used;
                        used = 1;
                    }
                }
            };
            if constexpr (ORD == 2) {
                for (long long pos = it_lo; pos < it_hi;) {
                    const int cb = (int)(pos % nchunks);
                    const int ce = (int)min((long long)nchunks, cb + (it_hi - pos));
                    produce(cb, ce);
                    pos += ce - cb;
                }
            } else {
                for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) produce(0, nchunks);
            }
        }
        return;
    }

    // ---- consumer warps
    const int r = threadIdx.x;
    const uint32_t xr = su32(xs) + 2u * rank_slot((uint32_t)r);
    const uint32_t TB = a.ring_tree_bytes;
    const int tile_vec = a.F * kB * 2 / 16;  // 16-byte pieces of a rank tile
    int s = 0;
    uint32_t ph = 0;
    auto consume = [&](const long long tile, const int cb, const int ce) {
        const long long row = tile * kB + r;
        const bool valid = row < a.n;
        consumer_sync<kB>();  // previous tile's walks are done with xs
        {
            const uint4 *src = reinterpret_cast<const uint4 *>(a.R + tile * a.F * kB);
            uint4 *dst = reinterpret_cast<uint4 *>(xs);
            for (int i = r; i < tile_vec; i += kB) dst[i] = __ldg(src + i);
        }
        consumer_sync<kB>();
        // balanced split: a tile walked only in part contributes a partial sum from 0
        const bool part = ORD == 2 && (cb != 0 || ce != nchunks);
        double acc = (a.accumulate && valid && !part) ? a.out[row] : 0.0;
        RankPend<K> pend;
        for (int c = cb; c < ce; c++) {
            mbar_wait(full + s, ph);
            const uint32_t buf = su32(ring + s * a.chunk_cap);
            const int t0 = a.t0 + c * a.tpc;
            const int trees = min(a.tpc, a.t1 - t0);
            int k = 0;
            for (; k + K <= trees; k += K)
                rank_group<D, K, UNIT_W, ORD, K>(buf + k * TB, TB, xr, acc, a, t0 + k, row,
                                                 valid, pend);
            for (; k < trees; k++)
                rank_group<D, 1, UNIT_W, ORD, K>(buf + k * TB, TB, xr, acc, a, t0 + k, row,
                                                 valid, pend);
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
            if (++s == kStages) {
                s = 0;
                ph ^= 1u;
            }
        }
        if constexpr (D >= 11) rank_flush<UNIT_W, K, ORD == 2>(pend, acc, a);
        if (part) {
            if (valid) {  // slice = this CTA's rank among the CTAs sharing the tile
                const long long W = ntiles * nchunks;
                const long long b0 = ((tile * nchunks + 1) * a.sk_ctas - 1) / W;
                const long long pj = (tile * a.sk_slices + (blockIdx.x - b0)) * kB + r;
                a.part_sum[pj] = acc;
                a.part_key[2 * pj] = pend.amax;
                a.part_key[2 * pj + 1] = pend.kmin1;
            }
        } else if (valid && a.out) {
            a.out[row] = acc;
        }
    };
    if constexpr (ORD == 2) {
        for (long long pos = it_lo; pos < it_hi;) {
            const long long tile = pos / nchunks;
            const int cb = (int)(pos - tile * nchunks);
            const int ce = (int)min((long long)nchunks, cb + (it_hi - pos));
            consume(tile, cb, ce);
            pos += ce - cb;
        }
    } else {
        for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) consume(tile, 0, nchunks);
    }
}

}  // namespace rank_detail
}  // namespace ts

namespace ts {
namespace rank_detail {

// Lockstep chains per depth: the tuned count, then a fallback for rows too
// wide to leave two ring stages of the tuned K-group.
__host__ __device__ constexpr int rank_chains(int d) {
    return d <= 8 ? 8 : d <= 10 ? 8 : d == 11 ? 6 : d == 12 ? 4 : d == 13 ? 2 : 1;
}
__host__ __device__ constexpr int rank_chains_fallback(int d) {
    return d <= 10 ? 4 : d == 11 ? 3 : d == 12 ? 2 : 1;
}

template <int D>
cudaError_t launch_rank_d(const RankArgs &a, int k, int device, cudaStream_t stream) {
    constexpr int K1 = rank_chains(D), K2 = rank_chains_fallback(D);
    auto pick = [&](auto kc) {
        constexpr int KK = decltype(kc)::value;
        if (a.sk_ctas > 0) return k_rstream<D, KK, true, 2>;  // unit weights, no ordinals
        if (a.ord) return a.unit_w ? k_rstream<D, KK, true, 1> : k_rstream<D, KK, false, 1>;
        return a.unit_w ? k_rstream<D, KK, true, 0> : k_rstream<D, KK, false, 0>;
    };
    auto kern = k == K1 ? pick(std::integral_constant<int, K1>{})
                        : pick(std::integral_constant<int, K2>{});
    const size_t smem = (size_t)a.xs_bytes + (size_t)a.stages * a.chunk_cap +
                        2 * kRankMaxStages * 8;
    cudaError_t e = ensure_smem((const void *)kern, smem);
    if (e != cudaSuccess) return e;
    const long long tiles = (a.n + kRankB - 1) / kRankB;
    const int sms = dev_attrs(device).sms;
    const int grid = a.sk_ctas > 0 ? a.sk_ctas : (int)std::min<long long>(tiles, sms);
    kern<<<grid, kThreads, smem, stream>>>(a);
    count_launch();
    return cudaGetLastError();
}

}  // namespace rank_detail
}  // namespace ts
