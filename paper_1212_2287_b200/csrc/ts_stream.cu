// ts_stream.cu -- planning and dispatch for the complete-tree streaming
// kernel (ts_stream_kernel.cuh; instantiated per depth in ts_stream_i*.cu so
// nvcc compiles them in parallel).
//
// plan_stream() sizes one CTA: x tile (B rows x F features, fp32,
// feature-major) + a ring of 2-4 stages, each holding a whole number of
// K-groups of kSplit tree records; it prefers two 128-row CTAs per SM
// (d <= 9) so one CTA's x staging overlaps the other's walks, and one 256-row
// CTA otherwise.  Trees that do not fit (d > 12 or rows too wide) fall back to
// the L1-path kernels in ts_kernels.cu.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "ts_internal.h"
#include "ts_stream_kernel.cuh"

namespace ts {
namespace stream_detail {
extern template cudaError_t launch_d<0>(const StreamArgs &, int, cudaStream_t);
extern template cudaError_t launch_d<1>(const StreamArgs &, int, cudaStream_t);
extern template cudaError_t launch_d<2>(const StreamArgs &, int, cudaStream_t);
extern template cudaError_t launch_d<3>(const StreamArgs &, int, cudaStream_t);
extern template cudaError_t launch_d<4>(const StreamArgs &, int, cudaStream_t);
extern template cudaError_t launch_d<5>(const StreamArgs &, int, cudaStream_t);
extern template cudaError_t launch_d<6>(const StreamArgs &, int, cudaStream_t);
extern template cudaError_t launch_d<7>(const StreamArgs &, int, cudaStream_t);
extern template cudaError_t launch_d<8>(const StreamArgs &, int, cudaStream_t);
extern template cudaError_t launch_d<9>(const StreamArgs &, int, cudaStream_t);
extern template cudaError_t launch_d<10>(const StreamArgs &, int, cudaStream_t);
extern template cudaError_t launch_d<11>(const StreamArgs &, int, cudaStream_t);
extern template cudaError_t launch_d<12>(const StreamArgs &, int, cudaStream_t);
#define TS_WS_EXTERN(D) extern template cudaError_t launch_ws_d<D>(const StreamArgs &, int, cudaStream_t);
TS_WS_EXTERN(0) TS_WS_EXTERN(1) TS_WS_EXTERN(2) TS_WS_EXTERN(3) TS_WS_EXTERN(4) TS_WS_EXTERN(5)
TS_WS_EXTERN(6) TS_WS_EXTERN(7) TS_WS_EXTERN(8) TS_WS_EXTERN(9) TS_WS_EXTERN(10) TS_WS_EXTERN(11)
TS_WS_EXTERN(12)
#undef TS_WS_EXTERN

namespace {
using StreamFn = cudaError_t (*)(const StreamArgs &, int, cudaStream_t);
const StreamFn kStreamTable[kStreamMaxDepth + 1] = {
    launch_d<0>, launch_d<1>, launch_d<2>, launch_d<3>, launch_d<4>, launch_d<5>,
    launch_d<6>, launch_d<7>, launch_d<8>, launch_d<9>, launch_d<10>, launch_d<11>, launch_d<12>};
const StreamFn kWsTable[kStreamMaxDepth + 1] = {
    launch_ws_d<0>, launch_ws_d<1>, launch_ws_d<2>,  launch_ws_d<3>,  launch_ws_d<4>,
    launch_ws_d<5>, launch_ws_d<6>, launch_ws_d<7>,  launch_ws_d<8>,  launch_ws_d<9>,
    launch_ws_d<10>, launch_ws_d<11>, launch_ws_d<12>};

}  // namespace
}  // namespace stream_detail


// Shared-memory plan for a segment of depth D over F features; returns false
// when the tile + two stages of at least K trees do not fit (the caller then
// uses the L1 kernel).
namespace {
bool plan_stream_cw(int F, int D, int optin, int cw, StreamArgs *a) {
    using namespace stream_detail;
    const int B = 32 * cw;
    int ctas = std::min(256 / B, 4);
    if (const char *fc = getenv("TS_STREAM_CTAS")) ctas = std::max(1, std::min(ctas, atoi(fc)));
    // per-CTA budget when several CTAs share an SM (1 KB reserved per CTA)
    if (ctas > 1) optin = std::min(optin, 228 * 1024 / ctas - 1024);
    const size_t xs = ((size_t)F * B * sizeof(float) + 127) & ~(size_t)127;
    a->fw = split_fid_width(F);
    a->tree_bytes = split_geom(D, a->fw).bytes;
    a->ring_tree_bytes = split_ring_bytes(D, a->fw);
    const uint32_t tb = a->ring_tree_bytes;
    const size_t bars = 2 * kMaxStages * 8;
    if (xs + bars + (size_t)2 * tb > (size_t)optin) return false;
    const size_t ring = (size_t)optin - xs - bars;
    // the tuned chain count first; the 256-row shape may fall back to
    // chains_fallback(D) (a second kernel instantiation) before single trees
    uint32_t K = 0;
    int stages = 0;
    uint32_t tpc = 0;
    const uint32_t cands[2] = {(uint32_t)chains_for_depth(D), (uint32_t)chains_fallback(D)};
    for (int ci = 0; ci < (cw == 8 ? 2 : 1) && !stages; ci++) {
        const size_t group = (size_t)cands[ci] * tb;
        for (int s = kMaxStages; s >= 2 && !stages; s--) {
            size_t cap = ring / s;
            if (cap < group) continue;
            size_t g = cap / group;
            const size_t soft = 48 * 1024;   // small chunks keep the ring turning over
            if (g > 1 && g * group > soft) g = std::max<size_t>(1, soft / group);
            stages = s;
            K = cands[ci];
            tpc = (uint32_t)(g * K);
        }
    }
    if (!stages) {
        if (cw != 8) return false;  // the 256-row shape handles it better
        stages = 2;                 // not even two K-groups fit: single trees
        K = cands[1];
        tpc = (uint32_t)std::max<size_t>(1, (ring / 2) / tb);
    }
    a->k = (int)K;
    a->cw = cw;
    a->xs_bytes = (uint32_t)xs;
    a->tpc = (int)tpc;
    a->stages = stages;
    a->chunk_cap = (tpc * tb + 15) & ~15u;  // TMA bulk copies need 16-byte granules
    return true;
}
}  // namespace

// Shared-memory plan for a segment of depth D over F features: two 128-row
// CTAs per SM when a full ring of K-groups fits (d <= 9), else one 256-row
// CTA; false when not even that fits (the caller uses the L1 kernel).
bool plan_stream(int F, int D, int device, StreamArgs *a, long long n) {
    if (D > kStreamMaxDepth) return false;
    const int optin = dev_attrs(device).smem_optin, sms = dev_attrs(device).sms;
    if (!optin || !sms) return false;
    (void)n;  // 32-row tiles for small batches measured slower (cfg0: 17.4 vs 15.2 us)
    if (const char *fc = getenv("TS_STREAM_CW")) {  // tuning experiments only
        const int cw = atoi(fc);
        if ((cw == 4 || cw == 8) && plan_stream_cw(F, D, optin, cw, a)) return true;
    }
    if (D <= 9 && plan_stream_cw(F, D, optin, 4, a)) return true;
    return plan_stream_cw(F, D, optin, 8, a);
}

// Warp-split shape: a 32-row x tile, two fp32 leaf buffers of tpc trees and a
// ring of 2-4 stages of tpc = kWsWarps * K trees (one K-group per walker warp
// per chunk), within a third of an SM's shared memory if it fits (three CTAs
// per SM), else half.
bool plan_stream_ws(int F, int D, int device, StreamArgs *a) {
    using namespace stream_detail;
    if (D > kStreamMaxDepth) return false;
    const size_t xs = ((size_t)F * 32 * sizeof(float) + 127) & ~(size_t)127;
    a->fw = split_fid_width(F);
    a->tree_bytes = split_geom(D, a->fw).bytes;
    a->ring_tree_bytes = split_ring_bytes(D, a->fw);
    const uint32_t tpc = (uint32_t)(kWsWarps * ws_chains(D));
    const size_t lb = 2ull * tpc * 32 * sizeof(float);
    const size_t chunk = ((size_t)tpc * a->ring_tree_bytes + 127) & ~(size_t)127;
    const size_t bars = (2 * kMaxStages + 4) * 8;
    for (int ctas = 3; ctas >= 2; ctas--) {
        const int budget = std::min(dev_attrs(device).smem_optin, 228 * 1024 / ctas - 1024);
        if (budget <= 0 || xs + lb + bars + 2 * chunk > (size_t)budget) continue;
        a->ws_ctas = ctas;
        a->xs_bytes = (uint32_t)xs;
        a->lb_bytes = (uint32_t)lb;
        a->tpc = (int)tpc;
        a->chunk_cap = (uint32_t)chunk;
        a->stages = (int)std::min<size_t>(kMaxStages, ((size_t)budget - xs - lb - bars) / chunk);
        return true;
    }
    return false;
}

namespace {
// Tree-order f64 fold of a tree-split launch (ref evaluators.py:529-535):
// one CTA per 32 rows; all 8 warps stream the rows' leaf values
// ([row/32][tree][row%32], 128 B per tree) into a double-buffered shared
// tile with cp.async while warp 0 folds the previous tile, one lane per row,
// acc = acc + w * leaf in tree order (__dmul_rn / __dadd_rn).
constexpr int kFoldTrees = 96;  // trees per shared tile (24 KB of f64 terms)
__device__ __forceinline__ void fold_load(double *dst, const double *src, int trees) {
    // trees * 32 doubles = trees * 16 16-byte pieces over the block's threads
    const uint32_t d0 = (uint32_t)__cvta_generic_to_shared(dst);
    for (int i = threadIdx.x; i < trees * 16; i += blockDim.x)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d0 + 16u * i),
                     "l"(src + 2 * i)
                     : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// Exactness test of a row's tree-split sum.  The terms of a unit-weight
// ensemble are fp32 leaf values: every term, and so every partial sum, is a
// multiple of 2^q, q the LSB exponent of the smallest nonzero |leaf| (and of
// the running sum acc0 the segment continues from).  M bounds every partial
// sum the tree-order chain or the splits can form: |acc0| plus the largest
// |running sum| each split reached (amax, rounded up).  If M < 2^m with
// m - q <= 53, every one of those sums is exactly representable in f64: no
// addition rounds, so the reference's tree-order sum (ref
// evaluators.py:529-535) equals the plain sum of the splits' own sums.
// kmin1: smallest nonzero |leaf| bit pattern minus 1 (0xffffffff: no nonzero
// term).  Otherwise (wide dynamic range; non-unit weights send amax = all
// ones, i.e. M = infinity) the caller adds the terms one by one in tree order.
__device__ __forceinline__ double amax_bound(uint32_t amax) {
    // >= the |sum| whose high word is amax; all ones (non-unit weights) and
    // anything at the top of the range: infinity, which fails the test
    return amax >= 0x7fe00000u ? INFINITY : __hiloint2double((int)(amax + 1u), 0);
}
__device__ __forceinline__ bool split_sum_exact(double M, uint32_t kmin1, double acc0) {
    if (kmin1 == 0xffffffffu) return !(acc0 == 0.0 && signbit(acc0)) && M < INFINITY;  // all terms zero
    int q = max((int)((kmin1 + 1u) >> 23), 1) - 150;  // every term is a multiple of 2^q
    if (acc0 != 0.0) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(acc0);
        const int ea = (int)((b >> 52) & 0x7ff);
        if (ea == 0 || ea == 0x7ff) return false;  // subnormal, inf, nan: take the slow path
        const unsigned long long mant = (b & 0xfffffffffffffull) | (1ull << 52);
        q = min(q, ea - 1075 + (__ffsll((long long)mant) - 1));
    } else if (signbit(acc0)) {
        return false;                              // -0.0 + (+0.0 sums): sign depends on the order
    }
    const double Mt = M + fabs(acc0);
    if (!(Mt < INFINITY)) return false;
    const int em = (int)(((unsigned long long)__double_as_longlong(Mt) >> 52) & 0x7ff);
    const int m = em - 1022 + 1;                   // Mt < 2^(em - 1022); one more for M's own rounding
    return m - q <= 53;
}

// One CTA per 32 rows.  Fast path (warp 0, one lane per row): add the splits'
// own sums when split_sum_exact proves the order cannot matter.  Otherwise
// all 8 warps pull the rows' f64 terms (w * leaf, already rounded by the walk)
// into double-buffered shared tiles with cp.async and warp 0 adds them, one
// lane per row, in tree order -- a bare DADD chain.
__global__ void __launch_bounds__(256) k_fold(const double *terms, long long T, int accumulate,
                                              double *out, long long n, const double *part_sum,
                                              const uint32_t *part_key, int splits,
                                              int no_fast) {
    __shared__ __align__(16) double tile[2][kFoldTrees * 32];
    const long long blk = blockIdx.x;
    const long long row = blk * 32 + (threadIdx.x & 31);
    const double *src = terms + blk * T * 32;
    double acc = 0.0;
    int done = 0;
    if (!no_fast) {
        // all 8 warps fetch the splits' partials (one round trip), warp 0 decides
        const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
        double sum = 0.0, M = 0.0;
        uint32_t kmin1 = 0xffffffffu;
        const double *ps = part_sum + blk * splits * 32 + lane;
        const uint32_t *pk = part_key + blk * splits * 64 + lane;
#pragma unroll 8
        for (int j = w; j < splits; j += 8) {
            sum = __dadd_rn(sum, ps[j * 32]);
            M += amax_bound(pk[j * 64]);
            kmin1 = min(kmin1, pk[j * 64 + 32]);
        }
        double *rs = tile[0];                                        // [8][32] sums
        double *rm = tile[0] + 256;                                  // [8][32] magnitude bounds
        uint32_t *rk = reinterpret_cast<uint32_t *>(tile[0] + 512);  // [8][32] keys
        rs[threadIdx.x] = sum;
        rm[threadIdx.x] = M;
        rk[threadIdx.x] = kmin1;
        __syncthreads();
        if (w == 0) {
            const bool valid = row < n;
            if (accumulate && valid) acc = out[row];
#pragma unroll
            for (int u = 1; u < 8; u++) {
                sum = __dadd_rn(sum, rs[u * 32 + lane]);
                M += rm[u * 32 + lane];
                kmin1 = min(kmin1, rk[u * 32 + lane]);
            }
            bool ok = !valid || split_sum_exact(M, kmin1, acc);
            ok = __all_sync(0xffffffffu, ok);
            if (ok && valid) out[row] = __dadd_rn(acc, sum);
            done = ok ? 1 : 0;
        }
    } else if (threadIdx.x < 32 && accumulate && row < n) {
        acc = out[row];
    }
    if (__syncthreads_or(done)) return;  // warp 0's verdict; also fences tile[0] before the loads
    const int ntile = (int)((T + kFoldTrees - 1) / kFoldTrees);
    fold_load(tile[0], src, (int)min(T, (long long)kFoldTrees));
    for (int i = 0; i < ntile; i++) {
        const int tb = i * kFoldTrees;
        const int nt = (int)min(T - tb, (long long)kFoldTrees);
        if (i + 1 < ntile) {
            fold_load(tile[(i + 1) & 1], src + (long long)(tb + kFoldTrees) * 32,
                      (int)min(T - tb - kFoldTrees, (long long)kFoldTrees));
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const double *lv = tile[i & 1] + threadIdx.x;
#pragma unroll 8
            for (int t = 0; t < nt; t++) acc = __dadd_rn(acc, lv[t * 32]);
        }
        __syncthreads();  // tile (i & 1) is refilled next iteration
    }
    if (threadIdx.x < 32 && row < n) out[row] = acc;
}
// One tree walked in global memory for one row, from the segment's packed
// records (LeafWalk, ts_internal.h) -- the predicate of the streaming walks,
// the reference's i = (i << 1) + 1 + (x[fid[i]] >= theta[i]) (ref
// evaluators.py:90-99).  Returns the leaf value.
//  * kSplit (ts_stream_kernel.cuh walk_group): header / top records / deep
//    arrays, fp32 thresholds against the row's fp32 values;
//  * kRank (ts_rank_kernel.cuh rank_group): 4-byte records fid << 24 | rank
//    against the row's u16 ranks in its rank tile;
//  * kCStream (ts_cstream_kernel.cuh): child-index records of an irregular
//    tree, down to its leaf.
__device__ __forceinline__ float leaf_walk_global(const LeafWalk &g, long long t, long long row) {
    uint32_t j = 0;  // 0-based heap index
    if (g.rank == 2) {
        // kCStream: {x offset << 14 | left child's record, theta}; a leaf's x
        // offset is the sentinel row F (ts_cstream_kernel.cuh)
        const uint2 *recs = reinterpret_cast<const uint2 *>(g.seg + 16ull * __ldg(g.tree_off16 + t));
        const float *xrow = g.x + row * g.ld;
        for (;;) {
            const uint2 q = __ldg(recs + j);
            const uint32_t fid = q.x >> (14 + g.xshift);
            if (fid >= (uint32_t)g.F) return __uint_as_float(q.y);
            j = (q.x & 0x3fffu) + (__ldg(xrow + fid) >= __uint_as_float(q.y) ? 1u : 0u);
        }
    }
    const unsigned char *tree = g.seg + t * g.tree_bytes;
    if (g.rank) {
        const uint16_t *rr = g.R + (row / kRankB) * g.F * kRankB + rank_slot((uint32_t)(row % kRankB));
        const uint32_t *recs = reinterpret_cast<const uint32_t *>(tree);
        for (int l = 0; l < g.D; l++) {
            const uint32_t rec = __ldg(recs + j);
            const uint32_t v = __ldg(rr + (rec >> 24) * kRankB);
            j = 2u * j + 1u + ((v | (rec & 0xff000000u)) >= rec ? 1u : 0u);
        }
        return __ldg(reinterpret_cast<const float *>(tree + g.leaf0) + (j + 1u - (1u << g.D)));
    }
    const float *xrow = g.x + row * g.ld;
    const int S = g.D < kTopLevels ? g.D : kTopLevels;
    int l = 0;
    if (g.header) {
        const uint4 hd = __ldg(reinterpret_cast<const uint4 *>(tree));
        const bool c0 = __ldg(xrow + (hd.x & 0xffu)) >= __uint_as_float(hd.y);
        const uint32_t f1 = (hd.x >> (c0 ? 16 : 8)) & 0xffu;
        const bool c1 = __ldg(xrow + f1) >= __uint_as_float(c0 ? hd.w : hd.z);
        j = 3u + (c0 ? 2u : 0u) + (c1 ? 1u : 0u);
        l = 2;
    }
    for (; l < S; l++) {
        const uint2 q = __ldg(reinterpret_cast<const uint2 *>(tree) + j);
        j = 2u * j + 1u + (__ldg(xrow + (q.x >> kFidShift)) >= __uint_as_float(q.y) ? 1u : 0u);
    }
    for (; l < g.D; l++) {
        const uint32_t k = j + 1u - (1u << S);  // index in the deep arrays
        const float th = __ldg(reinterpret_cast<const float *>(tree + g.thr0) + k);
        const uint32_t fid = g.fw == 1 ? (uint32_t)__ldg(tree + g.fid0 + k)
                                       : (uint32_t)__ldg(reinterpret_cast<const uint16_t *>(tree + g.fid0) + k);
        j = 2u * j + 1u + (__ldg(xrow + fid) >= th ? 1u : 0u);
    }
    return __ldg(reinterpret_cast<const float *>(tree + g.leaf0) + (j + 1u - (1u << g.D)));
}

// Balanced tree split, second kernel: one CTA per tile.  A tile shared by
// several walking CTAs (StreamArgs::sk_ctas) has one partial per CTA; a row
// whose partial sums provably cannot round (split_sum_exact) gets their sum,
// which then IS the tree-order sum.  Any other row (non-unit weights, a wide
// leaf range: ~2e-4 of the rows for N(0,1) leaves at T = 1000) is scored
// again here, in tree order: warps 1..15 walk its trees in the model blob
// (leaf_walk_global, 480 trees at a time), lane 0 of warp 0 adds the
// previous batch's terms -- term = w * leaf rounded to f64, then the add, the
// walk's own arithmetic (ref evaluators.py:529-535).
// kCombineThreads / B threads fetch each row's partials.
constexpr int kCombineThreads = 512;
constexpr int kCombineBatch = kCombineThreads - 32;  // trees walked per step of the slow path
__global__ void __launch_bounds__(kCombineThreads)
    k_combine(const double *part_sum, const uint32_t *part_key, int slices, int B,
              long long ntiles, int nchunks, int ctas, long long T, int accumulate, double *out,
              long long n, LeafWalk g, int no_fast) {
    __shared__ double rs[kCombineThreads];
    __shared__ double rm[kCombineThreads];
    __shared__ uint32_t rk[kCombineThreads];
    __shared__ double terms[2][kCombineBatch];
    __shared__ int slow_rows[256];
    __shared__ int n_slow;
    const long long tile = blockIdx.x;
    const long long W = ntiles * nchunks;
    const long long b0 = ((tile * nchunks + 1) * ctas - 1) / W;
    const long long b1 = ((tile + 1) * nchunks * ctas - 1) / W;
    const int cnt = (int)(b1 - b0 + 1);
    if (cnt == 1) return;  // walked whole by one CTA, which wrote the scores
    const int r = threadIdx.x % B, p = threadIdx.x / B, P = kCombineThreads / B;
    const long long row = tile * B + r;
    const bool valid = row < n;
    if (threadIdx.x == 0) n_slow = 0;
    double sum = 0.0, M = 0.0;
    uint32_t kmin1 = 0xffffffffu;
    if (valid) {
#pragma unroll 4
        for (int j = p; j < cnt; j += P) {
            const long long pj = (tile * slices + j) * B + r;
            sum = __dadd_rn(sum, part_sum[pj]);
            const uint2 k = *reinterpret_cast<const uint2 *>(part_key + 2 * pj);
            M += amax_bound(k.x);
            kmin1 = min(kmin1, k.y);
        }
    }
    rs[threadIdx.x] = sum;
    rm[threadIdx.x] = M;
    rk[threadIdx.x] = kmin1;
    __syncthreads();
    if (p == 0 && valid) {
        for (int u = 1; u < P; u++) {
            sum = __dadd_rn(sum, rs[u * B + r]);
            M += rm[u * B + r];
            kmin1 = min(kmin1, rk[u * B + r]);
        }
        const double acc = accumulate ? out[row] : 0.0;
        if (!no_fast && split_sum_exact(M, kmin1, acc)) out[row] = __dadd_rn(acc, sum);
        else slow_rows[atomicAdd(&n_slow, 1)] = r;
    }
    __syncthreads();
    const int ns = n_slow;
    if (threadIdx.x == 0 && g.slow_dev) {  // DeviceTables::slow_dev, slow_seen
        const unsigned int rows = (unsigned int)min((long long)B, n - tile * B);
        const unsigned int s1 = atomicAdd(g.slow_dev + 1, rows) + rows;
        const unsigned int s0 = ns ? atomicAdd(g.slow_dev, (unsigned int)ns) + ns : 0u;
        if (g.slow_seen_dev && (ns || blockIdx.x == 0)) {
            if (ns) g.slow_seen_dev[0] = s0;
            g.slow_seen_dev[1] = s1;
        }
    }
    for (int i = 0; i < ns; i++) {
        const long long srow = tile * B + slow_rows[i];
        double acc = 0.0;
        if (threadIdx.x == 0 && accumulate) acc = out[srow];
        auto walk_batch = [&](long long t0, double *dst) {
            const long long t = t0 + (threadIdx.x - 32);
            if (threadIdx.x >= 32 && t < T) {
                const float lv = leaf_walk_global(g, t, srow);
                dst[threadIdx.x - 32] = g.weight ? __dmul_rn(__ldg(g.weight + t), (double)lv) : (double)lv;
            }
        };
        walk_batch(0, terms[0]);
        __syncthreads();
        int b = 0;
        for (long long t0 = 0; t0 < T; t0 += kCombineBatch, b ^= 1) {
            if (t0 + kCombineBatch < T) walk_batch(t0 + kCombineBatch, terms[b ^ 1]);
            if (threadIdx.x == 0) {
                const int nt = (int)min((long long)kCombineBatch, T - t0);
#pragma unroll 8
                for (int k = 0; k < nt; k++) acc = __dadd_rn(acc, terms[b][k]);
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) out[srow] = acc;
    }
}
}  // namespace

cudaError_t launch_combine(const double *part_sum, const uint32_t *part_key, int slices, int B,
                           long long tiles, int nchunks, int ctas, long long T, int accumulate,
                           double *out, long long n, const LeafWalk &walk, cudaStream_t stream) {
    // TS_FOLD_FAST=0: every shared tile's rows on the tree-order path (tests, A/B)
    const char *ff = getenv("TS_FOLD_FAST");
    k_combine<<<(unsigned)tiles, kCombineThreads, 0, stream>>>(
        part_sum, part_key, slices, B, tiles, nchunks, ctas, T, accumulate, out, n, walk,
        ff && atoi(ff) == 0 ? 1 : 0);
    count_launch();
    return cudaGetLastError();
}

bool balanced_split_trusted(const DeviceTables *t) {
    if (!t || !t->slow_seen) return true;
    const unsigned int slow = t->slow_seen[0], rows = t->slow_seen[1];
    return !(rows >= 2048u && (unsigned long long)slow * 100ull > 3ull * rows);
}

// Where the balanced split measured faster (profiles/r2_balanced_split.txt):
// its time grows linearly with the batch, ~13 % above the whole-tile kernel's
// rate at full waves, while whole tiles cost whole waves -- so it pays while
// the last wave is poorly filled.  With fill = tiles / resident CTA slots: a
// first wave filled up to 0.8 at d = 7-9 and 0.7 elsewhere -- from 0.12 (d =
// 7-9) / 0.4 up where the uniform split and the warp-split kernel serve the
// smallest batches (has_small_batch_paths), from the first tile where nothing
// else does (the rank walk) -- or a second / third wave filled to at most 0.6
// (d >= 6).  The walk must be long enough to carry the second launch.
bool balanced_split_pays(int D, long long T, long long tiles, int resident,
                         bool has_small_batch_paths, long long max_trees) {
    if (T > max_trees || T * D < 6000) return false;
    const double fill = (double)tiles / resident;
    const int waves_done = (int)fill;
    const double frac = fill - waves_done;
    const bool mid = D >= 7 && D <= 9;
    // (the rank walk's balanced kernel carries no ordinal / split checks of
    // its own, so it stays ahead up to fuller waves: d=12 T=1000 n = 30k,
    // fill 0.8: 332 -> 294 us)
    const double lo = !has_small_batch_paths ? 0.0 : mid ? 0.12 : 0.4;
    const double hi = !has_small_batch_paths ? 0.90 : mid ? 0.80 : 0.70;
    const double hi2 = !has_small_batch_paths ? 0.75 : 0.60;
    return (waves_done == 0 && frac >= lo && frac <= hi) ||
           (waves_done >= 1 && waves_done <= 2 && frac <= hi2 && D >= 6);
}

// Balanced tree split ("stream-K"): batches of less than a few waves of tiles
// -- where whole-tile CTAs leave SMs idle or a last partial wave costs a whole
// one -- are cut into `ctas` equal runs of (tile, chunk) items
// (StreamArgs::sk_ctas).  Two launches: the walk and k_combine.
static cudaError_t launch_balanced(int D, const StreamArgs &a, int ctas, long long tiles,
                                   int nchunks, int device, cudaStream_t stream) {
    const int B = 32 * a.cw;
    const int T = a.t1 - a.t0;
    const int slices = (int)((ctas + tiles - 1) / tiles) + 1;
    const size_t psum_bytes = (size_t)tiles * slices * B * sizeof(double);
    cudaMemPool_t pool = scratch_pool(device);
    if (!pool) return cudaErrorNotSupported;
    unsigned char *scratch = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync((void **)&scratch, 2 * psum_bytes, pool, stream);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return cudaErrorNotSupported;  // the caller goes on to the other kernels
    }
    StreamArgs w = a;
    float *xcopy = nullptr;
    if (a.x_mapped) {
        // CTAs sharing a tile each read its rows: not over PCIe
        e = x_device_copy(a.x, a.n, a.ld, device, stream, &xcopy);
        if (e != cudaSuccess) {
            cudaFreeAsync(scratch, stream);
            return e;
        }
        if (xcopy) w.x = xcopy;
    }
    w.sk_ctas = ctas;
    w.sk_slices = slices;
    w.part_sum = reinterpret_cast<double *>(scratch);
    w.part_key = reinterpret_cast<uint32_t *>(scratch + psum_bytes);
    e = stream_detail::kStreamTable[D](w, device, stream);
    if (e == cudaSuccess) {
        const SplitGeom sg = split_geom(D, a.fw);
        LeafWalk g{};
        g.D = D;
        g.fw = a.fw;
        g.header = split_header(D, a.fw) ? 1 : 0;
        g.thr0 = sg.thr0;
        g.fid0 = sg.fid0;
        g.leaf0 = sg.leaf0;
        g.tree_bytes = sg.bytes;
        g.x = w.x;
        g.ld = a.ld;
        g.seg = a.blob + a.seg_byte0;
        g.weight = a.unit_w ? nullptr : a.weight + a.t0;
        g.slow_dev = a.tables ? a.tables->slow_dev : nullptr;
        g.slow_seen_dev = a.tables ? a.tables->slow_seen_dev : nullptr;
        e = launch_combine(w.part_sum, w.part_key, slices, B, tiles, nchunks, ctas, T, a.accumulate,
                           a.out, a.n, g, stream);
    }
    cudaError_t f = cudaFreeAsync(scratch, stream);
    if (xcopy) {
        const cudaError_t g2 = cudaFreeAsync(xcopy, stream);
        if (f == cudaSuccess) f = g2;
    }
    return e != cudaSuccess ? e : f;
}

// Small batches leave most SMs idle (one CTA walks ALL trees of its tile), so
// when the tiles fill less than half of the resident CTA slots the segment's
// chunks are split over `splits` CTAs per tile: phase 1 walks and stores each
// tree's f64 term w * leaf (stream-ordered scratch from the library's memory
// pool), phase 2 (k_fold) adds them in tree order -- bit-identical to the
// one-pass kernel.
// TS_SPLIT=0 disables, TS_SPLIT=J forces J splits (A/B experiments).
cudaError_t launch_stream(int D, const StreamArgs &a0, int device, cudaStream_t stream) {
    if (a0.n <= 0) return cudaSuccess;
    StreamArgs a = a0;
    a.splits = 1;
    a.leaf_out = nullptr;
    const long long B = 32ll * a.cw;
    const long long tiles = (a.n + B - 1) / B;
    const int resident = dev_attrs(device).sms * (a.cw == 4 ? 2 : 1);
    const int T = a.t1 - a.t0;
    const int nchunks = (T + a.tpc - 1) / a.tpc;
    // worth it only when a tile's walk is long (>= 2048 node visits per row)
    const bool long_walk = (long long)T * D >= 2048;
    int splits = (long_walk && tiles * 2 <= resident)
                     ? (int)std::min<long long>(nchunks, resident / tiles) : 1;
    if (const char *e = getenv("TS_SPLIT")) {
        const int f = atoi(e);
        splits = f <= 0 ? 1 : std::min(f, nchunks);
    }
    // Balanced tree split (launch_balanced) where it measured faster
    // (balanced_split_pays): d=8 T=1000: n = 5k 46 -> 34 us, 12k 87 -> 56,
    // 20k 124 -> 81, 40k 166 -> 149, 50k 212 -> 181; d=6: 16k 64 -> 52, 40k
    // 136 -> 112; d=10 (T = 300): 20k 61 -> 49, 40k 117 -> 83.  Unit weights
    // only (other sums are never provably exact) and leaves whose magnitudes
    // leave at most ~0.1 % of the rows to k_combine's one-at-a-time second
    // walk (Segment::slow_rows: 11.6 us per row at T = 1000).  TS_SK=1
    // forces it (any weights, any shape), TS_SK=0 disables it; TS_SK_CTAS
    // overrides the CTA count (tests, A/B).
    {
        const char *ske = getenv("TS_SK");
        bool sk = a.unit_w && long_walk && a.slow_rows <= 1e-3f && balanced_split_trusted(a.tables) &&
                  balanced_split_pays(D, T, tiles, resident, true) && !getenv("TS_SPLIT") &&
                  !getenv("TS_WS");
        if (ske) sk = atoi(ske) != 0;
        if (sk && !a.pipe.flags_in && !a.pipe.sums_out) {
            const long long W = tiles * nchunks;
            long long ctas = std::min<long long>(resident, W);
            if (const char *ce = getenv("TS_SK_CTAS")) ctas = std::min<long long>(std::max(1, atoi(ce)), W);
            if (ctas > tiles || tiles % ctas != 0) {
                const cudaError_t e = launch_balanced(D, a, (int)ctas, tiles, nchunks, device, stream);
                if (e != cudaErrorNotSupported) return e;
            }
        }
    }
    // Warp-split kernel (k_stream_ws) for batches whose 32-row tiles fill at
    // most 1.5 waves of its CTAs and give every SM one (or whose walk is too
    // short for the two-pass split): each tile's trees split over four walker
    // warps, no second pass (r1: cfg0 10.3 -> 8.1 us, 9k rows x 1000 d=8
    // trees 73 -> 49 us, 12k x 1000 d=8 98 -> 88 us, 20k x 100 d=6 14.6 ->
    // 12.1 us, 1k rows x 100 d=6 trees 10.1 -> 5.1 us; at ~2 waves the
    // one-pass kernel wins again; 3k rows x 1000 d=8 trees stay on the
    // two-pass split, 32 vs 43 us).  Depth <= 8 (deeper trees
    // leave it one chain per warp).  TS_WS=0|1 disables / forces it (A/B
    // experiments).
    {
        StreamArgs w = a;
        const long long tiles32 = (a.n + 31) / 32;
        const int sms = dev_attrs(device).sms;
        const bool fits = D <= 8 && plan_stream_ws(a.F, D, device, &w);
        bool ws = fits && 2 * tiles32 <= 3ll * w.ws_ctas * sms && (tiles32 >= sms || !long_walk);
        if (const char *e = getenv("TS_WS")) ws = atoi(e) != 0 && plan_stream_ws(a.F, D, device, &w);
        if (ws && !a.pipe.flags_in && !a.pipe.sums_out && !getenv("TS_SPLIT"))
            return stream_detail::kWsTable[D](w, device, stream);
    }
    const long long blocks = (a.n + 31) / 32;
    // terms, then each split's own sum and leaf-magnitude keys (StreamArgs::part_sum)
    const size_t term_bytes = (size_t)blocks * 32 * (size_t)T * sizeof(double);
    const size_t psum_bytes = (size_t)blocks * std::max(splits, 1) * 32 * sizeof(double);
    const size_t scratch_bytes = term_bytes + 2 * psum_bytes;
    if (splits < 2 || a.pipe.flags_in || a.pipe.sums_out || scratch_bytes > (256u << 20)) {
        // Wave tail: when the last wave of tiles would leave more than half
        // the CTA slots idle, the full waves run here and the remaining rows
        // go to k_stream_ws, whose 32-row tiles spread them over every SM.
        // Config 1: the 27th wave of 117 tiles cost a whole wave (2.1 % of
        // the pass); with the tail on k_stream_ws the pass is 0.6 % faster
        // (the warp-split kernel's own rate is lower).  d = 7-8 only: at d = 3
        // it measured 1.4 % slower.  TS_WS=0 disables it.
        const long long waves = tiles / resident, rem = tiles % resident;
        const char *wse = getenv("TS_WS");
        if (D >= 7 && D <= 8 && waves >= 1 && rem > 0 && 2 * rem <= resident && !a.pipe.flags_in &&
            !a.pipe.sums_out && !(wse && atoi(wse) == 0)) {
            StreamArgs w = a;
            if (plan_stream_ws(a.F, D, device, &w)) {
                const long long n_main = waves * resident * B;
                StreamArgs m = a;
                m.n = n_main;
                cudaError_t e = stream_detail::kStreamTable[D](m, device, stream);
                if (e != cudaSuccess) return e;
                w.x = a.x + n_main * a.ld;
                w.n = a.n - n_main;
                w.out = a.out ? a.out + n_main : nullptr;
                w.ord = a.ord ? a.ord + n_main : nullptr;  // row offset; ld_ord unchanged
                return stream_detail::kWsTable[D](w, device, stream);
            }
        }
        return stream_detail::kStreamTable[D](a, device, stream);
    }

    cudaMemPool_t pool = scratch_pool(device);
    if (!pool) return stream_detail::kStreamTable[D](a, device, stream);
    double *scratch = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync((void **)&scratch, scratch_bytes, pool, stream);
    if (e != cudaSuccess) {
        // out of memory for the split's scratch: the one-pass kernel needs
        // none and gives the same bits, only slower for this batch size
        (void)cudaGetLastError();
        return stream_detail::kStreamTable[D](a, device, stream);
    }
    StreamArgs w = a;
    float *xcopy = nullptr;
    if (a.x_mapped) {
        // every split CTA of a tile re-reads its rows: not over PCIe
        e = x_device_copy(a.x, a.n, a.ld, device, stream, &xcopy);
        if (e != cudaSuccess) {
            cudaFreeAsync(scratch, stream);
            return e;
        }
        if (xcopy) w.x = xcopy;
    }
    w.splits = splits;
    w.leaf_out = scratch;
    w.leaf_T = T;
    w.part_sum = reinterpret_cast<double *>(reinterpret_cast<unsigned char *>(scratch) + term_bytes);
    w.part_key = reinterpret_cast<uint32_t *>(reinterpret_cast<unsigned char *>(scratch) +
                                              term_bytes + psum_bytes);
    w.out = nullptr;
    w.accumulate = 0;
    e = stream_detail::kStreamTable[D](w, device, stream);
    if (e == cudaSuccess) {
        // TS_FOLD_FAST=0: always the tree-order chain (A/B experiments, tests)
        const char *ff = getenv("TS_FOLD_FAST");
        const int no_fast = ff && atoi(ff) == 0 ? 1 : 0;
        k_fold<<<(unsigned)blocks, 256, 0, stream>>>(scratch, T, a.accumulate, a.out, a.n,
                                                     w.part_sum, w.part_key, splits, no_fast);
        count_launch();
        e = cudaGetLastError();
    }
    cudaError_t f = cudaFreeAsync(scratch, stream);
    if (xcopy) {
        const cudaError_t g = cudaFreeAsync(xcopy, stream);
        if (f == cudaSuccess) f = g;
    }
    return e != cudaSuccess ? e : f;
}

}  // namespace ts
