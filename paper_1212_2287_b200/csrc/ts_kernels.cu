// ts_kernels.cu -- predicated tree-ensemble traversal for sm_100a.
//
// Replaces the reference's lockstep batch kernel (ref evaluators.py:90-99,
// `i = (i << 1) + 1 + (V[rows, fids[i]] >= thetas[i])` unrolled per depth and
// dispatched per depth, :102-119) and the f64 leaf-sum loop
// (ref evaluators.py:527-536).
//
// Work decomposition:
//  * one CTA owns a tile of B = 32*W consecutive instances; it stages their
//    feature rows from HBM and TRANSPOSES them into shared memory as
//    xs[f * B + r] (feature-major).  Lane r of the CTA scores instance r, so
//    every x[fid] read in the hot loop hits bank (r mod 32): conflict-free
//    whatever fid each lane is at.
//  * the CTA walks all trees of the segment in evaluation order; each thread
//    keeps K independent traversal chains in flight (trees t..t+K-1) for
//    latency hiding, then folds their leaves into one f64 accumulator in
//    tree order (acc = acc + w*leaf, __dmul_rn/__dadd_rn: no FMA), which is
//    bit-identical to the reference's numpy f64 accumulation.
//  * node records are read through the read-only L1 path (__ldg); all warps
//    of an SM walk the same few trees at a time, so the tables stream from
//    L2 once per SM per tile pass.
//  * persistent grid: one CTA per SM loops over tiles.
// Built without --use_fast_math: `x >= theta` must see denormals (no FTZ).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ts_internal.h"

namespace ts {
namespace {

constexpr int K = 4;           // traversal chains in flight per thread
constexpr int kMaxWarps = 16;  // 512 threads

__device__ __forceinline__ bool finite_f(float v) { return fabsf(v) <= 3.402823466e38f; }

// Stage rows [row0, row0 + B) into xs[f * B + r]; row F (sentinel) = -inf.
__device__ __forceinline__ void stage_tile(const ScoreArgs &a, float *xs, long long row0,
                                           int B, bool sentinel) {
    const int r = threadIdx.x;
    const long long row = row0 + r;
    const bool valid = row < a.n;
    const float *xrow = a.x + (valid ? row : 0) * a.ld;
    bool bad = false;
    const int F = a.F;
    const bool vec = ((F & 3) == 0) && ((a.ld & 3) == 0) &&
                     ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
    if (vec) {
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
                float *dst = xs + (size_t)(c + 4 * u) * B + r;
                dst[0] = v[u].x;
                dst[B] = v[u].y;
                dst[2 * B] = v[u].z;
                dst[3 * B] = v[u].w;
            }
        }
        for (; c < F; c += 4) {
            float4 v = valid ? __ldg(x4 + (c >> 2)) : make_float4(0.f, 0.f, 0.f, 0.f);
            bad |= !(finite_f(v.x) && finite_f(v.y) && finite_f(v.z) && finite_f(v.w));
            float *dst = xs + (size_t)c * B + r;
            dst[0] = v.x;
            dst[B] = v.y;
            dst[2 * B] = v.z;
            dst[3 * B] = v.w;
        }
    } else {
        for (int c = 0; c < F; c++) {
            float v = valid ? __ldg(xrow + c) : 0.f;
            bad |= !finite_f(v);
            xs[(size_t)c * B + r] = v;
        }
    }
    if (sentinel) xs[(size_t)F * B + r] = -INFINITY;
    if (bad && a.status) atomicOr(a.status, 1);
}

// Complete (implicit heap) segment: every tree has depth D.
template <int D, bool XG>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) k_complete(ScoreArgs a) {
    extern __shared__ float xs[];
    const int B = blockDim.x;
    const int r = threadIdx.x;
    const long long ntiles = (a.n + B - 1) / B;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long row = tile * B + r;
        const bool valid = row < a.n;
        const float *xr;
        int xstride;
        if (XG) {
            xr = a.x + (valid ? row : 0) * a.ld;
            xstride = 1;
            if (valid && a.status) {
                bool bad = false;
                for (int c = 0; c < a.F; c++) bad |= !finite_f(__ldg(xr + c));
                if (bad) atomicOr(a.status, 1);
            }
        } else {
            stage_tile(a, xs, tile * B, B, false);
            __syncthreads();
            xr = xs + r;
            xstride = B;
        }
        double acc = (a.accumulate && valid) ? a.out[row] : 0.0;
        int t = a.t0;
        for (; t + K <= a.t1; t += K) {
            const uint2 *nd[K];
            uint32_t j[K];
#pragma unroll
            for (int k = 0; k < K; k++) {
                nd[k] = reinterpret_cast<const uint2 *>(a.blob +
                                                        16ull * __ldg(a.tree_off16 + t + k));
                j[k] = 0;
            }
#pragma unroll
            for (int l = 0; l < D; l++) {
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const uint2 q = __ldg(nd[k] + j[k]);
                    const uint32_t fid = q.x >> kFidShift;
                    const float xv = XG ? __ldg(xr + fid) : xr[fid * xstride];
                    j[k] = 2u * j[k] + 1u + (xv >= __uint_as_float(q.y) ? 1u : 0u);
                }
            }
#pragma unroll
            for (int k = 0; k < K; k++) {
                const uint32_t ord = j[k] - ((1u << D) - 1u);
                const float lv = __ldg(reinterpret_cast<const float *>(nd[k] + ((1u << D) - 1u)) + ord);
                acc = a.unit_w ? __dadd_rn(acc, (double)lv)
                               : __dadd_rn(acc, __dmul_rn(__ldg(a.weight + t + k), (double)lv));
                if (a.ord && valid) a.ord[(long long)(t + k) * a.ld_ord + row] = (uint16_t)ord;
            }
        }
        for (; t < a.t1; t++) {
            const uint2 *nd = reinterpret_cast<const uint2 *>(a.blob + 16ull * __ldg(a.tree_off16 + t));
            uint32_t j = 0;
#pragma unroll
            for (int l = 0; l < D; l++) {
                const uint2 q = __ldg(nd + j);
                const uint32_t fid = q.x >> kFidShift;
                const float xv = XG ? __ldg(xr + fid) : xr[fid * xstride];
                j = 2u * j + 1u + (xv >= __uint_as_float(q.y) ? 1u : 0u);
            }
            const uint32_t ord = j - ((1u << D) - 1u);
            const float lv = __ldg(reinterpret_cast<const float *>(nd + ((1u << D) - 1u)) + ord);
            acc = a.unit_w ? __dadd_rn(acc, (double)lv)
                           : __dadd_rn(acc, __dmul_rn(__ldg(a.weight + t), (double)lv));
            if (a.ord && valid) a.ord[(long long)t * a.ld_ord + row] = (uint16_t)ord;
        }
        if (valid) a.out[row] = acc;
        if (!XG) __syncthreads();  // before the next tile overwrites xs
    }
}

// Compact (child-index, self-loop leaves) segment: depths vary per tree; a
// K-group walks max(depth) levels, shorter trees idle on their leaf.
template <bool XG>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) k_compact(ScoreArgs a) {
    extern __shared__ float xs[];
    const int B = blockDim.x;
    const int r = threadIdx.x;
    const long long ntiles = (a.n + B - 1) / B;
    const uint32_t F = (uint32_t)a.F;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long row = tile * B + r;
        const bool valid = row < a.n;
        const float *xr;
        if (XG) {
            xr = a.x + (valid ? row : 0) * a.ld;
            if (valid && a.status) {
                bool bad = false;
                for (int c = 0; c < a.F; c++) bad |= !finite_f(__ldg(xr + c));
                if (bad) atomicOr(a.status, 1);
            }
        } else {
            stage_tile(a, xs, tile * B, B, true);
            __syncthreads();
            xr = xs + r;
        }
        double acc = (a.accumulate && valid) ? a.out[row] : 0.0;
        for (int t = a.t0; t < a.t1; t += K) {
            const int kk = min(K, a.t1 - t);
            const uint2 *nd[K];
            uint32_t j[K], ob[K];
            int dk[K];
            int dmax = 0;
#pragma unroll
            for (int k = 0; k < K; k++) {
                const int tt = k < kk ? t + k : t;
                nd[k] = reinterpret_cast<const uint2 *>(a.blob + 16ull * __ldg(a.tree_off16 + tt));
                dk[k] = __ldg(a.depth + tt);
                dmax = max(dmax, dk[k]);
                j[k] = 0;
                ob[k] = 0;
            }
#pragma unroll 1
            for (int l = 0; l < dmax; l++) {
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const uint2 q = __ldg(nd[k] + j[k]);
                    const uint32_t fid = q.x & 0xffffu;
                    float xv;
                    if (XG) xv = fid < F ? __ldg(xr + fid) : -INFINITY;
                    else xv = xr[fid * (uint32_t)B];
                    const uint32_t c = xv >= __uint_as_float(q.y) ? 1u : 0u;
                    j[k] = (q.x >> 16) + c;
                    ob[k] = 2u * ob[k] + c;
                }
            }
#pragma unroll
            for (int k = 0; k < K; k++) {
                if (k < kk) {
                    const float lv = __uint_as_float(__ldg(nd[k] + j[k]).y);
                    acc = a.unit_w
                              ? __dadd_rn(acc, (double)lv)
                              : __dadd_rn(acc, __dmul_rn(__ldg(a.weight + t + k), (double)lv));
                    if (a.ord && valid)
                        a.ord[(long long)(t + k) * a.ld_ord + row] =
                            (uint16_t)(ob[k] >> (dmax - dk[k]));
                }
            }
        }
        if (valid) a.out[row] = acc;
        if (!XG) __syncthreads();
    }
}

template <typename Kern>
cudaError_t launch(Kern kern, const ScoreArgs &a, int device, size_t smem, int threads,
                   cudaStream_t stream) {
    const int sms = dev_attrs(device).sms;
    cudaError_t e;
    if (smem > 48 * 1024) {
        e = ensure_smem((const void *)kern, smem);
        if (e != cudaSuccess) return e;
    }
    const long long tiles = (a.n + threads - 1) / threads;
    const int grid = (int)(tiles < sms ? tiles : sms);
    kern<<<grid, threads, smem, stream>>>(a);
    count_launch();
    return cudaGetLastError();
}

template <int D>
cudaError_t launch_complete(const ScoreArgs &a, int device, bool xg, size_t smem, int threads,
                            cudaStream_t s) {
    return xg ? launch(k_complete<D, true>, a, device, 0, threads, s)
              : launch(k_complete<D, false>, a, device, smem, threads, s);
}

using LaunchFn = cudaError_t (*)(const ScoreArgs &, int, bool, size_t, int, cudaStream_t);
const LaunchFn kCompleteTable[TS_MAX_DEPTH + 1] = {
    launch_complete<0>,  launch_complete<1>,  launch_complete<2>,  launch_complete<3>,
    launch_complete<4>,  launch_complete<5>,  launch_complete<6>,  launch_complete<7>,
    launch_complete<8>,  launch_complete<9>,  launch_complete<10>, launch_complete<11>,
    launch_complete<12>, launch_complete<13>, launch_complete<14>, launch_complete<15>,
    launch_complete<16>};

}  // namespace

cudaError_t x_device_copy(const float *x, long long n, long long ld, int device,
                          cudaStream_t stream, float **dst) {
    *dst = nullptr;
    cudaMemPool_t pool = scratch_pool(device);
    if (!pool) return cudaSuccess;
    const size_t bytes = (size_t)n * ld * sizeof(float);
    cudaError_t e = cudaMallocFromPoolAsync((void **)dst, bytes, pool, stream);
    if (e != cudaSuccess) {
        *dst = nullptr;
        return e;
    }
    e = cudaMemcpyAsync(*dst, x, bytes, cudaMemcpyDefault, stream);
    if (e != cudaSuccess) {
        cudaFreeAsync(*dst, stream);
        *dst = nullptr;
    }
    return e;
}

cudaError_t launch_segment(const Segment &seg, const ScoreArgs &args0, int device,
                           cudaStream_t stream) {
    if (args0.n <= 0) return cudaSuccess;
    if (seg.layout == kRank) return launch_rank_segment(seg, args0, device, stream);
    if (args0.x_mapped && seg.layout != kSplit) {
        // the irregular and L1-path kernels may read a row more than once
        // (tree splits, per-visit global loads): score from a device copy
        float *xd = nullptr;
        cudaError_t e = x_device_copy(args0.x, args0.n, args0.ld, device, stream, &xd);
        if (e != cudaSuccess) return e;
        ScoreArgs a2 = args0;
        a2.x_mapped = 0;
        if (xd) a2.x = xd;
        e = launch_segment(seg, a2, device, stream);
        if (xd) {
            const cudaError_t f = cudaFreeAsync(xd, stream);
            if (e == cudaSuccess) e = f;
        }
        return e;
    }
    const ScoreArgs &args = args0;
    if (seg.layout == kCStream) {
        CStreamArgs ca{};
        // the records encode x-tile offsets for the tile planned at pack time
        if (!plan_cstream(args.F, device, &ca) || ca.B != seg.cs_b)
            return cudaErrorInvalidConfiguration;
        ca.x = args.x;
        ca.n = args.n;
        ca.ld = args.ld;
        ca.F = args.F;
        ca.blob = args.blob;
        ca.chunk_info = args.tables->chunk_info;
        ca.slot_meta = args.tables->slot_meta;
        ca.chunk0 = seg.chunk0;
        ca.nchunks = seg.nchunks;
        ca.weight = args.weight;
        ca.unit_w = args.unit_w;
        ca.accumulate = args.accumulate;
        ca.out = args.out;
        ca.ord = args.ord;
        ca.ld_ord = args.ld_ord;
        ca.status = args.status;
        // Balanced tree split (ts_stream.cu launch_balanced, same scheme): one
        // CTA walks a 32..256-row tile over ALL trees, so any batch up to one
        // wave of tiles costs the whole ensemble's walk (config 3's 5000
        // trees: 135 us from 1 to 4000 rows).  Unit weights, no ordinals; a
        // somewhat larger share of rows may take k_combine's second walk
        // than for complete trees (the alternative is that much slower).
        const int sms = dev_attrs(device).sms;
        const long long tiles = (args.n + ca.B - 1) / ca.B;
        const int T = args.t1 - args.t0;
        const char *ske = getenv("TS_SK");
        bool sk = args.unit_w && !args.ord && seg.slow_rows <= 2e-2f &&
                  balanced_split_trusted(args.tables) &&
                  balanced_split_pays(seg.depth, T, tiles, sms, false, 16384) &&
                  (tiles > sms || 10 * tiles <= 7 * sms);  // a first wave filled > 0.7 measured no gain (4000 rows: 135 -> 142 us)
        if (ske) sk = atoi(ske) != 0 && args.unit_w && !args.ord;
        const long long W = tiles * ca.nchunks;
        long long ctas = std::min<long long>(sms, W);
        if (const char *ce = getenv("TS_SK_CTAS")) ctas = std::min<long long>(std::max(1, atoi(ce)), W);
        cudaMemPool_t pool = scratch_pool(device);
        unsigned char *scratch = nullptr;
        size_t psum_bytes = 0;
        int slices = 0;
        if (sk && pool && (ctas > tiles || tiles % ctas != 0)) {
            slices = (int)((ctas + tiles - 1) / tiles) + 1;
            psum_bytes = (size_t)tiles * slices * ca.B * sizeof(double);
            if (cudaMallocFromPoolAsync((void **)&scratch, 2 * psum_bytes, pool, stream) != cudaSuccess) {
                (void)cudaGetLastError();
                scratch = nullptr;  // whole tiles instead
            }
        }
        if (!scratch) return launch_cstream(ca, device, stream);
        ca.sk_ctas = (int)ctas;
        ca.sk_slices = slices;
        ca.part_sum = reinterpret_cast<double *>(scratch);
        ca.part_key = reinterpret_cast<uint32_t *>(scratch + psum_bytes);
        cudaError_t e = launch_cstream(ca, device, stream);
        if (e == cudaSuccess) {
            LeafWalk g{};
            g.rank = 2;
            g.x = args.x;
            g.ld = args.ld;
            g.F = args.F;
            g.seg = args.blob;
            g.tree_off16 = args.tree_off16 + args.t0;
            int xs = 0;  // records hold fid * 4 B: B = 32 G, a power of two
            while ((1 << xs) < 4 * ca.B) xs++;
            g.xshift = xs;
            g.slow_dev = args.tables->slow_dev;
            g.slow_seen_dev = args.tables->slow_seen_dev;
            e = launch_combine(ca.part_sum, ca.part_key, slices, ca.B, tiles, ca.nchunks, (int)ctas, T,
                               args.accumulate, args.out, args.n, g, stream);
        }
        const cudaError_t f = cudaFreeAsync(scratch, stream);
        return e != cudaSuccess ? e : f;
    }
    if (seg.layout == kSplit) {
        StreamArgs sa{};
        if (plan_stream(args.F, seg.depth, device, &sa, args.n)) {
            sa.x = args.x;
            sa.n = args.n;
            sa.ld = args.ld;
            sa.F = args.F;
            sa.blob = args.blob;
            sa.seg_byte0 = seg.byte0;
            sa.slow_rows = seg.slow_rows;
            sa.tables = args.tables;
            sa.weight = args.weight;
            sa.t0 = args.t0;
            sa.t1 = args.t1;
            sa.unit_w = args.unit_w;
            sa.accumulate = args.accumulate;
            sa.out = args.out;
            sa.ord = args.ord;
            sa.ld_ord = args.ld_ord;
            sa.status = args.status;
            sa.pipe = args.pipe;
            sa.x_mapped = args.x_mapped;
            return launch_stream(seg.depth, sa, device, stream);
        }
        return cudaErrorInvalidConfiguration;  // packed for a device it does not fit
    }
    const int optin = dev_attrs(device).smem_optin;
    const int rows_per_feature = args.F + (seg.layout == kCompact ? 1 : 0);
    const size_t warp_bytes = (size_t)32 * rows_per_feature * sizeof(float);
    int warps = (int)(optin / warp_bytes);
    const bool xg = warps < 1;  // feature rows too wide for a shared-memory tile
    if (warps > kMaxWarps) warps = kMaxWarps;
    if (xg) warps = 8;
    const int threads = warps * 32;
    const size_t smem = xg ? 0 : (size_t)warps * warp_bytes;
    if (seg.layout == kComplete)
        return kCompleteTable[seg.depth](args, device, xg, smem, threads, stream);
    return xg ? launch(k_compact<true>, args, device, 0, threads, stream)
              : launch(k_compact<false>, args, device, smem, threads, stream);
}

}  // namespace ts
