// ts_rank.cu -- planning and launch of the rank kernels (kRank segments):
// the instance-rank pre-pass k_rank and the walk k_rstream
// (ts_rank_kernel.cuh, which explains the rank form and why it is exact).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "ts_internal.h"
#include "ts_rank_kernel.cuh"

namespace ts {
namespace rank_detail {
#define TS_RANK_EXTERN(D) \
    extern template cudaError_t launch_rank_d<D>(const RankArgs &, int, int, cudaStream_t);
TS_RANK_EXTERN(1) TS_RANK_EXTERN(2) TS_RANK_EXTERN(3) TS_RANK_EXTERN(4) TS_RANK_EXTERN(5)
TS_RANK_EXTERN(6) TS_RANK_EXTERN(7) TS_RANK_EXTERN(8) TS_RANK_EXTERN(9) TS_RANK_EXTERN(10)
TS_RANK_EXTERN(11) TS_RANK_EXTERN(12) TS_RANK_EXTERN(13) TS_RANK_EXTERN(14)
#undef TS_RANK_EXTERN

using RankFn = cudaError_t (*)(const RankArgs &, int, int, cudaStream_t);
const RankFn kRankTable[kRankMaxDepth + 1] = {
    nullptr,           launch_rank_d<1>,  launch_rank_d<2>,  launch_rank_d<3>, launch_rank_d<4>,
    launch_rank_d<5>,  launch_rank_d<6>,  launch_rank_d<7>,  launch_rank_d<8>, launch_rank_d<9>,
    launch_rank_d<10>, launch_rank_d<11>, launch_rank_d<12>, launch_rank_d<13>,
    launch_rank_d<14>};

// ---------------------------------------------------------------------------
// Pre-pass: instance ranks.  Block (feature group g, slice s): the group's
// Eytzinger trees e[eoff[f0] .. eoff[f1]) (RankSpace) are one contiguous
// run, loaded into shared memory once (bulk copies); then, for tiles s,
// s + slices, ... kRows at a time, thread r ranks rows r, r + 256, ... for
// every feature of the group: kRows independent L-step heap walks in flight
// (i = 2i + 1 + (e[i] <= v); rank = i - (2^L - 1)).
constexpr int kRows = 8;
struct RankPrepArgs {
    const float *x;
    long long n, ld;
    int F;
    const float *e;
    const uint32_t *eoff;
    const int2 *groups;
    uint16_t *R;
    int32_t *status;
    long long tiles;
};

__global__ void __launch_bounds__(256) k_rank(RankPrepArgs a) {
    extern __shared__ __align__(16) float se[];
    __shared__ __align__(8) uint64_t bar;
    const int2 gr = a.groups[blockIdx.x];
    const uint32_t ebase = a.eoff[gr.x], eend = a.eoff[gr.y];
    const uint32_t lead = ebase & 3u;  // bulk copies move 16-byte granules
    const uint32_t words = (lead + (eend - ebase) + 3u) & ~3u;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(&bar, words * 4u);
        for (uint32_t o = 0; o < words; o += 8192)  // <= 32 KB per bulk copy
            bulk_g2s(se + o, a.e + (ebase - lead) + o, min(8192u, words - o) * 4u, &bar);
    }
    mbar_wait(&bar, 0);
    const uint32_t e0 = su32(se) + 4u * lead;
    const int r = threadIdx.x;
    const int nf_g = gr.y - gr.x;
    // (tile block, feature) pairs in order; the next pair's values are loaded
    // while the current pair is searched (the strided global loads' latency
    // stays off the critical path)
    const long long tstep = (long long)kRows * gridDim.y;
    long long tq = (long long)kRows * blockIdx.y;
    int f = gr.x;
    bool bad = false;
    float v[kRows];
    auto load = [&](long long tq_, int f_, float *dst) {
#pragma unroll
        for (int q = 0; q < kRows; q++) {
            const long long row = (tq_ + q) * kRankB + r;
            const bool ok = tq_ + q < a.tiles && row < a.n;
            dst[q] = ok ? __ldg(a.x + row * a.ld + f_) : 0.f;
        }
    };
    if (tq < a.tiles) load(tq, f, v);
    while (tq < a.tiles) {
        long long tq2 = tq;
        int f2 = f + 1;
        if (f2 == gr.y) {
            f2 = gr.x;
            tq2 += tstep;
        }
        float vn[kRows];
        if (tq2 < a.tiles) load(tq2, f2, vn);
        const uint32_t eb = e0 + 4u * (a.eoff[f] - ebase);
        const uint32_t nf = a.eoff[f + 1] - a.eoff[f];  // 2^L - 1
        uint32_t i[kRows];
#pragma unroll
        for (int q = 0; q < kRows; q++) i[q] = 0;
        for (uint32_t lvl = nf; lvl; lvl >>= 1) {  // L iterations
#pragma unroll
            for (int q = 0; q < kRows; q++) {
                float u;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(u) : "r"(eb + 4u * i[q]));
                i[q] = 2u * i[q] + (u <= v[q] ? 2u : 1u);
            }
        }
#pragma unroll
        for (int q = 0; q < kRows; q++) {
            if (tq + q < a.tiles) {
                a.R[((tq + q) * a.F + f) * kRankB + rank_slot((uint32_t)r)] = (uint16_t)(i[q] - nf);
                bad |= (tq + q) * kRankB + r < a.n && !finite_f(v[q]);
            }
            v[q] = vn[q];
        }
        tq = tq2;
        f = f2;
        (void)nf_g;
    }
    if (bad && a.status) atomicOr(a.status, 1);
}

// Shared-memory plan of the walk: the 256-row u16 rank tile plus a ring of
// 2-4 stages of whole K-groups (the tuned K, else the fallback).
bool plan_rank(int F, int D, int device, RankArgs *a, int *k) {
    if (D < 1 || D > kRankMaxDepth || F > 256) return false;
    const int optin = dev_attrs(device).smem_optin;
    if (!optin) return false;
    const size_t xs = ((size_t)F * kRankB * 2 + 127) & ~(size_t)127;
    const size_t bars = 2 * kRankMaxStages * 8;
    const uint32_t tb = rank_ring_bytes(D);
    if (xs + bars + 2 * (size_t)tb > (size_t)optin) return false;
    const size_t ring = (size_t)optin - xs - bars;
    const int cands[2] = {rank_chains(D), rank_chains_fallback(D)};
    for (int K : cands) {
        const size_t group = (size_t)K * tb;
        for (int s = kRankMaxStages; s >= 2; s--) {
            const size_t cap = ring / s;
            if (cap < group) continue;
            size_t g = cap / group;
            const size_t soft = 48 * 1024;  // small chunks keep the ring turning over
            if (g > 1 && g * group > soft) g = std::max<size_t>(1, soft / group);
            const RankGeom geo = rank_geom(D);
            a->F = F;
            a->tree_bytes = geo.bytes;
            a->ring_tree_bytes = tb;
            a->leaf0 = geo.leaf0;
            a->tpc = (int)(g * K);
            a->chunk_cap = ((uint32_t)(g * K) * tb + 15u) & ~15u;
            a->stages = s;
            a->xs_bytes = (uint32_t)xs;
            *k = K;
            return true;
        }
    }
    return false;
}

}  // namespace rank_detail

bool rank_plan_ok(int F, int D, int device) {
    rank_detail::RankArgs a{};
    int k = 0;
    return rank_detail::plan_rank(F, D, device, &a, &k);
}

// One kRank segment: instance ranks into pool scratch (k_rank), then the
// walk (k_rstream), then the scratch goes back to the pool -- all
// stream-ordered.  Mapped host rows are fine here: the pre-pass reads each
// value once per feature group.
namespace {
cudaError_t rank_chunk(const Segment &seg, const ScoreArgs &args, int device,
                       cudaStream_t stream);
}  // namespace

// Rows go through in chunks of <= kRankChunkRows (the rank scratch stays
// <= ~0.6 GB at F = 136, within what the pool keeps cached between calls);
// rows in mapped host memory (ts_score_host's small
// batches) are first copied to the device -- the pre-pass reads every row
// once per feature group, which over PCIe would cost far more than one copy.
constexpr long long kRankChunkRows = 2ll << 20;
cudaError_t launch_rank_segment(const Segment &seg, const ScoreArgs &args0, int device,
                                cudaStream_t stream) {
    if (args0.n <= 0) return cudaSuccess;
    ScoreArgs args = args0;
    float *xd = nullptr;
    if (args.x_mapped) {
        cudaError_t e = x_device_copy(args.x, args.n, args.ld, device, stream, &xd);
        if (e != cudaSuccess) return e;
        if (xd) args.x = xd;
        args.x_mapped = 0;
    }
    cudaError_t e = cudaSuccess;
    for (long long r0 = 0; r0 < args.n && e == cudaSuccess; r0 += kRankChunkRows) {
        ScoreArgs c = args;
        c.n = std::min(kRankChunkRows, args.n - r0);
        c.x = args.x + r0 * args.ld;
        c.out = args.out ? args.out + r0 : nullptr;
        c.ord = args.ord ? args.ord + r0 : nullptr;  // row offset; ld_ord unchanged
        e = rank_chunk(seg, c, device, stream);
    }
    if (xd) {
        const cudaError_t f = cudaFreeAsync(xd, stream);
        if (e == cudaSuccess) e = f;
    }
    return e;
}

namespace {
cudaError_t rank_chunk(const Segment &seg, const ScoreArgs &args, int device,
                       cudaStream_t stream) {
    using namespace rank_detail;
    const DeviceTables &dt = *args.tables;
    if (seg.rank_space < 0 || (size_t)seg.rank_space >= dt.rank_spaces.size())
        return cudaErrorInvalidConfiguration;
    const RankSpace &tb = dt.rank_spaces[seg.rank_space];
    if (!tb.e || tb.ngroups < 1) return cudaErrorInvalidConfiguration;
    RankArgs a{};
    int K = 0;
    if (!plan_rank(args.F, seg.depth, device, &a, &K)) return cudaErrorInvalidConfiguration;
    cudaMemPool_t pool = scratch_pool(device);
    if (!pool) return cudaErrorNotSupported;
    const long long tiles = (args.n + kRankB - 1) / kRankB;
    const size_t rbytes = (size_t)tiles * args.F * kRankB * sizeof(uint16_t);
    uint16_t *R = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync((void **)&R, rbytes, pool, stream);
    if (e != cudaSuccess) return e;
    {
        RankPrepArgs p{};
        p.x = args.x;
        p.n = args.n;
        p.ld = args.ld;
        p.F = args.F;
        p.e = tb.e;
        p.eoff = tb.eoff;
        p.groups = tb.groups;
        p.R = R;
        p.status = args.status;
        p.tiles = tiles;
        const size_t smem = std::max<size_t>(16, (size_t)tb.group_words * 4);
        e = ensure_smem((const void *)k_rank, smem);
        if (e == cudaSuccess) {
            const int sms = dev_attrs(device).sms;
            const long long blocks = (tiles + kRows - 1) / kRows;
            const int slices = (int)std::max<long long>(
                1, std::min<long long>(blocks, (2LL * sms + tb.ngroups - 1) / tb.ngroups));
            k_rank<<<dim3((unsigned)tb.ngroups, (unsigned)slices), 256, smem, stream>>>(p);
            count_launch();
            e = cudaGetLastError();
        }
    }
    if (e == cudaSuccess) {
        a.R = R;
        a.n = args.n;
        a.blob = args.blob;
        a.seg_byte0 = seg.byte0;
        a.weight = args.weight;
        a.t0 = args.t0;
        a.t1 = args.t1;
        a.unit_w = args.unit_w;
        a.accumulate = args.accumulate;
        a.out = args.out;
        a.ord = args.ord;
        a.ld_ord = args.ld_ord;
        // Balanced tree split (ts_stream.cu launch_balanced; the rank walk has
        // no other small-batch path: a 256-row tile is walked by one CTA over
        // all trees, so d=12 T=1000 cost ~250 us for ANY batch up to 30k
        // rows).  Unit weights, no ordinals, few rows whose sums may round.
        const int sms = dev_attrs(device).sms;
        const int T = args.t1 - args.t0;
        const int nchunks = (T + a.tpc - 1) / a.tpc;
        const char *ske = getenv("TS_SK");
        bool sk = args.unit_w && !args.ord && seg.slow_rows <= 1e-3f &&
                  balanced_split_trusted(args.tables) &&
                  balanced_split_pays(seg.depth, T, tiles, sms, false);
        if (ske) sk = atoi(ske) != 0 && args.unit_w && !args.ord;
        const long long W = tiles * nchunks;
        long long ctas = std::min<long long>(sms, W);
        if (const char *ce = getenv("TS_SK_CTAS")) ctas = std::min<long long>(std::max(1, atoi(ce)), W);
        unsigned char *scratch = nullptr;
        size_t psum_bytes = 0;
        int slices = 0;
        if (sk && (ctas > tiles || tiles % ctas != 0)) {
            slices = (int)((ctas + tiles - 1) / tiles) + 1;
            psum_bytes = (size_t)tiles * slices * kRankB * sizeof(double);
            if (cudaMallocFromPoolAsync((void **)&scratch, 2 * psum_bytes, pool, stream) != cudaSuccess) {
                (void)cudaGetLastError();
                scratch = nullptr;  // whole tiles instead
            }
        }
        if (scratch) {
            a.sk_ctas = (int)ctas;
            a.sk_slices = slices;
            a.part_sum = reinterpret_cast<double *>(scratch);
            a.part_key = reinterpret_cast<uint32_t *>(scratch + psum_bytes);
        }
        e = kRankTable[seg.depth](a, K, device, stream);
        if (scratch) {
            if (e == cudaSuccess) {
                LeafWalk g{};
                g.rank = 1;
                g.D = seg.depth;
                g.leaf0 = a.leaf0;
                g.tree_bytes = a.tree_bytes;
                g.R = R;
                g.F = args.F;
                g.seg = args.blob + seg.byte0;
                g.slow_dev = dt.slow_dev;
                g.slow_seen_dev = dt.slow_seen_dev;
                e = launch_combine(a.part_sum, a.part_key, slices, kRankB, tiles, nchunks, (int)ctas,
                                   T, args.accumulate, args.out, args.n, g, stream);
            }
            const cudaError_t f2 = cudaFreeAsync(scratch, stream);
            if (e == cudaSuccess) e = f2;
        }
    }
    const cudaError_t f = cudaFreeAsync(R, stream);
    return e != cudaSuccess ? e : f;
}
}  // namespace

}  // namespace ts
