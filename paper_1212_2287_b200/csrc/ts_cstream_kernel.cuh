#pragma once
// ts_cstream_kernel.cuh -- streaming kernel for IRREGULAR trees (BASELINE
// config 3: LambdaMART-shaped trees of <= 64 leaves and depth <= 16 over
// F = 700 features).  Complete expansion would cost 2^16 slots per tree, so
// these trees keep their own nodes (kCStream records, ts_internal.h) and are
// streamed through shared memory by TMA exactly like ts_stream_kernel.cuh.
// Planning and dispatch: ts_cstream.cu; instantiations: ts_cstream_w*.cu.
//
// What differs from the complete-tree kernel:
//  * wide feature rows leave room for only B = 32*G instances (G instance
//    groups of 32), so the W walker warps split the TREES of each chunk as
//    well: warp w walks instance group w % G over K-groups of K consecutive
//    tree slots, S = W / G warps per instance group (W = 16 walkers when the
//    x tile is small enough to leave room for the wider ring: more chains in
//    flight);
//  * inside a chunk the packer orders tree slots by depth, so the K trees a
//    thread walks in lockstep have nearly equal depth (a K-group steps
//    max(depth) times; a leaf is a self-loop whose x row is the -inf sentinel
//    row F, so shorter trees idle on their leaf);
//  * each walk writes its leaf value to a double-buffered shared leaf buffer
//    lb[tree][inst]; a dedicated accumulator warp folds each chunk's leaves
//    into the f64 sums in TREE order (acc = acc + w * leaf, __dmul_rn /
//    __dadd_rn), so the result stays bit-identical to the reference's
//    sequential sum (ref evaluators.py:529-535) whatever order the walks ran
//    in; walkers and accumulator hand buffers over with mbarriers.
// The per-level step is the reference predicate (ref evaluators.py:90-99)
// on child-index records rec = {xoff << 14 | left, theta} with xoff = fid*4B
// the feature's byte offset in the x tile (the packer knows B) and left the
// left child's record index:
//     v = xs[xr + (rec.x >> 14)]            LEA.HI + LDS
//     p = (v >= theta ? tree + 8 : tree) + 8 * (rec.x & 0x3fff)   SEL, LOP3, LEA
#include "ts_stream_kernel.cuh"

namespace ts {
namespace cstream_detail {

using namespace stream_detail;

constexpr int kMaxStagesC = 4;
constexpr uint32_t kMetaBytes = kCStreamMaxT * 4;  // slot table at the head of a stage
constexpr uint32_t kHeadBytes = kMetaBytes + 16;   // + the chunk's chunk_info entry
__host__ __device__ constexpr int threads_c(int W) { return 32 * W + 64; }

// Stage B rows x F features into xs[f * B + r] (+ sentinel row F = -inf),
// all walker threads cooperating.
template <int NT, int B>
__device__ __forceinline__ void stage_rows_c(const CStreamArgs &a, float *xs, long long row0) {
    const int F = a.F;
    const int tid = threadIdx.x;
    bool bad = false;
    const bool vec = ((F & 3) == 0) && ((a.ld & 3) == 0) &&
                     ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
    if (vec) {
        const int F4 = F >> 2;
        constexpr int U = 8;  // independent loads in flight per thread
        for (int e0 = tid; e0 < B * F4; e0 += U * NT) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int e = e0 + u * NT;
                const int r = e % B, c4 = e / B;
                const long long row = row0 + r;
                v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (e < B * F4 && row < a.n)
                    v[u] = __ldg(reinterpret_cast<const float4 *>(a.x + row * a.ld) + c4);
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int e = e0 + u * NT;
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
        for (int e = tid; e < B * F; e += NT) {
            const int r = e % B, c = e / B;
            const long long row = row0 + r;
            float v = row < a.n ? __ldg(a.x + row * a.ld + c) : 0.f;
            bad |= !finite_f(v);
            xs[c * B + r] = v;
        }
    }
    for (int r = tid; r < B; r += NT) xs[F * B + r] = -INFINITY;
    if (bad && a.status) atomicOr(a.status, 1);
}

// base + 8 * (rec & 0x3fff) as LOP3 + LEA (ptxas otherwise emits SHL, LOP3, IADD).
__device__ __forceinline__ uint32_t child_addr(uint32_t rec, uint32_t base) {
    uint32_t r;
    asm("{\n\t.reg .u32 t;\n\tand.b32 t, %1, 0x3fff;\n\tshl.b32 t, t, 3;\n\t"
        "add.u32 %0, t, %2;\n\t}"
        : "=r"(r)
        : "r"(rec), "r"(base));
    return r;
}

// One lockstep step's loads for a chain: the record at p and the lane's
// x value for its feature -- skipped (predicated off, no shared-memory
// wavefront) once the previous record was a leaf: the lane is parked on its
// self-loop leaf and q / v already hold that leaf record and the sentinel's
// -inf, so the step below leaves p unchanged and adds a 0 ordinal bit.
__device__ __forceinline__ void walk_loads(uint2 &q, float &v, uint32_t p, uint32_t xr,
                                           uint32_t leafmark) {
    TS_DBG(p, 8);
    asm volatile(
        "{\n\t.reg .pred live;\n\t.reg .u32 a;\n\t"
        "setp.lt.u32 live, %0, %4;\n\t"
        "@live ld.shared.v2.u32 {%0, %1}, [%3];\n\t"
        "shr.u32 a, %0, 14;\n\t"
        "add.u32 a, a, %5;\n\t"
        "@live ld.shared.f32 %2, [a];\n\t}"
        : "+r"(q.x), "+r"(q.y), "+f"(v)
        : "r"(p), "r"(leafmark), "r"(xr));
}

// SK: balanced tree split (CStreamArgs::sk_ctas; unit weights, no ordinals):
// the CTA walks a run of (tile, chunk) items; the accumulator warp also keeps
// the bookkeeping of ts_stream.cu split_sum_exact and stores a partial for a
// tile it walked only in part.
template <int kK, int G, int W, bool UNIT_W, bool ORD, bool SK = false>
__global__ void __launch_bounds__(threads_c(W), 1) k_cstream(CStreamArgs a) {
    // G (instance groups of 32, B = 32 * G) is a template parameter so the
    // accumulator's per-lane instance loop is fully unrolled with exactly G
    // independent f64 chains.
    constexpr int kConsumers = 32 * W;
    extern __shared__ __align__(128) unsigned char smem[];
    float *xs = reinterpret_cast<float *>(smem);
    float *lb0 = reinterpret_cast<float *>(smem + a.xs_bytes);  // two leaf buffers
    unsigned char *ring = smem + a.xs_bytes + a.lb_bytes;
    const int nst = a.stages;  // ring stages (2-4)
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + nst * a.stage_bytes);
    uint64_t *empty = full + kMaxStagesC;  // ring stage consumed (W walker warps)
    uint64_t *lbf = empty + kMaxStagesC;   // leaf buffer written (W walker warps)
    uint64_t *lbe = lbf + 2;            // leaf buffer folded (accumulator warp)
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; s++) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, W);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(lbf + b, W);
            mbar_init(lbe + b, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    constexpr int B = 32 * G;
    const long long ntiles = (a.n + B - 1) / B;
    const uint32_t lb_half = a.lb_bytes / 2;
    // Spans (a tile and the chunk range [cb, ce) walked of it) of this CTA:
    // tiles blockIdx.x, +gridDim.x, ... whole, or (SK) an equal run of the
    // tile-major (tile, chunk) items.  Every role iterates the same spans.
    struct Span {
        long long tile, pos, end;
        int cb, ce;
    };
    auto span_load = [&](Span &sp) -> bool {
        if (sp.pos >= sp.end) return false;
        if (SK) {
            sp.tile = sp.pos / a.nchunks;
            sp.cb = (int)(sp.pos - sp.tile * a.nchunks);
            sp.ce = (int)min((long long)a.nchunks, sp.cb + (sp.end - sp.pos));
        } else {
            sp.tile = sp.pos;
            sp.cb = 0;
            sp.ce = a.nchunks;
        }
        return true;
    };
    auto span_first = [&](Span &sp) -> bool {
        if (SK) {
            const long long Wk = ntiles * a.nchunks;
            sp.pos = (long long)blockIdx.x * Wk / a.sk_ctas;
            sp.end = (long long)(blockIdx.x + 1) * Wk / a.sk_ctas;
        } else {
            sp.pos = blockIdx.x;
            sp.end = ntiles;
        }
        return span_load(sp);
    };
    auto span_next = [&](Span &sp) -> bool {
        sp.pos += SK ? (long long)(sp.ce - sp.cb) : (long long)gridDim.x;
        return span_load(sp);
    };

    if (warp == W + 1) {  // ---- producer: TMA bulk copies per chunk
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0, used = 0;  // phase of stage s's next reuse; first lap done?
            Span sp;
            for (bool more = span_first(sp); more; more = span_next(sp)) {
                for (int c = sp.cb; c < sp.ce; c++) {
                    if (used) mbar_wait(empty + s, ph);
                    const uint4 ci = __ldg(a.chunk_info + a.chunk0 + c);
                    unsigned char *stage = ring + s * a.stage_bytes;
                    mbar_expect_tx(full + s, ci.y + kMetaBytes + 16);
                    bulk_g2s(stage, a.slot_meta + (size_t)(a.chunk0 + c) * kCStreamMaxT,
                             kMetaBytes, full + s);
                    bulk_g2s(stage + kMetaBytes, a.chunk_info + a.chunk0 + c, 16, full + s);
                    bulk_g2s(stage + kHeadBytes, a.blob + 16ull * ci.x, ci.y, full + s);
                    if (++s == nst) {
                        s = 0;
                        ph ^= used;
                        used = 1;
                    }
                }
            }
        }
        return;
    }

    if (warp == W) {  // ---- accumulator: folds leaves in TREE order
        uint32_t it = 0;
        Span sp;
        for (bool more = span_first(sp); more; more = span_next(sp)) {
            const long long tile = sp.tile;
            const long long row0 = tile * B;
            // SK: a tile walked only in part contributes a partial sum from 0
            const bool part = SK && (sp.cb != 0 || sp.ce != a.nchunks);
            double acc[G];
            uint32_t amax[G], kmin1[G];
#pragma unroll
            for (int g = 0; g < G; g++) {
                const long long row = row0 + g * 32 + lane;
                acc[g] = (a.accumulate && row < a.n && !part) ? a.out[row] : 0.0;
                amax[g] = 0u;
                kmin1[g] = 0xffffffffu;
            }
            for (int c = sp.cb; c < sp.ce; c++, it++) {
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
                        const float lf = lbc[i * B + g * 32 + lane];
                        const double lv = (double)lf;
                        acc[g] = UNIT_W ? __dadd_rn(acc[g], lv) : __dadd_rn(acc[g], __dmul_rn(w, lv));
                        if constexpr (SK) {
                            kmin1[g] = min(kmin1[g], (__float_as_uint(lf) & 0x7fffffffu) - 1u);
                            amax[g] = max(amax[g], (uint32_t)__double2hiint(acc[g]) & 0x7fffffffu);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(lbe + b);
            }
            long long pj0 = 0;
            if (part) {  // slice = this CTA's rank among the CTAs sharing the tile
                const long long Wk = ntiles * a.nchunks;
                const long long b0 = ((tile * a.nchunks + 1) * a.sk_ctas - 1) / Wk;
                pj0 = (tile * a.sk_slices + (blockIdx.x - b0)) * B;
            }
#pragma unroll
            for (int g = 0; g < G; g++) {
                const long long row = row0 + g * 32 + lane;
                if (row >= a.n) continue;
                if (part) {
                    const long long pj = pj0 + g * 32 + lane;
                    a.part_sum[pj] = acc[g];
                    a.part_key[2 * pj] = amax[g];
                    a.part_key[2 * pj + 1] = kmin1[g];
                } else {
                    a.out[row] = acc[g];
                }
            }
        }
        return;
    }

    // ---- walkers (W warps)
    const int grp = warp % G;
    constexpr int S = W / G;
    const int sub = warp / G;
    const int inst = grp * 32 + lane;
    const uint32_t xr = su32(xs) + 4u * inst;
    const uint32_t lbase0 = su32(lb0);
    // records at or above leafmark are leaves (x offset of the sentinel row F)
    const uint32_t leafmark = ((uint32_t)a.F * (uint32_t)(4 * B)) << 14;
    // teams: a.teams (1 or 2) sets of SR = S / teams warps per instance group
    const int team_shift = a.teams == 2 ? 1 : 0;
    const uint32_t team_mask = (uint32_t)a.teams - 1u;
    const int SR = S >> team_shift;
    const int team = sub / SR, sidx = sub % SR;
    int s = 0;
    uint32_t ph = 0;  // parity of stage s's current fill
    uint32_t it = 0;
    Span sp;
    for (bool more = span_first(sp); more; more = span_next(sp)) {
        const long long row0 = sp.tile * B;
        consumer_sync<kConsumers>();  // all walks of the previous tile are done
        stage_rows_c<kConsumers, B>(a, xs, row0);
        consumer_sync<kConsumers>();
        const long long walk_row = row0 + inst;
        const bool walk_valid = walk_row < a.n;
        for (int c = sp.cb; c < sp.ce; c++, it++) {
            const int b = it & 1;
            const uint32_t lbase = lbase0 + b * lb_half;
            mbar_wait(full + s, ph);
            const uint32_t meta = su32(ring + s * a.stage_bytes);
            uint32_t nt, tree0;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(nt), "=r"(tree0)
                         : "r"(meta + kMetaBytes + 8));  // chunk_info .z/.w
            const uint32_t buf = meta + kHeadBytes;
            bool waited = it < 2;  // this leaf buffer's previous fold must be done
            // K-groups of K consecutive (depth-sorted) slots, so a group's
            // trees have nearly equal depth; the group a warp takes rotates
            // with the chunk so no warp always draws the deepest trees.  With
            // two teams (chunks of S*K/2 trees, more ring stages in flight)
            // the teams take alternate chunks.
            const bool mine = (int)(it & team_mask) == team;
            const int rot = (int)((sidx + (it >> team_shift)) & (SR - 1));
            for (int s0 = mine ? rot * kK : (int)nt; s0 < (int)nt; s0 += SR * kK) {
                uint32_t p[kK], tb[kK], tb8[kK], ob[kK], rel[kK];
                uint2 q[kK];
                float v[kK];
                int dk[kK];
                int dmax = 0;
#pragma unroll
                for (int k = 0; k < kK; k++) {
                    const int slot = s0 + k;
                    uint32_t m;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(m)
                                 : "r"(meta + 4u * (slot < (int)nt ? slot : s0)));
                    rel[k] = m >> 21;
                    tb[k] = buf + 8u * (m & 0xffffu);
                    tb8[k] = tb[k] + 8u;
                    p[k] = tb[k];
                    dk[k] = (m >> 16) & 31;
                    dmax = max(dmax, dk[k]);
                    ob[k] = 0;
                    q[k] = make_uint2(0u, 0u);  // "not on a leaf"
                    v[k] = 0.f;
                }
                // Two levels per trip, then leave as soon as every lane of
                // the warp sits on a leaf in all K chains: the rows' paths
                // are much shorter than the trees are deep (config 3: 4.8
                // visits on average in trees 11.6 deep), so the padded
                // levels of a group are mostly skipped.  le = levels walked.
                int le = 0;
#pragma unroll 1
                while (le < dmax) {
#pragma unroll
                    for (int h = 0; h < 2; h++) {
#pragma unroll
                        for (int k = 0; k < kK; k++) {
                            walk_loads(q[k], v[k], p[k], xr, leafmark);
                            const bool c = v[k] >= __uint_as_float(q[k].y);
                            p[k] = child_addr(q[k].x, c ? tb8[k] : tb[k]);
                            if constexpr (ORD) ob[k] = 2u * ob[k] + (c ? 1u : 0u);
                        }
                    }
                    le += 2;
                    uint32_t qmin = q[0].x;
#pragma unroll
                    for (int k = 1; k < kK; k++) qmin = min(qmin, q[k].x);
                    if (!__any_sync(0xffffffffu, qmin < leafmark)) break;
                }
                if (!waited) {
                    mbar_wait(lbe + b, ((it >> 1) - 1) & 1);
                    waited = true;
                }
#pragma unroll
                for (int k = 0; k < kK; k++) {
                    const int slot = s0 + k;
                    if (slot < (int)nt) {
                        const float lv = ldsf(p[k] + 4u);
                        asm volatile("st.shared.f32 [%0], %1;" ::"r"(lbase + 4u * (rel[k] * B + inst)),
                                     "f"(lv));
                        if constexpr (ORD) {
                            if (walk_valid)
                                a.ord[(long long)(tree0 + rel[k]) * a.ld_ord + walk_row] =
                                    (uint16_t)(le >= dk[k] ? ob[k] >> (le - dk[k]) : ob[k] << (dk[k] - le));
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
            if (++s == nst) {
                s = 0;
                ph ^= 1u;
            }
        }
    }
}

inline size_t cstream_smem(const CStreamArgs &a) {
    return (size_t)a.xs_bytes + a.lb_bytes + (size_t)a.stages * a.stage_bytes +
           (2 * kMaxStagesC + 4) * 8;
}

template <int K, int G, int W>
cudaError_t launch_kgw(const CStreamArgs &a, int device, cudaStream_t stream) {
    auto kern = a.sk_ctas > 0 ? k_cstream<K, G, W, true, false, true>  // unit weights, no ordinals
                : a.ord ? (a.unit_w ? k_cstream<K, G, W, true, true> : k_cstream<K, G, W, false, true>)
                        : (a.unit_w ? k_cstream<K, G, W, true, false> : k_cstream<K, G, W, false, false>);
    const size_t smem = cstream_smem(a);
    cudaError_t e = ensure_smem((const void *)kern, smem);
    if (e != cudaSuccess) return e;
    const long long tiles = (a.n + a.B - 1) / a.B;
    const int sms = dev_attrs(device).sms;
    const int grid = a.sk_ctas > 0 ? a.sk_ctas : (int)(tiles < sms ? tiles : sms);
    kern<<<grid, threads_c(W), smem, stream>>>(a);
    count_launch();
    return cudaGetLastError();
}

}  // namespace cstream_detail
}  // namespace ts
