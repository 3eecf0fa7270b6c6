#pragma once
// ts_stream_kernel.cuh -- the main sm_100a traversal kernel: complete trees
// whose node tables are STREAMED through shared memory by the TMA bulk-copy
// engine (planning/dispatch: ts_stream.cu).
//
// Per CTA (persistent over instance tiles; 1 or 2 per SM, see Shape):
//   * CW consumer warps own a tile of B = 32*CW instances, staged from HBM
//     and transposed to xs[f * B + r] (feature-major: lane r's x[fid] reads
//     are bank-conflict-free for any mix of fids);
//   * 1 producer warp streams the segment's packed trees, chunk by chunk, into
//     a 2-4 stage shared-memory ring with cp.async.bulk (TMA, UBLKCP in SASS);
//     full/empty mbarriers hand stages between producer and consumers, so the
//     next chunk (and the next tile's first chunks) land while the current
//     one is walked;
//   * each consumer thread walks K trees of the chunk in lockstep (K
//     independent chains for latency hiding), level by level:
//         levels 0-1 (split_header depths): one 16-byte header (LDS.128)
//         top levels (< kTopLevels): rec = {fid << 10, theta} (LDS.64),
//           v = xs[fid][r] (LDS), heap step j -> 2j + 1 + (v >= theta)
//         deep levels: theta (LDS.32) and fid (LDS.U8/U16) from per-level
//           arrays, same predicate
//     -- the reference's update i = (i<<1)+1+(x[fid[i]] >= theta[i])
//     (ref evaluators.py:90-99) -- then adds w*leaf in f64, tree order
//     (ref evaluators.py:529-535; __dmul_rn/__dadd_rn, never an FMA).
//
// Chunk = `tpc` consecutive trees of one complete segment (all of depth D,
// so every tree record has the same size and chunk c starts at
// c * tpc * tree_bytes).  Record layout: kSplit / split_geom (ts_internal.h);
// trees of depth >= kGLeafDepth stream only their node part and read leaves
// from global memory.
//
// k_stream_ws (below): the same walk for small batches -- 32-row CTAs whose
// four walker warps split each chunk's trees, an accumulator warp folding
// the leaves in tree order; also runs the last partial wave of a large batch.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>

#include "ts_internal.h"

namespace ts {
namespace stream_detail {

// CTA shape: CW consumer warps own a tile of B = 32*CW instances, plus one
// producer warp.  CW = 8: one 256-row CTA per SM; CW = 4: two 128-row CTAs
// per SM, so one CTA's x staging overlaps the other's walks (used when the
// trees are small enough for the halved ring, d <= 9).  (Four 32-row CTAs
// per SM for small batches were tried for config 0 and measured slower.)
template <int CW>
struct Shape {
    static constexpr int kConsumerWarps = CW;
    static constexpr int kB = CW * 32;
    static constexpr int kThreads = kB + 32;
    static constexpr int kCtasPerSm = kB >= 64 ? 256 / kB : 4;
    // Top-level records hold fid << kFidShift = byte offset in a 256-row
    // x tile; smaller tiles shift it down.
    static constexpr int kXShift = kB == 256 ? 0 : kB == 128 ? 1 : kB == 64 ? 2 : 3;
};
constexpr int kB = 256;  // the irregular-tree kernel's consumer count (ts_cstream.cu)
constexpr int kMaxStages = 4;

// Chains per thread by depth: deeper trees are bigger, so fewer fit in a
// ring stage (a K-group must fit one stage).  16 chains for d <= 6 measured
// +4 % on config 2 d = 3/4/6 over 8 (more independent walks to interleave),
// 32 for d <= 3 another +4 % at d = 3 (but -2 % at d = 4).  r1 session-2
// sweep (config 2, 1M rows x 1000 trees): d = 5-6 24 chains +2.2 % over 16
// (d = 4: 24 once the level-0/1 header is on, +1.9 %),
// d = 7 16 chains +8 % over 8; 48 at d = 3, 24 at d = 4 and 9 at d = 9 were
// within 1 % or slower, 64 at d = 3 -29 %.  d = 10: 5 chains
// (two stages of five 9312-byte trees fill the 93120 bytes a 256 x 136 tile
// leaves exactly) measured -8 % time against 4 at F = 100; 6 gained nothing
// more.  d = 8: 9 chains (two stages of nine 2400-byte trees in a 128-row
// CTA's 46 KB ring) +1.5 % over 8 on config 1.  d >= 11 streams only the
// trees' node parts (leaves read from global memory): 4 chains at d = 11, 2
// at d = 12 (was 2 and 1 with whole records; d = 12 16.7 -> 11.5 ms, d = 11
// 8.8 -> 7.1 ms).  Rows too wide for that use chains_fallback(d) (a second
// instantiation picked by the planner).
__host__ __device__ constexpr int chains_for_depth(int d) {
    return d <= 3 ? 32 : d <= 6 ? 24 : d == 7 ? 16 : d == 8 ? 9 : d == 9 ? 8
         : d == 10 ? 5 : d == 11 ? 4 : 2;
}
// The second instantiation per depth, for rows too wide to leave room for two
// stages of the tuned K-group (the chains the r1 session-1 kernel used; a
// plan with room for neither walks single trees).
__host__ __device__ constexpr int chains_fallback(int d) {
    return d <= 3 ? 8 : d == 4 ? 8 : d <= 6 ? 16 : d == 7 ? 8 : d == 8 ? 8 : d == 9 ? 4
         : d == 10 ? 4 : d == 11 ? 2 : 1;
}

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
// try_wait with a suspend-time hint: a waiting warp (the producer waiting for
// a free stage, consumers waiting for data) sleeps until the phase flips
// instead of spinning on issue slots the walking warps need.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(su32(bar)),
        "r"(parity), "r"(1000000u)
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
template <int NT = kB>
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}
__device__ __forceinline__ bool finite_f(float v) { return fabsf(v) <= 3.402823466e38f; }

// Pipeline flags: system-scope acquire/release, written by one GPU and read
// by another over NVLink (ts_score_pipe).  A producer that never publishes
// (its rank died) traps after kPipeTimeoutNs instead of hanging the GPU (the
// launch then fails with cudaErrorLaunchFailure on the host).
constexpr unsigned long long kPipeTimeoutNs = 20ull * 1000 * 1000 * 1000;
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void pipe_wait(const uint32_t *flag, uint32_t epoch) {
    uint32_t v;
    unsigned long long t0 = 0;
    while (true) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (v == epoch) break;
        const unsigned long long t = global_ns();
        if (t0 == 0) t0 = t;
        else if (t - t0 > kPipeTimeoutNs) __trap();
        __nanosleep(256);
    }
}
__device__ __forceinline__ void pipe_signal(uint32_t *flag, uint32_t epoch) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
}

// Transposing stage of B rows into xs[f * B + r] (consumer threads only).
// DEEP: also compile the tree-split modes' 12-wide path (kept out of the plain
// kernels: its 48 live registers change their allocation, +2-3 % at d = 4-10).
template <int B, bool DEEP = false>
__device__ __forceinline__ void stage_rows(const StreamArgs &a, float *xs, long long row0) {
    constexpr int kB = B;
    const int r = threadIdx.x;
    const long long row = row0 + r;
    const bool valid = row < a.n;
    const float *xrow = a.x + (valid ? row : 0) * a.ld;
    const int F = a.F;
    bool bad = false;
    if (((F & 3) == 0) && ((a.ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0)) {
        const float4 *x4 = reinterpret_cast<const float4 *>(xrow);
        int c = 0;
        if (DEEP && (a.splits > 1 || a.sk_ctas > 0)) {
            // tree-split CTAs walk a few trees each, so the staging round
            // trips are their critical path: 12 float4 in flight per thread
            // (a 136-feature row in 3 trips instead of 9)
            constexpr int U = 12;
            const int F4 = F >> 2;
            for (int c0 = 0; c0 < F4; c0 += U) {
                float4 v[U];
#pragma unroll
                for (int u = 0; u < U; u++)
                    v[u] = (valid && c0 + u < F4) ? __ldg(x4 + c0 + u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int u = 0; u < U; u++) {
                    if (c0 + u >= F4) break;
                    bad |= !(finite_f(v[u].x) && finite_f(v[u].y) && finite_f(v[u].z) &&
                             finite_f(v[u].w));
                    float *dst = xs + 4 * (c0 + u) * kB + r;
                    dst[0] = v[u].x;
                    dst[kB] = v[u].y;
                    dst[2 * kB] = v[u].z;
                    dst[3 * kB] = v[u].w;
                }
            }
            c = F;
        }
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

#ifdef TS_DEBUG
// Debug builds (TS_NVCC_EXTRA=-DTS_DEBUG): every shared load of the walk is
// bounds-checked against the CTA's shared allocation and traps (device-side
// assert) on a violation.  compute-sanitizer is unavailable on this pool, so
// this is the memory-safety net for the parity suite.
__device__ __forceinline__ void dbg_check(uint32_t addr, uint32_t width) {
    uint32_t total, dyn;
    asm("mov.u32 %0, %%total_smem_size;" : "=r"(total));
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if (addr + width > total + 1024u || width == 0) {
        printf("ts debug: shared load out of range addr=%u width=%u total=%u dyn=%u\n", addr,
               width, total, dyn);
        __trap();
    }
}
#define TS_DBG(addr, w) dbg_check((addr), (w))
#else
#define TS_DBG(addr, w) ((void)0)
#endif

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
    TS_DBG(addr, 8);
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    TS_DBG(addr, 16);
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr));
    return v;
}
__device__ __forceinline__ float ldsf(uint32_t addr) {
    TS_DBG(addr, 4);
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint32_t ldsu(uint32_t addr, int fw) {
    TS_DBG(addr, fw);
    uint32_t v;
    if (fw == 1) asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    else asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// Compile-time kSplit record geometry (same formulas as split_geom and
// split_ring_bytes).  kRing: a tree's stride in a ring stage.
template <int D, int FW>
struct SplitRec {
    static constexpr uint32_t S = D < kTopLevels ? D : kTopLevels;
    static constexpr uint32_t kThr0 = ((1u << S) - 1u) * 8u;
    static constexpr uint32_t kDeep = (1u << D) - (1u << S);
    static constexpr uint32_t kFid0 = kThr0 + kDeep * 4u;
    static constexpr uint32_t kLeaf0 = (kFid0 + kDeep * FW + 15u) & ~15u;
    static constexpr uint32_t kBytes = (kLeaf0 + (1u << D) * 4u + 15u) & ~15u;
    static constexpr bool kGLeaf = D >= kGLeafDepth;
    static constexpr uint32_t kRing = kGLeaf ? kLeaf0 : kBytes;
};

// Producer: chunk c (`trees` trees from tree a.t0 + c * a.tpc) into a ring
// stage, completing on `bar`.  Whole records in one bulk copy, or for
// global-leaf depths each tree's node part (kRing bytes) on its own.
template <int D, int FW>
__device__ __forceinline__ void produce_chunk(const StreamArgs &a, unsigned char *stage,
                                              uint64_t *bar, int c, int trees) {
    using R = SplitRec<D, FW>;
    const unsigned char *src = a.blob + a.seg_byte0 + (size_t)c * a.tpc * R::kBytes;
    mbar_expect_tx(bar, (uint32_t)trees * R::kRing);
    if constexpr (R::kGLeaf) {
        for (int i = 0; i < trees; i++)
            bulk_g2s(stage + (size_t)i * R::kRing, src + (size_t)i * R::kBytes, R::kRing, bar);
    } else {
        bulk_g2s(stage, src, (uint32_t)trees * R::kBytes, bar);
    }
}

// sel = (v >= th) ? on_ge : on_lt, kept as one FSETP + SEL on registers
// (ptxas otherwise rematerialises the per-chain constants).
__device__ __forceinline__ uint32_t sel_ge(float v, float th, uint32_t on_ge, uint32_t on_lt) {
    uint32_t r;
    asm("{\n\t.reg .pred q;\n\tsetp.ge.f32 q, %1, %2;\n\tselp.u32 %0, %3, %4, q;\n\t}"
        : "=r"(r)
        : "f"(v), "f"(th), "r"(on_ge), "r"(on_lt));
    return r;
}

// Global-leaf depths (kGLeaf): a group's leaf loads go out at the end of its
// walk and are added to acc only after the NEXT group's walk (still in tree
// order), so their L2 latency hides behind shared-memory work.
template <int KP>
struct LeafPend {
    float lv[KP];
    int t = 0, n = 0;  // first tree, count
    // tree-split modes (StreamArgs::part_key): high word of the largest
    // |running sum| this thread reached, and the smallest nonzero |leaf| bit
    // pattern minus 1 among its trees
    uint32_t amax = 0u, kmin1 = 0xffffffffu;
};
template <int D, int FW, bool UNIT_W, int KP>
__device__ __forceinline__ void flush_leaves(LeafPend<KP> &pend, double &acc, const StreamArgs &a) {
#pragma unroll
    for (int j = 0; j < KP; j++) {
        if (j < pend.n) {
            const double term = UNIT_W ? (double)pend.lv[j]
                                       : __dmul_rn(__ldg(a.weight + pend.t + j), (double)pend.lv[j]);
            acc = __dadd_rn(acc, term);
            if (a.leaf_out || a.sk_ctas > 0)
                pend.amax = max(pend.amax, (uint32_t)__double2hiint(acc) & 0x7fffffffu);
        }
    }
    pend.n = 0;
}

// Walk NK consecutive trees of one chunk in lockstep (NK independent chains)
// over the kSplit record (ts_internal.h), tree k at tree0 + k * kBytes.
//  * heap levels 0-1 (split_header depths): the 16-byte tree header, one
//    broadcast LDS.128 (ts_internal.h);
//  * top levels (< kTopLevels): the chain state is the record's shared
//    address p; the heap step j -> 2j + 1 + c (the reference's
//    i = (i<<1)+1+(x >= theta)) becomes p -> 2p + (c ? 16 - base : 8 - base):
//    LDS.64, LEA.HI, LDS, FSETP, SEL, IADD3 per visit;
//  * deep levels: state u = address of the node's fid byte(s); theta sits at
//    (4/FW) u + per-chain constant, and the step is u -> 2u + (c ? FW - cf : -cf)
//    with cf = the level-independent fid origin;
//  * leaf: ordinal from the final state, fp32 leaf value, f64 add in tree order.
//  * TERMS (warp-split kernel k_stream_ws): the fp32 leaf value of tree k
//    goes to the shared leaf buffer at lbt + k * 128 (one 32-row slab per
//    tree) instead of into acc; the accumulator warp adds w * leaf in tree
//    order.
// ORD: 0 scores only; 1 also ordinals (a.ord) and / or the tree split's terms
// (a.leaf_out), checked at run time; 2 balanced tree split of a unit-weight
// ensemble without ordinals (partial-sum bookkeeping only).
template <int D, int NK, int FW, bool UNIT_W, int ORD, int CW, bool TERMS = false, int KP = 1>
__device__ __forceinline__ void walk_group(uint32_t tree0, uint32_t xr, double &acc,
                                           const StreamArgs &a, int t, long long row,
                                           bool valid, uint32_t lbt = 0,
                                           LeafPend<KP> *pend = nullptr) {
    using R = SplitRec<D, FW>;
    constexpr uint32_t S = R::S;
    constexpr uint32_t TB = R::kRing;
    constexpr int kShift = FW == 1 ? 2 : 1;  // theta address = u << kShift + kq
    uint32_t p[NK], lo[NK], hi[NK];
#pragma unroll
    for (int k = 0; k < NK; k++) {
        const uint32_t base = tree0 + k * TB;
        p[k] = base;
        lo[k] = 8u - base;
        hi[k] = 16u - base;
    }
    uint32_t l0 = 0;
    if constexpr (split_header(D, FW)) {
        // heap levels 0-1 from the tree's 16-byte header {fid0 | fid1 << 8 |
        // fid2 << 16, theta0, theta1, theta2}: one broadcast LDS.128 instead
        // of a broadcast LDS.64 plus a two-address LDS.64 (2 wavefronts)
        constexpr uint32_t kXB = Shape<CW>::kB * 4u;  // bytes per feature row of the x tile
#pragma unroll
        for (int k = 0; k < NK; k++) {
            const uint4 hd = lds128(p[k]);
            const float v0 = ldsf((hd.x & 0xffu) * kXB + xr);
            const bool c0 = v0 >= __uint_as_float(hd.y);
            const uint32_t f1 = __byte_perm(hd.x, 0u, c0 ? 0x4442u : 0x4441u);
            const float v1 = ldsf(f1 * kXB + xr);
            const bool c1 = v1 >= __uint_as_float(c0 ? hd.w : hd.z);
            // level-2 heap index 3 + 2 c0 + c1 at base + 8 * index
            p[k] += 24u + (c0 ? 16u : 0u) + (c1 ? 8u : 0u);
        }
        l0 = 2;
    }
#pragma unroll
    for (uint32_t l = l0; l < S; l++) {
#pragma unroll
        for (int k = 0; k < NK; k++) {
            const uint2 q = lds64(p[k]);
            const float v = ldsf((q.x >> Shape<CW>::kXShift) + xr);
            p[k] = p[k] + p[k] + sel_ge(v, __uint_as_float(q.y), hi[k], lo[k]);
        }
    }
    // leaf / deep origin: cf = tree + kFid0 - FW * 2^S, u = cf + FW * h
    uint32_t u[NK];
    if constexpr (D > S) {
#pragma unroll
        for (int k = 0; k < NK; k++) {
            const uint32_t base = tree0 + k * TB;
            const uint32_t cf = base + R::kFid0 - FW * (1u << S);
            // leaving the top: h = (p - base) / 8 + 1
            u[k] = cf + FW * (((p[k] - base) >> 3) + 1u);
            lo[k] = 0u - cf;
            hi[k] = FW - cf;
            // theta(u) = (u << kShift) + kq[k]: reuse p[] for kq
            p[k] = base + R::kThr0 - 4u * (1u << S) - (cf << kShift);
        }
#pragma unroll
        for (uint32_t l = S; l < (uint32_t)D; l++) {
#pragma unroll
            for (int k = 0; k < NK; k++) {
                const float th = ldsf((u[k] << kShift) + p[k]);
                const uint32_t fid = ldsu(u[k], FW);
                const float v = ldsf(fid * (Shape<CW>::kB * 4u) + xr);
                u[k] = u[k] + u[k] + sel_ge(v, th, hi[k], lo[k]);
            }
        }
    }
    constexpr bool kDefer = R::kGLeaf && !TERMS;
    if constexpr (kDefer) flush_leaves<D, FW, UNIT_W, KP>(*pend, acc, a);  // previous group
#pragma unroll
    for (int k = 0; k < NK; k++) {
        const uint32_t base = tree0 + k * TB;
        uint32_t h;  // 1-based heap index at level D
        if constexpr (D > S) h = (u[k] - (base + R::kFid0 - FW * (1u << S))) / FW;
        else h = ((p[k] - base) >> 3) + 1u;
        float lv;
        if constexpr (R::kGLeaf)  // leaves stay in the blob (L2): node parts only in the ring
            lv = __ldg(reinterpret_cast<const float *>(a.blob + a.seg_byte0 +
                                                       (size_t)(t + k - a.t0) * R::kBytes +
                                                       R::kLeaf0) +
                       (h - (1u << D)));
        else
            lv = ldsf(base + R::kLeaf0 + 4u * (h - (1u << D)));
        if constexpr (kDefer) {  // added after the next group's walk
            pend->lv[k] = lv;
            if (k == NK - 1) {
                pend->t = t;
                pend->n = NK;
            }
        } else
        // w * leaf rounded to f64 first, then the add (never an FMA)
        if constexpr (TERMS) {
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(lbt + k * 128u), "f"(lv) : "memory");
        } else {
            const double term =
                UNIT_W ? (double)lv : __dmul_rn(__ldg(a.weight + t + k), (double)lv);
            acc = __dadd_rn(acc, term);
        }
        if constexpr (ORD == 2) {
            pend->kmin1 = min(pend->kmin1, (__float_as_uint(lv) & 0x7fffffffu) - 1u);  // zero wraps: ignored
            if constexpr (!kDefer)
                pend->amax = max(pend->amax, (uint32_t)__double2hiint(acc) & 0x7fffffffu);
        } else if constexpr (ORD == 1) {
            if (a.ord && valid) a.ord[(long long)(t + k) * a.ld_ord + row] = (uint16_t)(h - (1u << D));
            // tree-split mode: [row / 32][tree][row % 32] for k_fold.  Only rows
            // < n: the scratch holds ceil(n / 32) blocks, and a 128-row tile's
            // rows past them would write into whatever the memory pool handed
            // out next (another stream's scratch -- a concurrent-callers race).
            if (!TERMS && a.leaf_out && valid)
                a.leaf_out[((row >> 5) * a.leaf_T + (t + k - a.t0)) * 32 + (row & 31)] =
                    UNIT_W ? (double)lv : __dmul_rn(__ldg(a.weight + t + k), (double)lv);
            if constexpr (!TERMS) {
                if (a.leaf_out || a.sk_ctas > 0) {
                    // fp32-valued terms only (w * leaf has a full f64
                    // mantissa: amax = all ones makes the exactness test fail)
                    if constexpr (UNIT_W) {
                        pend->kmin1 = min(pend->kmin1, (__float_as_uint(lv) & 0x7fffffffu) - 1u);  // zero wraps: ignored
                        if constexpr (!kDefer)
                            pend->amax = max(pend->amax, (uint32_t)__double2hiint(acc) & 0x7fffffffu);
                    } else {
                        pend->amax = 0xffffffffu;
                    }
                }
            }
        }
    }
}

template <int D, int K, int FW, bool UNIT_W, int ORD, int CW>
__global__ void __launch_bounds__(Shape<CW>::kThreads, Shape<CW>::kCtasPerSm)
    k_stream(StreamArgs a) {
    constexpr int kB = Shape<CW>::kB;
    constexpr int kConsumerWarps = CW;
    extern __shared__ __align__(128) unsigned char smem[];
    float *xs = reinterpret_cast<float *>(smem);
    unsigned char *ring = smem + a.xs_bytes;
    const int kStages = a.stages;
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + kStages * a.chunk_cap);
    uint64_t *empty = full + kMaxStages;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kMaxStages; s++) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long ntiles = (a.n + kB - 1) / kB;
    const int nchunks = (a.t1 - a.t0 + a.tpc - 1) / a.tpc;
    // Spans (a tile and the chunk range [cb, ce) walked of it) this CTA owns:
    // all chunks of tiles blockIdx.x, +gridDim.x, ... normally; one tile and 1/splits of its chunks in
    // small-batch tree-split mode; an equal run of the tile-major (tile,
    // chunk) items in balanced mode (a.sk_ctas), which may end one tile and
    // start the next.
    struct Span {
        long long tile, pos, end;
        int cb, ce;
    };
    // (the split modes run on the ORD != 0 instantiations only)
    constexpr bool kSplitModes = ORD != 0;
    // The plain kernels keep the loop form they were tuned with (run-time
    // start / step / chunk range, the uniform split folded in): ptxas's
    // register allocation of the walk follows it, and the simpler constant
    // form measured -1 % at d = 4 but +2 % at d = 3 and +3.5 % at d = 10.
    long long tile0 = blockIdx.x, tstep = gridDim.x;
    int cb0 = 0, ce0 = nchunks;
    if (!kSplitModes && a.splits > 1) {
        tile0 = blockIdx.x % ntiles;
        tstep = ntiles;
        const long long j = blockIdx.x / ntiles;
        cb0 = (int)(j * nchunks / a.splits);
        ce0 = (int)((j + 1) * nchunks / a.splits);
    }
    auto span_load = [&](Span &sp) -> bool {
        if (sp.pos >= sp.end) return false;
        if (kSplitModes && a.sk_ctas > 0) {
            sp.tile = sp.pos / nchunks;
            sp.cb = (int)(sp.pos - sp.tile * nchunks);
            sp.ce = (int)min((long long)nchunks, sp.cb + (sp.end - sp.pos));
        } else if (kSplitModes && a.splits > 1) {
            sp.tile = blockIdx.x % ntiles;
            const long long j = blockIdx.x / ntiles;
            sp.cb = (int)(j * nchunks / a.splits);
            sp.ce = (int)((j + 1) * nchunks / a.splits);
        } else {
            sp.tile = sp.pos;
            sp.cb = 0;
            sp.ce = nchunks;
        }
        return true;
    };
    auto span_first = [&](Span &sp) -> bool {
        if (kSplitModes && a.sk_ctas > 0) {
            const long long W = ntiles * nchunks;
            sp.pos = (long long)blockIdx.x * W / a.sk_ctas;
            sp.end = (long long)(blockIdx.x + 1) * W / a.sk_ctas;
        } else if (kSplitModes && a.splits > 1) {
            sp.pos = 0;
            sp.end = 1;
        } else {
            sp.pos = blockIdx.x;
            sp.end = ntiles;
        }
        return span_load(sp);
    };
    auto span_next = [&](Span &sp) -> bool {
        sp.pos += (kSplitModes && a.sk_ctas > 0) ? (long long)(sp.ce - sp.cb)
                  : (kSplitModes && a.splits > 1) ? 1 : (long long)gridDim.x;
        return span_load(sp);
    };

    if (warp == kConsumerWarps) {  // ---- producer warp: TMA bulk copies
        if (lane == 0) {
            // ring position tracked incrementally (no runtime division)
            int s = 0;
            uint32_t ph = 0, used = 0;  // phase of stage s's next reuse; first lap done?
            auto produce = [&](int cb, int ce) {
                for (int c = cb; c < ce; c++) {
                    if (used) mbar_wait(empty + s, ph);
                    const int trees = min(a.tpc, a.t1 - a.t0 - c * a.tpc);
                    produce_chunk<D, FW>(a, ring + s * a.chunk_cap, full + s, c, trees);
                    if (++s == kStages) {
                        s = 0;
                        ph ^= used;
                        used = 1;
                    }
                }
            };
            if constexpr (kSplitModes) {
                Span sp;
                for (bool more = span_first(sp); more; more = span_next(sp)) produce(sp.cb, sp.ce);
            } else {
                for (long long tile = tile0; tile < ntiles; tile += tstep) produce(cb0, ce0);
            }
        }
        return;
    }

    // ---- consumer warps
    const int r = threadIdx.x;
    const uint32_t xr = su32(xs) + 4u * r;
    int s = 0;
    uint32_t ph = 0;  // parity of stage s's current fill
    auto consume = [&](const long long tile, const int cb, const int ce) {
        const long long row = tile * kB + r;
        const bool valid = row < a.n;
        consumer_sync<kB>();  // previous tile's walks are done with xs
        stage_rows<kB, ORD != 0>(a, xs, tile * kB);
        consumer_sync<kB>();
        // balanced mode: a tile walked only in part contributes a partial sum from 0
        const bool part = kSplitModes && a.sk_ctas > 0 && (cb != 0 || ce != nchunks);
        double acc = (a.accumulate && valid && !part) ? a.out[row] : 0.0;
        LeafPend<K> pend;  // global-leaf depths: the last group's leaves, added late
        // Cross-GPU running-sum pipeline (ts_score_pipe): this warp's 32-row
        // block continues the sums the previous rank published for it.
        const long long blk = tile * (long long)CW + warp;
        if (a.pipe.flags_in) {
            if (lane == 0 && blk < a.pipe.nblocks) pipe_wait(a.pipe.flags_in + blk, a.pipe.epoch);
            __syncwarp();
            acc = valid ? __ldcv(a.pipe.sums_in + row) : 0.0;
        }
        for (int c = cb; c < ce; c++) {
            mbar_wait(full + s, ph);
            const uint32_t buf = su32(ring + s * a.chunk_cap);
            const int t0 = a.t0 + c * a.tpc;
            const int trees = min(a.tpc, a.t1 - t0);
            int k = 0;
            for (; k + K <= trees; k += K)
                walk_group<D, K, FW, UNIT_W, ORD, CW, false, K>(
                    buf + k * SplitRec<D, FW>::kRing, xr, acc, a, t0 + k, row, valid, 0, &pend);
            for (; k < trees; k++)
                walk_group<D, 1, FW, UNIT_W, ORD, CW, false, K>(
                    buf + k * SplitRec<D, FW>::kRing, xr, acc, a, t0 + k, row, valid, 0, &pend);
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
            if (++s == kStages) {
                s = 0;
                ph ^= 1u;
            }
        }
        if constexpr (SplitRec<D, FW>::kGLeaf) flush_leaves<D, FW, UNIT_W, K>(pend, acc, a);
        if constexpr (ORD) {
            if (a.leaf_out && valid) {  // tree-split mode: this CTA's partials (StreamArgs::part_sum)
                const long long pj = (row >> 5) * a.splits + blockIdx.x / ntiles;
                a.part_sum[pj * 32 + (row & 31)] = acc;
                a.part_key[pj * 64 + (row & 31)] = pend.amax;
                a.part_key[pj * 64 + 32 + (row & 31)] = pend.kmin1;
            }
        }
        if (part) {
            // slice = this CTA's rank among the CTAs sharing the tile (the
            // first of them holds item tile * nchunks)
            if (valid) {
                const long long W = ntiles * nchunks;
                const long long b0 = ((tile * nchunks + 1) * a.sk_ctas - 1) / W;
                const long long pj = (tile * a.sk_slices + (blockIdx.x - b0)) * kB + r;
                a.part_sum[pj] = acc;
                a.part_key[2 * pj] = pend.amax;
                a.part_key[2 * pj + 1] = pend.kmin1;
            }
        } else if (a.pipe.sums_out) {
            // publish to the next rank (peer memory over NVLink), then flag
            if (valid) a.pipe.sums_out[row] = acc;
            __threadfence_system();
            __syncwarp();
            if (lane == 0 && blk < a.pipe.nblocks) pipe_signal(a.pipe.flags_out + blk, a.pipe.epoch);
        } else if (valid && a.out) {
            a.out[row] = acc;
        }
    };
    if constexpr (kSplitModes) {
        Span sp;
        for (bool more = span_first(sp); more; more = span_next(sp)) consume(sp.tile, sp.cb, sp.ce);
    } else {
        for (long long tile = tile0; tile < ntiles; tile += tstep) consume(tile, cb0, ce0);
    }
}

// ---------------------------------------------------------------------------
// Warp-split variant for small batches (k_stream_ws).  k_stream gives each
// warp its own 32 rows and ALL trees, so a batch of a few thousand rows
// occupies a fraction of the SMs and each warp walks the whole ensemble
// serially.  Here a CTA owns only 32 rows; its kWsWarps walker warps share
// them and split each chunk's K-groups round-robin; every walk stores its f64
// term w * leaf in a double-buffered shared leaf buffer lb[tree][row], and an
// accumulator warp adds the chunk's terms in TREE order (acc = acc + term,
// __dadd_rn) -- the same sequence of roundings as k_stream, so scores stay
// bit-identical.  Walkers and accumulator hand buffers over with mbarriers
// (lbf: written by all walkers, lbe: folded), the producer streams chunks
// exactly as in k_stream.  Two or three CTAs per SM (plan_stream_ws).
constexpr int kWsWarps = 4;
__host__ __device__ constexpr int ws_chains(int d) {
    return d <= 6 ? 8 : d <= 8 ? 4 : d <= 9 ? 2 : 1;
}

// Stage 32 rows x F features into xs[f * 32 + r] with all 32 * kWsWarps
// walker threads (row r = tid % 32, a quarter of the row's columns each).
__device__ __forceinline__ void stage_rows_ws(const StreamArgs &a, float *xs, long long row0) {
    constexpr int B = 32;
    const int tid = threadIdx.x;
    const int r = tid & 31, q = tid >> 5;
    const long long row = row0 + r;
    const bool valid = row < a.n;
    const float *xrow = a.x + (valid ? row : 0) * a.ld;
    const int F = a.F;
    bool bad = false;
    if (((F & 3) == 0) && ((a.ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0)) {
        const int F4 = F >> 2;
        const float4 *x4 = reinterpret_cast<const float4 *>(xrow);
        // 12 float4 per thread: a row of up to 192 features lands in one
        // round trip (the latency a small batch waits on)
        constexpr int U = 12;
        for (int c0 = q * U; c0 < F4; c0 += kWsWarps * U) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; u++)
                v[u] = (valid && c0 + u < F4) ? __ldg(x4 + c0 + u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (c0 + u >= F4) break;
                bad |= !(finite_f(v[u].x) && finite_f(v[u].y) && finite_f(v[u].z) &&
                         finite_f(v[u].w));
                float *dst = xs + 4 * (c0 + u) * B + r;
                dst[0] = v[u].x;
                dst[B] = v[u].y;
                dst[2 * B] = v[u].z;
                dst[3 * B] = v[u].w;
            }
        }
    } else {
        for (int c = q; c < F; c += kWsWarps) {
            const float v = valid ? __ldg(xrow + c) : 0.f;
            bad |= !finite_f(v);
            xs[c * B + r] = v;
        }
    }
    if (bad && a.status) atomicOr(a.status, 1);
}

template <int D, int K, int FW, bool UNIT_W, bool ORD>
__global__ void __launch_bounds__(32 * (kWsWarps + 2), 3) k_stream_ws(StreamArgs a) {
    constexpr int B = 32;
    constexpr int NW = kWsWarps;
    using R = SplitRec<D, FW>;
    extern __shared__ __align__(128) unsigned char smem[];
    float *xs = reinterpret_cast<float *>(smem);
    unsigned char *lb = smem + a.xs_bytes;  // 2 x tpc x 32 fp32 leaf values
    unsigned char *ring = lb + a.lb_bytes;
    const int kStages = a.stages;
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + kStages * a.chunk_cap);
    uint64_t *empty = full + kMaxStages;
    uint64_t *lbf = empty + kMaxStages;  // leaf buffer written (NW walker warps)
    uint64_t *lbe = lbf + 2;             // leaf buffer folded (accumulator warp)
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kMaxStages; s++) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, NW);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(lbf + b, NW);
            mbar_init(lbe + b, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long ntiles = (a.n + B - 1) / B;
    const int nchunks = (a.t1 - a.t0 + a.tpc - 1) / a.tpc;
    const uint32_t lb_half = a.lb_bytes / 2;

    if (warp == NW + 1) {  // ---- producer warp: TMA bulk copies (as k_stream)
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0, used = 0;
            for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int c = 0; c < nchunks; c++) {
                    if (used) mbar_wait(empty + s, ph);
                    const int trees = min(a.tpc, a.t1 - a.t0 - c * a.tpc);
                    produce_chunk<D, FW>(a, ring + s * a.chunk_cap, full + s, c, trees);
                    if (++s == kStages) {
                        s = 0;
                        ph ^= used;
                        used = 1;
                    }
                }
            }
        }
        return;
    }

    if (warp == NW) {  // ---- accumulator warp: tree-order f64 fold
        uint32_t it = 0;
        for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const long long row = tile * B + lane;
            const bool valid = row < a.n;
            double acc = (a.accumulate && valid) ? a.out[row] : 0.0;
            for (int c = 0; c < nchunks; c++, it++) {
                const int b = it & 1;
                const int trees = min(a.tpc, a.t1 - a.t0 - c * a.tpc);
                mbar_wait(lbf + b, (it >> 1) & 1);
                const float *lv = reinterpret_cast<const float *>(lb + b * lb_half) + lane;
                const double *w = a.weight + a.t0 + c * a.tpc;
                // w * leaf rounded to f64 first (off the DADD chain), then the add
#pragma unroll 8
                for (int i = 0; i < trees; i++)
                    acc = __dadd_rn(acc, UNIT_W ? (double)lv[i * B]
                                                : __dmul_rn(__ldg(w + i), (double)lv[i * B]));
                __syncwarp();
                if (lane == 0) mbar_arrive(lbe + b);
            }
            if (valid && a.out) a.out[row] = acc;
        }
        return;
    }

    // ---- walker warps
    const uint32_t xr = su32(xs) + 4u * lane;
    int s = 0;
    uint32_t ph = 0;
    uint32_t it = 0;
    double unused = 0.0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long row = tile * B + lane;
        const bool valid = row < a.n;
        consumer_sync<NW * 32>();  // previous tile's walks are done with xs
        stage_rows_ws(a, xs, tile * B);
        consumer_sync<NW * 32>();
        for (int c = 0; c < nchunks; c++, it++) {
            const int b = it & 1;
            mbar_wait(full + s, ph);
            if (it >= 2) mbar_wait(lbe + b, ((it >> 1) - 1) & 1);  // buffer b folded
            const uint32_t buf = su32(ring + s * a.chunk_cap);
            const uint32_t lbt = su32(lb + b * lb_half) + 4u * lane;
            const int t0 = a.t0 + c * a.tpc;
            const int trees = min(a.tpc, a.t1 - t0);
            const int ng = trees / K;
            for (int g = warp; g < ng; g += NW)
                walk_group<D, K, FW, UNIT_W, ORD, 1, true>(buf + g * K * R::kRing, xr, unused, a,
                                                           t0 + g * K, row, valid,
                                                           lbt + g * K * 128u);
            for (int k = ng * K + warp; k < trees; k += NW)
                walk_group<D, 1, FW, UNIT_W, ORD, 1, true>(buf + k * R::kRing, xr, unused, a,
                                                           t0 + k, row, valid, lbt + k * 128u);
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(empty + s);  // ring stage read
                mbar_arrive(lbf + b);    // terms published (release orders the stores)
            }
            if (++s == kStages) {
                s = 0;
                ph ^= 1u;
            }
        }
    }
}

template <int D>
cudaError_t launch_ws_d(const StreamArgs &a, int device, cudaStream_t stream) {
    constexpr int K = ws_chains(D);
    auto pick = [&](auto fw) {
        constexpr int FW = decltype(fw)::value;
        if (a.ord) return a.unit_w ? k_stream_ws<D, K, FW, true, true> : k_stream_ws<D, K, FW, false, true>;
        return a.unit_w ? k_stream_ws<D, K, FW, true, false> : k_stream_ws<D, K, FW, false, false>;
    };
    auto kern = a.fw == 1 ? pick(std::integral_constant<int, 1>{})
                          : pick(std::integral_constant<int, 2>{});
    const size_t smem = (size_t)a.xs_bytes + a.lb_bytes + (size_t)a.stages * a.chunk_cap +
                        (2 * kMaxStages + 4) * 8;
    cudaError_t e = ensure_smem((const void *)kern, smem);
    if (e != cudaSuccess) return e;
    const long long tiles = (a.n + 31) / 32;
    const int sms = dev_attrs(device).sms;
    const int grid = (int)std::min<long long>(tiles, (long long)a.ws_ctas * sms);
    kern<<<grid, 32 * (kWsWarps + 2), smem, stream>>>(a);
    count_launch();
    return cudaGetLastError();
}

template <int D, int K, int FW, int CW>
auto pick_kernel_k(const StreamArgs &a) {
    if (a.sk_ctas > 0 && a.unit_w && !a.ord) return k_stream<D, K, FW, true, 2, CW>;
    if (a.ord || a.leaf_out || a.sk_ctas > 0)
        return a.unit_w ? k_stream<D, K, FW, true, 1, CW> : k_stream<D, K, FW, false, 1, CW>;
    return a.unit_w ? k_stream<D, K, FW, true, 0, CW> : k_stream<D, K, FW, false, 0, CW>;
}
template <int D, int FW, int CW>
auto pick_kernel(const StreamArgs &a) {
    constexpr int K = chains_for_depth(D), K2 = chains_fallback(D);
    if constexpr (K2 != K) {
        if (a.k == K2) return pick_kernel_k<D, K2, FW, CW>(a);
    }
    return pick_kernel_k<D, K, FW, CW>(a);
}

template <int D, int CW>
cudaError_t launch_dc(const StreamArgs &a, int device, cudaStream_t stream) {
    constexpr int kB = Shape<CW>::kB;
    constexpr int kCtasPerSm = Shape<CW>::kCtasPerSm;
    constexpr int kThreads = Shape<CW>::kThreads;
    auto kern = a.fw == 1 ? pick_kernel<D, 1, CW>(a) : pick_kernel<D, 2, CW>(a);
    const int sms = dev_attrs(device).sms;
    cudaError_t e;
    const size_t smem = a.xs_bytes + (size_t)a.stages * a.chunk_cap + 2 * kMaxStages * 8;
    e = ensure_smem((const void *)kern, smem);
    if (e != cudaSuccess) return e;
    const long long tiles = (a.n + kB - 1) / kB;
    const int grid = a.sk_ctas > 0 ? a.sk_ctas
                     : a.splits > 1 ? (int)(tiles * a.splits)
                                    : (int)(tiles < (long long)sms * kCtasPerSm
                                                ? tiles : (long long)sms * kCtasPerSm);
    kern<<<grid, kThreads, smem, stream>>>(a);
    count_launch();
    return cudaGetLastError();
}

template <int D>
cudaError_t launch_d(const StreamArgs &a, int device, cudaStream_t stream) {
    return a.cw == 4 ? launch_dc<D, 4>(a, device, stream) : launch_dc<D, 8>(a, device, stream);
}

}  // namespace stream_detail
}  // namespace ts
