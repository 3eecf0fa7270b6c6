// Internal declarations shared by the packer, the kernels and the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/treescore_gpu.h"

namespace ts {

// Node-table layouts.
//  kComplete: implicit breadth-first heap of the tree's complete expansion to
//             its own depth d: 2^d - 1 node records {fid, theta bits} with the
//             children of slot i at 2i+1 / 2i+2, plus 2^d fp32 leaves.  Dummy
//             padding slots hold (fid 0, theta +inf) exactly as
//             expand_to_complete (ref model.py:315-349) writes them.
//  kCompact:  the tree's own nodes in BFS order with sibling pairs adjacent:
//             record {fid | left << 16, theta bits}; right child = left + 1.
//             A leaf is a self-loop {F | self << 16, leaf value bits}: the
//             x-tile row F holds -inf, so `x >= value` is false and the walk
//             stays put for the remaining levels of its K-group (and the
//             predicated ordinal gains the same zero bits a dummy subtree
//             would give it).
//  kSplit:    the streaming kernel's form of a complete tree (ts_stream.cu):
//             heap levels < kTopLevels as {fid << kFidShift, theta} records,
//             deeper levels as separate fp32-threshold and 1- or 2-byte fid
//             arrays (smaller, less bank-conflicted shared-memory reads).
//  kCStream:  kCompact for the irregular-tree streaming kernel (ts_cstream.cu):
//             record {(4 B fid) << 14 | left, theta} with B the kernel's
//             instance tile (so 4 B fid is the feature's byte offset in the x
//             tile, < 2^18); leaf {(4 B F) << 14 | self, value}; trees of
//             <= 8191 nodes, grouped into chunks of <= kCStreamMaxT trees.
//  kRank:     a complete tree for the rank kernels (ts_rank.cu): every
//             threshold replaced by its rank among the ensemble's distinct
//             thresholds of the same feature, so a node is ONE 4-byte record
//             rec = fid << 24 | rank (rank 1-based, < 2^15; kRankInf for
//             dummy +inf nodes) in heap order, then 2^d fp32 leaves; the
//             instances go through the same map (ts_rank.cu k_rank: rank(x) =
//             number of distinct thresholds <= x), and x >= theta <=>
//             rank(x) >= rank(theta) exactly.
enum Layout : int { kComplete = 0, kCompact = 1, kSplit = 2, kCStream = 3, kRank = 4 };

struct Segment {
    int layout;   // Layout
    int depth;    // kComplete: the common depth of every tree in the segment
    int t0, t1;   // tree range [t0, t1) in evaluation order
    uint64_t byte0;  // blob offset of tree t0
    int chunk0 = 0, nchunks = 0;  // kCStream: chunk table range
    int cs_b = 0;                 // kCStream: instance tile the records were encoded for
    int rank_space = 0;           // kRank: index into DeviceTables::rank_spaces
    // Streaming layouts: expected fraction of rows whose tree-order sum may round (pack-
    // time estimate from the leaf magnitudes, ts_pack.cpp slow_row_rate): the
    // balanced tree split scores such rows a second time, one after another.
    float slow_rows = 0.f;
};

// All trees live in one byte blob, tree t at byte 16 * tree_off16[t]:
//  kComplete: (2^d - 1) uint2 {fid << kFidShift, theta bits} in heap order, then 2^d fp32
//             leaves, padded to 16 bytes (so a run of equal-depth trees is a
//             regular array the TMA streams chunk by chunk);
//  kCompact:  n_t uint2 records (see Layout), padded to 16 bytes.
// Logical node for the tracer (ts_trace.cu): fid -1 marks a leaf whose
// `left` holds its left-to-right ordinal and `value` its leaf value.
struct TraceNode {
    int32_t fid;
    float value;
    int32_t left, right;  // tree-local node ids
};

// A rank space: per feature the sorted distinct thresholds (-0.0 folded into
// +0.0) of a run of rank-layout trees (their node ranks index these lists;
// at most kRankMaxU per feature, so an ensemble with more distinct
// thresholds is split into several spaces, each scored by its own
// pre-pass).  The pre-pass searches each list as a complete binary search
// tree in breadth-first (Eytzinger) order padded with +inf to 2^L - 1
// entries: rank = (leaf reached after L steps) - (2^L - 1), the same heap
// walk as the trees', and bank-conflict-light (a sorted array's binary
// search probes one bank from every lane); feature f's tree is
// e[eoff[f] .. eoff[f + 1]).
struct RankSpace {
    float *e = nullptr;
    uint32_t *eoff = nullptr;        // [F + 1]
    int2 *groups = nullptr;          // pre-pass feature groups {f0, f1}
    int ngroups = 0;
    uint32_t group_words = 0;        // largest group's float count (+ alignment)
};

struct DeviceTables {
    unsigned char *blob = nullptr;
    uint32_t *tree_off16 = nullptr;  // [T]
    int32_t *depth = nullptr;        // [T]
    double *weight = nullptr;        // [T]
    // kCStream chunk tables
    uint4 *chunk_info = nullptr;     // {blob off / 16, bytes, trees, first tree}
    uint32_t *slot_meta = nullptr;   // [chunks][kCStreamMaxT] rec_off/8 | depth<<16 | rel<<21
    // TS_PACK_TRACE only
    TraceNode *trace_nodes = nullptr;
    uint32_t *trace_base = nullptr;  // [T] first node of tree t
    // kRank: the rank spaces (RankSpace; a segment of kRank trees uses one)
    std::vector<RankSpace> rank_spaces;
    // Balanced tree split, observed: {rows scored a second time by k_combine,
    // rows of the tiles it combined} counted on the device (slow_dev); a CTA
    // that saw such rows (and CTA 0) also posts the running totals into
    // mapped pinned host memory (slow_seen; slow_seen_dev is its device
    // address) -- plain stores, last writer wins, good enough for a heuristic
    // (a stream-ordered copy after each call cost ~10 us of latency).  The pack-time estimate (Segment::slow_rows) knows the leaves
    // but not how often the data reaches the tiny ones; once > 3 % of the
    // combined rows needed the second walk the planner stops splitting this
    // model (balanced_split_trusted).
    unsigned int *slow_dev = nullptr;
    unsigned int *slow_seen = nullptr, *slow_seen_dev = nullptr;
};



// kComplete records store fid << kFidShift: the byte offset of feature fid's
// row in the streaming kernel's 256-instance x tile (256 * 4 = 1 << 10).
constexpr int kFidShift = 10;

inline uint32_t complete_tree_bytes(int d) {
    return (uint32_t)((((1u << d) - 1u) * 8u + (1u << d) * 4u + 15u) & ~15u);
}

// kSplit tree record: [top records][deep thresholds][leaves][deep fids].
constexpr int kTopLevels = 5;
// kSplit record of a depth-d tree: top-level records | deep thresholds |
// deep fids | (16-byte aligned) leaves.  The node part [0, leaf0) is what the
// shared-memory walk needs; trees with d >= kGLeafDepth stream only that part
// through the ring and read their leaf from the record in global memory
// (L2), which doubles the trees in flight (ts_stream_kernel.cuh; at d = 10 it
// measured 4 % slower: the extra L1TEX wavefronts of the leaf gather cost more
// than the chains gained).
constexpr int kGLeafDepth = 11;
struct SplitGeom {
    uint32_t thr0, fid0, leaf0, bytes;
};
inline SplitGeom split_geom(int d, int fw) {
    const uint32_t S = d < kTopLevels ? d : kTopLevels;
    const uint32_t deep = (1u << d) - (1u << S);
    SplitGeom g;
    g.thr0 = ((1u << S) - 1u) * 8u;
    g.fid0 = g.thr0 + deep * 4u;
    g.leaf0 = (g.fid0 + deep * (uint32_t)fw + 15u) & ~15u;
    g.bytes = (g.leaf0 + (1u << d) * 4u + 15u) & ~15u;
    return g;
}
// Heap levels 0-1 as a 16-byte header {fid0 | fid1 << 8 | fid2 << 16, theta0,
// theta1, theta2} in record slots 0-1 (one broadcast LDS.128 for both levels;
// single-byte fids).  Per depth as measured (r1 session 2, 1M rows x 1000
// trees, F = 136): +2-4 % at d = 2, 3, 5, 6, 7, 9, +1.9 % at d = 4 together
// with 24 chains (-0.7 % with 16); -0.5 % at d = 8 (the headline), neutral
// at 10-12.
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr bool split_header(int d, int fw) { return fw == 1 && d >= 2 && d != 8; }
// kRank record geometry: 4-byte records in heap order, then the leaves.
constexpr uint32_t kRankInf = 0x7fffu;   // rank of a dummy (+inf) threshold
constexpr int kRankMaxU = 0x7ffe;        // distinct thresholds per feature
constexpr int kRankB = 256;              // rows per rank tile (R layout and kernel)
constexpr int kRankMaxDepth = 14;        // deepest tree the rank walk streams (d = 13-14:
                                         // the fp32 layouts only have the L1 path there)
// u16 slot of row r (0..255) in a feature's 512-byte run of a rank tile:
// warps 2k and 2k+1 share 32-bit words (low / high halves), lane l of a warp
// in word 32k + l -- so a warp's 32 lanes read 32 distinct banks for any mix
// of features (two rows of one warp in one word would be a 2-way conflict on
// every x read).
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr uint32_t rank_slot(uint32_t r) {
    return ((((r >> 5) >> 1) << 5) + (r & 31u)) * 2u + ((r >> 5) & 1u);
}
struct RankGeom {
    uint32_t leaf0, bytes;
};
inline RankGeom rank_geom(int d) {
    RankGeom g;
    g.leaf0 = ((((1u << d) - 1u) * 4u) + 15u) & ~15u;
    g.bytes = (g.leaf0 + (1u << d) * 4u + 15u) & ~15u;
    return g;
}
inline uint32_t rank_ring_bytes(int d) {
    const RankGeom g = rank_geom(d);
    return d >= 11 ? g.leaf0 : g.bytes;  // node part only at global-leaf depths
}
// Bytes of one tree in a ring stage: the node part for global-leaf depths.
inline uint32_t split_ring_bytes(int d, int fw) {
    const SplitGeom g = split_geom(d, fw);
    return d >= kGLeafDepth ? g.leaf0 : g.bytes;
}

struct HostScratch {
    float *x[2] = {nullptr, nullptr};
    double *out = nullptr;
    int32_t *status = nullptr;
    int64_t x_rows = 0, out_rows = 0;
    cudaStream_t copy = nullptr, compute = nullptr;
    cudaEvent_t copied[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
    // pinned staging for pageable caller buffers (ts_score_host)
    float *hx[2] = {nullptr, nullptr};
    double *hout[2] = {nullptr, nullptr};
    int64_t hx_rows = 0, hout_rows = 0;
    cudaEvent_t d2h[2] = {nullptr, nullptr};
    // small batches (ts_score_host direct path): mapped pinned memory the
    // kernel reads rows from and writes scores and status into over PCIe,
    // so a call is one launch and one stream sync (no copy commands)
    unsigned char *map = nullptr;   // rows | scores | status
    size_t map_bytes = 0;
};

}  // namespace ts

struct ts_model {
    int device = 0;
    int num_features = 0;
    int num_trees = 0;
    bool unit_weights = true;
    std::vector<ts::Segment> segments;
    ts::DeviceTables dev;
    ts_model_info info{};
    // Host-buffer pipelines (ts_score_host): one HostScratch (streams, device
    // chunks, pinned staging) per concurrent caller, reused across calls;
    // callers beyond kMaxHostScratch wait for one to come back.
    static constexpr int kMaxHostScratch = 8;
    std::mutex scratch_mu;
    std::condition_variable scratch_cv;
    std::vector<std::unique_ptr<ts::HostScratch>> scratch_all;
    std::vector<ts::HostScratch *> scratch_free;
};

namespace ts {

void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t err, const char *what);

// Cross-GPU running-sum pipeline of ts_score_pipe (32-row blocks).
struct PipeArgs {
    const double *sums_in = nullptr;       // running sums from the previous rank
    const uint32_t *flags_in = nullptr;    // [nblocks], == epoch when published
    double *sums_out = nullptr;            // next rank's sums_in (peer pointer)
    uint32_t *flags_out = nullptr;         // next rank's flags_in (peer pointer)
    uint32_t epoch = 0;
    long long nblocks = 0;
};

struct ScoreArgs {
    const float *x;
    long long n, ld;
    int F;
    const DeviceTables *tables;
    const unsigned char *blob;
    const uint32_t *tree_off16;
    const int32_t *depth;
    const double *weight;
    int t0, t1;
    int unit_w;
    int accumulate;
    double *out;
    uint16_t *ord;
    long long ld_ord;
    int32_t *status;
    PipeArgs pipe;  // k_stream only (ts_score_pipe)
    // x is mapped pinned HOST memory (ts_score_host's small-batch path):
    // kernels that stage each row once read it over PCIe; the others get a
    // device copy first (x_device_copy)
    int x_mapped;
};

// Arguments of the shared-memory streaming kernel (ts_stream.cu).
constexpr int kStreamMaxDepth = 12;
struct StreamArgs {
    int cw;                        // consumer warps per CTA (1: 8 CTAs/SM, 4: 2, 8: 1)
    int fw;                        // deep fid width in bytes (1: F <= 256, else 2)
    const float *x;
    long long n, ld;
    int F;
    const unsigned char *blob;
    unsigned long long seg_byte0;  // blob offset of tree t0
    uint32_t tree_bytes;           // split_geom(D, fw).bytes: record stride in the blob
    uint32_t ring_tree_bytes;      // bytes per tree in a ring stage (split_ring_bytes)
    int tpc;                       // trees per chunk
    uint32_t chunk_cap;            // bytes per ring stage
    int stages;                    // ring stages (2..4)
    uint32_t xs_bytes;             // instance tile bytes
    const double *weight;
    int t0, t1;
    int unit_w;
    int accumulate;
    double *out;
    uint16_t *ord;
    long long ld_ord;
    int32_t *status;
    PipeArgs pipe;
    // > 1: small-batch tree split -- CTA b walks tile b % tiles over chunk
    // range b / tiles of `splits`, writing each tree's f64 term w * leaf to
    // leaf_out ([row / 32][tree - t0][row % 32], leaf_T trees) instead of
    // summing (out unused); k_fold (ts_stream.cu) then adds them in tree order.
    int splits;
    double *leaf_out;
    long long leaf_T;
    // Tree split, per (32-row block, split CTA): the CTA's own sequential sum
    // of its terms and the largest / smallest nonzero |leaf| bit pattern it
    // saw ([row / 32][split][row % 32]; part_key: max then min-1, 2 x 32 per
    // split).  k_fold uses them to prove that every partial sum of the row is
    // exactly representable -- then the sum does not depend on the order and
    // the splits' sums simply add up (ts_stream.cu).
    double *part_sum;
    uint32_t *part_key;
    // Balanced tree split ("stream-K"; ts_stream.cu launch_balanced): the
    // (tile, chunk) work items, tile-major, are cut into sk_ctas equal runs,
    // one per CTA.  A tile walked by ONE CTA is finished by it; a tile shared
    // by several gets one partial per CTA (part_sum / part_key indexed
    // [tile][slice][row in tile], sk_slices slots per tile) and k_combine
    // adds them when split_sum_exact allows, else walks the row's trees
    // again in the blob and adds the leaves in tree order.
    int sk_ctas, sk_slices;
    float slow_rows;  // Segment::slow_rows
    const DeviceTables *tables;  // observed second-walk counters (may be null)
    uint32_t lb_bytes;  // warp-split kernel (k_stream_ws): two tpc x 32 fp32 leaf buffers
    int ws_ctas;        // warp-split kernel: CTAs per SM (2 or 3)
    int k;              // k_stream lockstep chains per thread (chains_for_depth / _fallback)
    int x_mapped;       // see ScoreArgs::x_mapped
};
// n: rows of the launch (-1 at pack time: shape-independent checks only).
bool plan_stream(int F, int D, int device, StreamArgs *a, long long n = -1);
// Warp-split small-batch kernel shape (32-row CTAs, three or two per SM,
// returned in a->ws_ctas); false if it does not fit.
bool plan_stream_ws(int F, int D, int device, StreamArgs *a);
inline int split_fid_width(int F) { return F <= 256 ? 1 : 2; }
cudaError_t launch_stream(int D, const StreamArgs &a, int device, cudaStream_t stream);
// Stream-ordered device copy of rows [0, n) x ld of (mapped host) x from the
// library's memory pool; *dst is nullptr (and cudaSuccess) if no pool.
cudaError_t x_device_copy(const float *x, long long n, long long ld, int device,
                          cudaStream_t stream, float **dst);

// Irregular-tree streaming kernel (ts_cstream.cu).
constexpr int kCStreamMaxT = 64;     // tree slots per chunk
constexpr int kCStreamMaxNodes = 8191;
struct CStreamArgs {
    const float *x;
    long long n, ld;
    int F;
    int B;                 // instances per tile (32 * G)
    const unsigned char *blob;
    const uint4 *chunk_info;
    const uint32_t *slot_meta;
    int chunk0, nchunks;
    int tpc;               // max trees per chunk
    int w;                 // walker warps (8 or 16)
    int stages;            // ring stages (2-4)
    int teams;             // 1: every walker warp on every chunk; 2: alternate chunks
    int k;                 // lockstep chains per thread (3..8)
    uint32_t chunk_cap, stage_bytes, xs_bytes, lb_bytes;
    const double *weight;
    int unit_w, accumulate;
    double *out;
    uint16_t *ord;
    long long ld_ord;
    int32_t *status;
    // Balanced tree split (ts_stream.cu launch_balanced, same scheme): sk_ctas
    // CTAs take equal runs of the tile-major (tile, chunk) items; a tile
    // shared by several CTAs gets one partial per CTA ([tile][slice][row]).
    int sk_ctas, sk_slices;
    double *part_sum;
    uint32_t *part_key;
};
bool plan_cstream(int F, int device, CStreamArgs *a);

// Rank kernels (ts_rank.cu): whether depth D over F features has a plan on
// this device, and the launch of one kRank segment (pre-pass + walk).
// Second kernel of a balanced tree split (ts_stream.cu k_combine): adds the
// partials of every tile shared by several CTAs, or scores a row again in tree
// order when its sums could round.  The record form the second walk reads:
struct LeafWalk {
    int rank;                 // 0: kSplit record + fp32 rows; 1: kRank record + rank tiles;
                              // 2: kCStream child-index records + fp32 rows
    int D, fw, header;        // kSplit: depth, fid width, 16-byte header
    uint32_t thr0, fid0, leaf0, tree_bytes;
    const float *x;           // kSplit / kCStream: rows, stride ld
    long long ld;
    const uint16_t *R;        // kRank: [tile][F][256] instance ranks
    int F;
    const unsigned char *seg; // first tree of the segment (kCStream: the blob)
    const double *weight;     // nullptr: unit weights
    const uint32_t *tree_off16;  // kCStream: tree t of the segment at 16 * tree_off16[t]
    unsigned int *slow_dev, *slow_seen_dev;  // DeviceTables::slow_dev / slow_seen_dev (may be null)
    int xshift;               // kCStream: record x offset = fid << xshift (4 B bytes per feature)
};
cudaError_t launch_combine(const double *part_sum, const uint32_t *part_key, int slices, int B,
                           long long tiles, int nchunks, int ctas, long long T, int accumulate,
                           double *out, long long n, const LeafWalk &walk, cudaStream_t stream);
// The planner's test for the balanced split (fill of the last wave of tiles).
bool balanced_split_pays(int D, long long T, long long tiles, int resident, bool has_small_batch_paths,
                         long long max_trees = 16384);
// false once the model's observed share of second-walk rows says the split does not pay
bool balanced_split_trusted(const DeviceTables *t);
bool rank_plan_ok(int F, int D, int device);
cudaError_t launch_rank_segment(const Segment &seg, const ScoreArgs &args, int device,
                                cudaStream_t stream);
cudaError_t launch_cstream(const CStreamArgs &a, int device, cudaStream_t stream);

// Launch the kernel of one segment; returns cudaSuccess or the launch error.
cudaError_t launch_segment(const Segment &seg, const ScoreArgs &args, int device,
                           cudaStream_t stream);

void count_launch();

// Cached per-device attributes (queried once; cudaDeviceGetAttribute per
// launch is measurable for small batches).
struct DevAttrs {
    int sms = 0;
    int smem_optin = 0;
};
const DevAttrs &dev_attrs(int device);
cudaMemPool_t scratch_pool(int device);  // nullptr if the device has no pool support

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when a kernel needs
// more than it was last granted.
cudaError_t ensure_smem(const void *kernel, size_t bytes);
int kernel_path();  // ts_set_kernel_path value (0 auto, 1 L1-only)

}  // namespace ts
