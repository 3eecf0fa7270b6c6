// ts_pack.cpp -- native node-table packer (replaces the reference's per-tree
// Python recursion expand_to_complete, ref model.py:315-349, and the
// VPredicatedEvaluator build, ref evaluators.py:490-512).
//
// Input: the flat logical model of include/treescore_gpu.h.  Output: device
// tables in one of two layouts (ts_internal.h) plus the segment list the
// scorer launches in tree order.  Validation mirrors the reference's model
// checks (ref model.py:100-119 node values, :143-175 tree shape,
// :197-220 ensemble, :538-602 parser graph checks) so that a model the
// reference rejects is rejected here with the same class of error.
#include <math.h>
#include <string.h>

#include <cmath>
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "ts_internal.h"

namespace ts {
namespace {

struct TreeShape {
    int depth = 0;
    bool complete = false;
    std::vector<int32_t> bfs;    // logical ids in BFS order
    std::vector<int32_t> level;  // depth of each logical id
};

std::string tree_msg(int t, const char *what) {
    char buf[256];
    snprintf(buf, sizeof buf, "tree %d: %s", t, what);
    return buf;
}

// Structure check + depth.  Returns TS_OK or an error code (message set).
int analyse_tree(const ts_model_desc *d, int t, TreeShape *s, int max_depth) {
    const int64_t o = d->tree_node_offset[t];
    const int64_t n64 = d->tree_node_offset[t + 1] - o;
    if (n64 <= 0) return fail(TS_ERR_INVALID, tree_msg(t, "empty tree block"));
    if (n64 > (int64_t)1 << 30) return fail(TS_ERR_INVALID, tree_msg(t, "too many nodes"));
    const int32_t n = (int32_t)n64;
    const int32_t *fid = d->node_fid + o;
    const float *val = d->node_value + o;
    const int32_t *lc = d->node_left + o;
    const int32_t *rc = d->node_right + o;
    std::vector<uint8_t> parents(n, 0);
    for (int32_t i = 0; i < n; i++) {
        if (!isfinite(val[i]))
            return fail(TS_ERR_INVALID, tree_msg(t, fid[i] < 0 ? "leaf value must be finite"
                                                               : "threshold must be finite"));
        if (fid[i] < -1) return fail(TS_ERR_INVALID, tree_msg(t, "feature id must be non-negative"));
        if (fid[i] < 0) continue;
        if (fid[i] >= d->num_features)
            return fail(TS_ERR_INVALID, tree_msg(t, "feature id out of range"));
        for (int32_t c : {lc[i], rc[i]}) {
            if (c < 0 || c >= n) return fail(TS_ERR_INVALID, tree_msg(t, "dangling child id"));
            if (c == 0) return fail(TS_ERR_INVALID, tree_msg(t, "root must not appear as a child"));
            if (++parents[c] > 1) return fail(TS_ERR_INVALID, tree_msg(t, "node has multiple parents"));
        }
    }
    s->bfs.clear();
    s->bfs.reserve(n);
    s->level.assign(n, -1);
    s->bfs.push_back(0);
    s->level[0] = 0;
    int depth = 0, leaves = 0;
    for (size_t h = 0; h < s->bfs.size(); h++) {
        int32_t i = s->bfs[h];
        if (fid[i] < 0) {
            leaves++;
            depth = std::max(depth, (int)s->level[i]);
            continue;
        }
        for (int32_t c : {lc[i], rc[i]}) {
            if (s->level[c] >= 0) return fail(TS_ERR_INVALID, tree_msg(t, "cycle in tree"));
            s->level[c] = s->level[i] + 1;
            s->bfs.push_back(c);
        }
    }
    if ((int32_t)s->bfs.size() != n)
        return fail(TS_ERR_INVALID, tree_msg(t, "node unreachable from the root"));
    if (depth > max_depth) {
        char buf[160];
        snprintf(buf, sizeof buf, "tree %d: depth %d exceeds MAX_DEPTH=%d for complete-table "
                 "layouts", t, depth, max_depth);
        return fail(TS_ERR_DEPTH, buf);
    }
    s->depth = depth;
    s->complete = (int64_t)n == ((int64_t)1 << (depth + 1)) - 1 && leaves == (1 << depth);
    return TS_OK;
}

// Complete expansion to heap arrays (same slot algebra as the reference:
// children of slot i at 2i+1 and 2i+2; an early leaf becomes a dummy subtree
// of (fid 0, theta +inf) nodes whose leaves repeat its value).
void expand_heap(const int32_t *fid, const float *val, const int32_t *lc, const int32_t *rc,
                 int depth, std::vector<uint32_t> *hfid, std::vector<float> *hthr,
                 std::vector<float> *hleaf) {
    hfid->assign(((size_t)1 << depth) - 1, 0u);
    hthr->assign(((size_t)1 << depth) - 1, INFINITY);
    std::vector<int32_t> src(1, 0), nxt;
    for (int l = 0; l < depth; l++) {
        const size_t base = ((size_t)1 << l) - 1;
        nxt.resize(src.size() * 2);
        for (size_t k = 0; k < src.size(); k++) {
            int32_t i = src[k];
            if (fid[i] < 0) {
                nxt[2 * k] = nxt[2 * k + 1] = i;
            } else {
                (*hfid)[base + k] = (uint32_t)fid[i];
                (*hthr)[base + k] = val[i];
                nxt[2 * k] = lc[i];
                nxt[2 * k + 1] = rc[i];
            }
        }
        src.swap(nxt);
    }
    hleaf->resize(src.size());
    for (size_t k = 0; k < src.size(); k++) (*hleaf)[k] = val[src[k]];
}

// kComplete: (2^d - 1) records {fid << kFidShift, theta}, then the leaves.
void fill_complete(const int32_t *fid, const float *val, const int32_t *lc, const int32_t *rc,
                   int depth, unsigned char *out) {
    std::vector<uint32_t> hf;
    std::vector<float> ht, hl;
    expand_heap(fid, val, lc, rc, depth, &hf, &ht, &hl);
    uint2 *recs = reinterpret_cast<uint2 *>(out);
    for (size_t j = 0; j < hf.size(); j++) {
        recs[j].x = hf[j] << kFidShift;
        memcpy(&recs[j].y, &ht[j], 4);
    }
    memcpy(out + hf.size() * 8, hl.data(), hl.size() * 4);
}

// kSplit: see split_geom (ts_internal.h).
void fill_split(const int32_t *fid, const float *val, const int32_t *lc, const int32_t *rc,
                int depth, int fw, unsigned char *out) {
    std::vector<uint32_t> hf;
    std::vector<float> ht, hl;
    expand_heap(fid, val, lc, rc, depth, &hf, &ht, &hl);
    const SplitGeom g = split_geom(depth, fw);
    const int S = depth < kTopLevels ? depth : kTopLevels;
    uint2 *recs = reinterpret_cast<uint2 *>(out);
    for (size_t j = 0; j + 1 < ((size_t)1 << S); j++) {
        recs[j].x = hf[j] << kFidShift;
        memcpy(&recs[j].y, &ht[j], 4);
    }
    if (split_header(depth, fw)) {
        // heap levels 0-1 as the 16-byte header (ts_internal.h) in record
        // slots 0-1, slot 2 unused
        uint32_t hdr[4];
        hdr[0] = hf[0] | hf[1] << 8 | hf[2] << 16;
        memcpy(&hdr[1], &ht[0], 4);
        memcpy(&hdr[2], &ht[1], 4);
        memcpy(&hdr[3], &ht[2], 4);
        memcpy(out, hdr, 16);
        recs[2] = make_uint2(0u, 0u);
    }
    for (int l = S; l < depth; l++) {
        for (size_t i = 0; i < ((size_t)1 << l); i++) {
            const size_t heap = ((size_t)1 << l) - 1 + i;
            const size_t k = ((size_t)1 << l) - ((size_t)1 << S) + i;
            memcpy(out + g.thr0 + 4 * k, &ht[heap], 4);
            if (fw == 1) out[g.fid0 + k] = (unsigned char)hf[heap];
            else {
                const uint16_t f16 = (uint16_t)hf[heap];
                memcpy(out + g.fid0 + 2 * k, &f16, 2);
            }
        }
    }
    memcpy(out + g.leaf0, hl.data(), hl.size() * 4);
}

// kRank: 4-byte records fid << 24 | rank (see Layout), then the leaves.
// u: the feature's sorted distinct thresholds (rank = 1-based position).
void fill_rank(const int32_t *fid, const float *val, const int32_t *lc, const int32_t *rc,
               int depth, const std::vector<float> &u, const std::vector<uint32_t> &uoff,
               unsigned char *out) {
    std::vector<uint32_t> hf;
    std::vector<float> ht, hl;
    expand_heap(fid, val, lc, rc, depth, &hf, &ht, &hl);
    const RankGeom g = rank_geom(depth);
    uint32_t *recs = reinterpret_cast<uint32_t *>(out);
    for (size_t j = 0; j < hf.size(); j++) {
        uint32_t rank = kRankInf;  // dummy padding node (+inf): never taken
        if (!(std::isinf(ht[j]) && ht[j] > 0)) {
            const float th = ht[j] == 0.0f ? 0.0f : ht[j];  // -0.0 is +0.0 here
            const float *b = u.data() + uoff[hf[j]], *e = u.data() + uoff[hf[j] + 1];
            rank = (uint32_t)(std::upper_bound(b, e, th) - b);  // its own 1-based position
        }
        recs[j] = hf[j] << 24 | rank;
    }
    memcpy(out + g.leaf0, hl.data(), hl.size() * 4);
}

// Compact BFS layout with adjacent sibling pairs and self-loop leaves.
// xstride 0: kCompact {fid | left << 16, theta}; xstride 4B: kCStream
// {(xstride * fid) << 14 | left, theta} (ts_internal.h).
void fill_compact(const int32_t *fid, const float *val, const int32_t *lc, const int32_t *rc,
                  const TreeShape &s, int F, uint2 *nodes, uint32_t xstride) {
    const int32_t n = (int32_t)s.bfs.size();
    std::vector<int32_t> newid(n, -1);
    std::vector<int32_t> order;
    order.reserve(n);
    order.push_back(0);
    newid[0] = 0;
    for (size_t h = 0; h < order.size(); h++) {
        int32_t i = order[h];
        if (fid[i] < 0) continue;
        newid[lc[i]] = (int32_t)order.size();
        order.push_back(lc[i]);
        newid[rc[i]] = (int32_t)order.size();
        order.push_back(rc[i]);
    }
    for (int32_t k = 0; k < n; k++) {
        int32_t i = order[k];
        uint2 rec;
        memcpy(&rec.y, &val[i], 4);
        const uint32_t f = fid[i] < 0 ? (uint32_t)F : (uint32_t)fid[i];
        const uint32_t left = fid[i] < 0 ? (uint32_t)k : (uint32_t)newid[lc[i]];
        rec.x = xstride ? (xstride * f) << 14 | left : f | left << 16;
        nodes[k] = rec;
    }
}

template <class T>
int upload(T **dptr, const std::vector<T> &h) {
    size_t bytes = std::max<size_t>(1, h.size()) * sizeof(T);
    cudaError_t e = cudaMalloc((void **)dptr, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(model tables)");
    if (!h.empty()) {
        e = cudaMemcpy(*dptr, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(model tables)");
    }
    return TS_OK;
}

}  // namespace

void free_tables(DeviceTables *t) {
    cudaFree(t->blob);
    cudaFree(t->tree_off16);
    cudaFree(t->depth);
    cudaFree(t->weight);
    cudaFree(t->trace_nodes);
    cudaFree(t->trace_base);
    cudaFree(t->chunk_info);
    cudaFree(t->slot_meta);
    cudaFree(t->slow_dev);
    cudaFreeHost(t->slow_seen);
    for (RankSpace &r : t->rank_spaces) {
        cudaFree(r.e);
        cudaFree(r.eoff);
        cudaFree(r.groups);
    }
    *t = DeviceTables{};
}

}  // namespace ts

extern "C" int ts_pack(const ts_model_desc *d, int device, ts_model **out) {
    return ts_pack_ex(d, device, 0, out);
}

extern "C" int ts_pack_ex(const ts_model_desc *d, int device, int flags, ts_model **out) {
    using namespace ts;
    if (!out) return fail(TS_ERR_INVALID, "out is NULL");
    *out = nullptr;
    if (!d || !d->tree_node_offset || !d->tree_weight || !d->node_fid || !d->node_value ||
        !d->node_left || !d->node_right)
        return fail(TS_ERR_INVALID, "model description has NULL arrays");
    if (d->num_features < 1) return fail(TS_ERR_INVALID, "num_features must be positive");
    if (d->num_trees < 1) return fail(TS_ERR_INVALID, "ensemble must contain at least one tree");
    if (d->tree_node_offset[0] != 0) return fail(TS_ERR_INVALID, "tree_node_offset[0] must be 0");
    const int T = d->num_trees, F = d->num_features;
    // Compact records hold fid and the sentinel row F in 16 bits.
    const bool compact_ok_f = F <= 65534;

    // Which complete depths the shared-memory streaming kernel can run on this
    // device (instance tile + 3 ring stages fit); those trees get kSplit.
    int prev_dev = -1;
    cudaGetDevice(&prev_dev);
    bool split_ok[TS_MAX_DEPTH + 1] = {};
    if (kernel_path() == 0 && cudaSetDevice(device) == cudaSuccess) {
        for (int dd = 0; dd <= TS_MAX_DEPTH; dd++) {
            StreamArgs probe{};
            split_ok[dd] = plan_stream(F, dd, device, &probe);
        }
    }
    CStreamArgs cplan{};
    const bool cstream_ok = kernel_path() == 0 && compact_ok_f &&
                            cudaSetDevice(device) == cudaSuccess &&
                            plan_cstream(F, device, &cplan);
    if (prev_dev >= 0) cudaSetDevice(prev_dev);
    const int fw = split_fid_width(F);

    // TS_FORCE_CSTREAM: pack complete trees as kCStream too (tests / A/B only)
    const bool force_cs = getenv("TS_FORCE_CSTREAM") != nullptr;
    std::vector<TreeShape> shapes(T);
    std::vector<int> layout(T);
    int64_t sum_depth = 0, entries = 0;
    int max_depth = 0, n_complete = 0, n_compact = 0;
    bool unit = true;
    for (int t = 0; t < T; t++) {
        if (!isfinite(d->tree_weight[t]))
            return fail(TS_ERR_INVALID, tree_msg(t, "tree weight must be finite"));
        if (d->tree_weight[t] != 1.0) unit = false;
        int rc = analyse_tree(d, t, &shapes[t],
                              (flags & TS_PACK_ANY_DEPTH) ? TS_MAX_LINKED_DEPTH : TS_MAX_DEPTH);
        if (rc) return rc;
        const TreeShape &s = shapes[t];
        const int64_t nn = (int64_t)s.bfs.size();
        if (s.depth > TS_MAX_DEPTH && (!compact_ok_f || nn > 65535))
            return fail(TS_ERR_DEPTH, tree_msg(t, "deeper than MAX_DEPTH and too large for the "
                                                  "child-index layout"));
        const bool deep = s.depth > TS_MAX_DEPTH;  // no complete table: child-index records
        const uint64_t tb = ((uint64_t)nn * 8u + 15u) & ~(uint64_t)15u;
        const bool cs_fits = cstream_ok && nn <= kCStreamMaxNodes && tb <= cplan.chunk_cap;
        // Complete trees stream as kSplit; when their rows are too wide for the
        // complete-tree kernel's tile (e.g. F = 700) the irregular kernel's
        // 32-row tiles still fit, and beat the L1 path (4.4x at F=700, d=8).
        const bool complete_form = !deep && ((s.complete && !force_cs) || !compact_ok_f ||
                                             nn > 65535);
        if (complete_form && (split_ok[s.depth] || !cs_fits || !s.complete)) {
            layout[t] = split_ok[s.depth] ? kSplit : kComplete;
            n_complete++;
        } else {
            layout[t] = cs_fits ? kCStream : kCompact;
            n_compact++;
        }
        sum_depth += s.depth;
        entries += ((int64_t)1 << (s.depth + 1)) - 1;
        max_depth = std::max(max_depth, s.depth);
    }
    // Blob layout: tree t at 16 * tree_off16[t] (see DeviceTables).
    // Rank layout (ts_rank.cu) for complete trees where it measured faster:
    // the instance-rank pre-pass costs ~1.4 ms per 1M rows x 136 features
    // whatever the ensemble, the walk saves per tree -- a lot where the fp32
    // layouts are capacity-starved (d = 12) or have only the L1 path (d =
    // 13-14), little at d = 10-11, nothing below (profiles/r2_rank_layout.txt).
    // So a depth takes the rank layout when it has at least kRankMinTrees[d] x
    // F / 136 trees (the break-even, rounded up), and every feature has <=
    // kRankMaxU distinct thresholds among them.  TS_RANK_MIN_DEPTH=d forces it
    // for all depths >= d (tests); TS_RANK=0 or TS_PACK_NO_RANK never.
    struct RankHost {
        std::vector<float> u;        // sorted distinct thresholds, feature-major
        std::vector<uint32_t> off;   // [F + 1]
    };
    std::vector<RankHost> rank_hosts;
    std::vector<int> space_of(T, -1);
    {
        const char *re = getenv("TS_RANK");
        const char *rd = getenv("TS_RANK_MIN_DEPTH");
        const int forced_d = rd ? atoi(rd) : -1;
        bool want = !(flags & TS_PACK_NO_RANK) && F <= 256 && !(re && atoi(re) == 0) &&
                    kernel_path() == 0;
        bool rank_ok[TS_MAX_DEPTH + 1] = {};
        if (want && cudaSetDevice(device) == cudaSuccess) {
            for (int dd = 1; dd <= kRankMaxDepth; dd++) rank_ok[dd] = rank_plan_ok(F, dd, device);
            if (prev_dev >= 0) cudaSetDevice(prev_dev);
        }
        int count[TS_MAX_DEPTH + 1] = {};
        for (int t = 0; want && t < T; t++)
            if ((layout[t] == kSplit || layout[t] == kComplete) && rank_ok[shapes[t].depth])
                count[shapes[t].depth]++;
        static const int kRankMinTrees[kRankMaxDepth + 1] = {0, 0, 0, 0, 0, 0, 0, 0,
                                                             0, 0, 2000, 1500, 500, 150, 300};
        bool use_d[TS_MAX_DEPTH + 1] = {};
        for (int dd = 1; dd <= kRankMaxDepth; dd++) {
            if (!rank_ok[dd] || !count[dd]) continue;
            if (forced_d >= 0) use_d[dd] = dd >= forced_d;
            else use_d[dd] = kRankMinTrees[dd] > 0 &&
                             (int64_t)count[dd] * 136 >= (int64_t)kRankMinTrees[dd] * F;
        }
        auto rank_tree = [&](int t) {
            return (layout[t] == kSplit || layout[t] == kComplete) && use_d[shapes[t].depth];
        };
        // Rank spaces: consecutive runs of rank trees whose thresholds stay
        // <= kRankMaxU per feature.  A space closes when the run's NODE count
        // for some feature would pass the limit (an upper bound of its
        // distinct thresholds, so no space overflows; repeated thresholds
        // only make spaces smaller than they need be), then its lists are
        // sorted and deduplicated once.
        std::vector<std::vector<float>> per(F);   // the open space's values
        std::vector<uint32_t> used(F, 0u);
        auto close_space = [&]() {
            RankHost h;
            h.off.assign(F + 1, 0u);
            {
                auto su = [&](int f0, int f1) {
                    for (int f = f0; f < f1; f++) {
                        std::sort(per[f].begin(), per[f].end());
                        per[f].erase(std::unique(per[f].begin(), per[f].end()), per[f].end());
                    }
                };
                const int nth = (int)std::min<unsigned>(
                    (unsigned)F, std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
                std::vector<std::thread> th;
                for (int k = 0; k < nth; k++)
                    th.emplace_back(su, F * k / nth, F * (k + 1) / nth);
                for (auto &x : th) x.join();
            }
            for (int f = 0; f < F; f++) h.off[f + 1] = h.off[f] + (uint32_t)per[f].size();
            h.u.reserve(h.off[F]);
            for (int f = 0; f < F; f++) {
                h.u.insert(h.u.end(), per[f].begin(), per[f].end());
                per[f].clear();
                used[f] = 0u;
            }
            rank_hosts.push_back(std::move(h));
        };
        std::vector<uint32_t> cnt(F);
        bool open = false;
        for (int t = 0; want && t < T; t++) {
            if (!rank_tree(t)) continue;
            const int64_t o = d->tree_node_offset[t], nn = d->tree_node_offset[t + 1] - o;
            std::fill(cnt.begin(), cnt.end(), 0u);
            for (int64_t i = 0; i < nn; i++)
                if (d->node_fid[o + i] >= 0) cnt[d->node_fid[o + i]]++;
            bool fits = true;
            for (int f = 0; f < F && fits; f++) fits = used[f] + cnt[f] <= (uint32_t)kRankMaxU;
            if (!fits && open) {
                close_space();
                open = false;
            }
            for (int64_t i = 0; i < nn; i++) {
                const int32_t f = d->node_fid[o + i];
                if (f < 0) continue;
                const float v = d->node_value[o + i];
                per[f].push_back(v == 0.0f ? 0.0f : v);
            }
            for (int f = 0; f < F; f++) used[f] += cnt[f];
            space_of[t] = (int)rank_hosts.size();
            open = true;
        }
        if (open) close_space();
        for (int t = 0; t < T; t++)
            if (space_of[t] >= 0) layout[t] = kRank;
    }
    std::vector<uint64_t> off(T + 1, 0);
    for (int t = 0; t < T; t++) {
        uint64_t bytes = layout[t] == kComplete ? complete_tree_bytes(shapes[t].depth)
                         : layout[t] == kRank ? rank_geom(shapes[t].depth).bytes
                         : layout[t] == kSplit ? split_geom(shapes[t].depth, fw).bytes
                         : ((uint64_t)shapes[t].bfs.size() * 8u + 15u) & ~(uint64_t)15u;
        off[t + 1] = off[t] + bytes;
    }
    if (off[T] / 16 >= ((uint64_t)1 << 32))
        return fail(TS_ERR_UNSUPPORTED, "packed tables exceed 64 GiB");
    std::vector<unsigned char> blob(off[T], 0);
    std::vector<uint32_t> off16(T);
    std::vector<int32_t> depth(T);
    std::vector<double> weight(d->tree_weight, d->tree_weight + T);
    // Trees fill disjoint byte ranges of the blob: several host threads for
    // big ensembles (config 4b: 20,000 depth-10 trees)
    auto fill = [&](int t0, int t1) {
        for (int t = t0; t < t1; t++) {
            const int64_t o = d->tree_node_offset[t];
            const int32_t *fid = d->node_fid + o;
            const float *val = d->node_value + o;
            const int32_t *lc = d->node_left + o;
            const int32_t *rcc = d->node_right + o;
            off16[t] = (uint32_t)(off[t] / 16);
            depth[t] = shapes[t].depth;
            unsigned char *dst = blob.data() + off[t];
            if (layout[t] == kComplete)
                fill_complete(fid, val, lc, rcc, shapes[t].depth, dst);
            else if (layout[t] == kSplit)
                fill_split(fid, val, lc, rcc, shapes[t].depth, fw, dst);
            else if (layout[t] == kRank)
                fill_rank(fid, val, lc, rcc, shapes[t].depth, rank_hosts[space_of[t]].u,
                          rank_hosts[space_of[t]].off, dst);
            else
                fill_compact(fid, val, lc, rcc, shapes[t], F, reinterpret_cast<uint2 *>(dst),
                             layout[t] == kCStream ? 4u * (uint32_t)cplan.B : 0u);
        }
    };
    {
        const int64_t nodes = d->tree_node_offset[T];
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const int nth = nodes < (1 << 20) ? 1 : (int)std::min<unsigned>(16u, hw);
        if (nth == 1) {
            fill(0, T);
        } else {
            std::vector<std::thread> th;
            for (int k = 0; k < nth; k++)
                th.emplace_back(fill, (int)((int64_t)T * k / nth), (int)((int64_t)T * (k + 1) / nth));
            for (auto &x : th) x.join();
        }
    }

    ts_model *m = new ts_model();
    m->device = device;
    m->num_features = F;
    m->num_trees = T;
    m->unit_weights = unit;
    for (int t = 0; t < T; t++) {
        const bool any_depth = layout[t] == kCompact || layout[t] == kCStream;
        const int key_depth = any_depth ? -1 : shapes[t].depth;
        const int space = layout[t] == kRank ? space_of[t] : 0;
        if (!m->segments.empty()) {
            Segment &b = m->segments.back();
            if (b.layout == layout[t] && (any_depth || b.depth == key_depth) &&
                b.rank_space == space) {
                b.t1 = t + 1;
                continue;
            }
        }
        m->segments.push_back(Segment{layout[t], any_depth ? max_depth : key_depth, t, t + 1,
                                      off[t]});
        m->segments.back().rank_space = space;
    }
    // Streaming segments: how often a row's tree-order sum may round (see
    // Segment::slow_rows).  The running sums of a row stay below about
    // M = 4 sqrt(sum_t mean(leaf_t^2)) + sum_t |mean(leaf_t)|; an add is exact
    // while the leaf's LSB, 2^(e - 23), is no finer than 2^(m - 53) with M <
    // 2^m, i.e. |leaf| >= 2^(m - 30).  A row meets T leaves, so about
    // T x (share of nonzero leaves below that) of the rows are not provably
    // exact -- 2e-4 for N(0,1) leaves at T = 1000, most rows for leaves
    // spread over many decades.
    for (Segment &sg : m->segments) {
        if (sg.layout != kSplit && sg.layout != kRank && sg.layout != kCStream) continue;
        double sum_ms = 0.0, sum_mean = 0.0;
        std::vector<double> mags;
        for (int t = sg.t0; t < sg.t1; t++) {
            const int64_t o = d->tree_node_offset[t], e = d->tree_node_offset[t + 1];
            double s1 = 0.0, s2 = 0.0;
            int64_t nl = 0;
            for (int64_t i = o; i < e; i++) {
                if (d->node_fid[i] >= 0) continue;
                const double v = d->node_value[i];
                s1 += v;
                s2 += v * v;
                nl++;
                if (v != 0.0) mags.push_back(fabs(v));
            }
            if (nl) {
                sum_ms += s2 / nl;
                sum_mean += fabs(s1 / nl);
            }
        }
        const double M = 4.0 * sqrt(sum_ms) + sum_mean;
        if (mags.empty() || !(M > 0.0)) continue;
        const double thr = ldexp(M, 1 - 30);
        size_t tiny = 0;
        for (double v : mags) tiny += v < thr;
        sg.slow_rows = (float)std::min(1.0, (double)(sg.t1 - sg.t0) * tiny / mags.size());
    }
    // kCStream chunk tables: consecutive trees up to tpc / chunk_cap bytes;
    // inside a chunk the slots are ordered by depth (deepest first) so the
    // kernel's lockstep K-groups walk trees of nearly equal depth.
    std::vector<uint4> chunk_info;
    std::vector<uint32_t> slot_meta;
    for (Segment &sg : m->segments) {
        if (sg.layout != kCStream) continue;
        sg.chunk0 = (int)chunk_info.size();
        sg.cs_b = cplan.B;
        int t = sg.t0;
        while (t < sg.t1) {
            int e = t;
            while (e < sg.t1 && e - t < cplan.tpc && off[e + 1] - off[t] <= cplan.chunk_cap) e++;
            const int nt = e - t;
            chunk_info.push_back(make_uint4((uint32_t)(off[t] / 16), (uint32_t)(off[e] - off[t]),
                                            (uint32_t)nt, (uint32_t)t));
            std::vector<int> order(nt);
            for (int i = 0; i < nt; i++) order[i] = i;
            std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
                return shapes[t + x].depth > shapes[t + y].depth;
            });
            const size_t base = slot_meta.size();
            slot_meta.resize(base + kCStreamMaxT, 0u);
            for (int sl = 0; sl < nt; sl++) {
                const int rel = order[sl];
                const uint32_t rec8 = (uint32_t)((off[t + rel] - off[t]) / 8);
                slot_meta[base + sl] = rec8 | ((uint32_t)shapes[t + rel].depth << 16) |
                                       ((uint32_t)rel << 21);
            }
            t = e;
        }
        sg.nchunks = (int)chunk_info.size() - sg.chunk0;
    }
    int prev = -1;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        delete m;
        return cuda_fail(e, "cudaSetDevice");
    }
    int rc = upload(&m->dev.blob, blob);
    if (!rc) rc = upload(&m->dev.tree_off16, off16);
    if (!rc) rc = upload(&m->dev.depth, depth);
    if (!rc) rc = upload(&m->dev.weight, weight);
    if (!rc) rc = upload(&m->dev.chunk_info, chunk_info);
    if (!rc) rc = upload(&m->dev.slot_meta, slot_meta);
    if (!rc) {  // second-walk counters (DeviceTables::slow_dev / slow_seen); optional
        if (cudaMalloc((void **)&m->dev.slow_dev, 2 * sizeof(unsigned int)) != cudaSuccess ||
            cudaMemset(m->dev.slow_dev, 0, 2 * sizeof(unsigned int)) != cudaSuccess ||
            cudaHostAlloc((void **)&m->dev.slow_seen, 2 * sizeof(unsigned int), cudaHostAllocMapped) !=
                cudaSuccess ||
            cudaHostGetDevicePointer((void **)&m->dev.slow_seen_dev, m->dev.slow_seen, 0) != cudaSuccess) {
            (void)cudaGetLastError();
            cudaFree(m->dev.slow_dev);
            cudaFreeHost(m->dev.slow_seen);
            m->dev.slow_dev = nullptr;
            m->dev.slow_seen = m->dev.slow_seen_dev = nullptr;
        } else {
            m->dev.slow_seen[0] = m->dev.slow_seen[1] = 0u;
        }
    }
    for (size_t sp = 0; !rc && sp < rank_hosts.size(); sp++) {
        // Eytzinger trees of the space's sorted lists (see RankSpace), and the
        // pre-pass's feature groups: consecutive features whose trees share
        // one CTA's shared memory
        const std::vector<float> &rank_u = rank_hosts[sp].u;
        const std::vector<uint32_t> &rank_off = rank_hosts[sp].off;
        std::vector<uint32_t> eoff(F + 1, 0u);
        for (int f = 0; f < F; f++) {
            const uint32_t m_f = rank_off[f + 1] - rank_off[f];
            uint32_t L = 0;
            while (((1u << L) - 1u) < m_f) L++;
            eoff[f + 1] = eoff[f] + ((1u << L) - 1u);
        }
        std::vector<float> et(eoff[F] + 8, INFINITY);  // the pre-pass reads whole 16-byte granules
        for (int f = 0; f < F; f++) {
            const uint32_t n_f = eoff[f + 1] - eoff[f], m_f = rank_off[f + 1] - rank_off[f];
            // in-order traversal of the complete BST = sorted order
            uint32_t next = 0;
            std::vector<uint32_t> stack;
            uint32_t i = 0;
            while (i < n_f || !stack.empty()) {
                while (i < n_f) {
                    stack.push_back(i);
                    i = 2 * i + 1;
                }
                i = stack.back();
                stack.pop_back();
                et[eoff[f] + i] = next < m_f ? rank_u[rank_off[f] + next] : INFINITY;
                next++;
                i = 2 * i + 2;
            }
        }
        std::vector<int2> groups;
        // <= 40 KB per group (a feature's tree alone may be bigger): several
        // pre-pass CTAs per SM hide the heap walk's load latency better than
        // fewer, wider groups reading each row fewer times (d = 10, 1M rows:
        // 160 KB groups 1.5 ms, 72 KB 1.3 ms, 40 KB 1.1 ms)
        constexpr uint32_t kMaxWords = 40 * 1024 / 4 - 8;
        int f0 = 0;
        uint32_t maxw = 0;
        for (int f = 0; f <= F; f++) {
            if (f == F || (f > f0 && eoff[f + 1] - eoff[f0] + 3 > kMaxWords)) {
                groups.push_back(int2{f0, f});
                maxw = std::max(maxw, eoff[f] - eoff[f0] + 8u);  // + 16-byte alignment lead and tail
                f0 = f;
            }
        }
        m->dev.rank_spaces.emplace_back();
        RankSpace &r = m->dev.rank_spaces.back();
        rc = upload(&r.e, et);
        if (!rc) rc = upload(&r.eoff, eoff);
        if (!rc) rc = upload(&r.groups, groups);
        r.ngroups = (int)groups.size();
        r.group_words = maxw;
    }
    if (!rc && (flags & TS_PACK_TRACE)) {
        // logical trees for the tracer: file-order nodes, leaf ordinals left-to-right
        std::vector<TraceNode> tn(d->tree_node_offset[T]);
        std::vector<uint32_t> tbase(T);
        for (int t = 0; t < T; t++) {
            const int64_t o = d->tree_node_offset[t], n = d->tree_node_offset[t + 1] - o;
            tbase[t] = (uint32_t)o;
            for (int64_t i = 0; i < n; i++) {
                TraceNode &x = tn[o + i];
                x.fid = d->node_fid[o + i];
                x.value = d->node_value[o + i];
                x.left = x.fid >= 0 ? d->node_left[o + i] : 0;
                x.right = x.fid >= 0 ? d->node_right[o + i] : 0;
            }
            int32_t ord = 0;  // depth-first, left child first
            std::vector<int32_t> stack(1, 0);
            while (!stack.empty()) {
                int32_t i = stack.back();
                stack.pop_back();
                if (tn[o + i].fid < 0) {
                    tn[o + i].left = ord++;
                } else {
                    stack.push_back(tn[o + i].right);
                    stack.push_back(tn[o + i].left);
                }
            }
        }
        if (d->tree_node_offset[T] >= ((int64_t)1 << 32)) rc = fail(TS_ERR_UNSUPPORTED, "too many nodes to trace");
        if (!rc) rc = upload(&m->dev.trace_nodes, tn);
        if (!rc) rc = upload(&m->dev.trace_base, tbase);
    }
    if (prev >= 0) cudaSetDevice(prev);
    if (rc) {
        free_tables(&m->dev);
        delete m;
        return rc;
    }
    ts_model_info &info = m->info;
    info.num_features = F;
    info.num_trees = T;
    info.max_depth = max_depth;
    info.num_segments = (int32_t)m->segments.size();
    info.sum_depth = sum_depth;
    info.table_entries = entries;
    info.device_bytes = (int64_t)off[T] + (int64_t)T * (4 + 4 + 8);
    info.complete_trees = n_complete;
    info.compact_trees = n_compact;
    info.device = device;
    info.unit_weights = unit ? 1 : 0;
    info.rank_trees = (int32_t)std::count(layout.begin(), layout.end(), (int)kRank);
    *out = m;
    return TS_OK;
}
