// Internal declarations shared by the packer, the kernels and the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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
enum Layout : int { kComplete = 0, kCompact = 1 };

struct Segment {
    int layout;   // Layout
    int depth;    // kComplete: the common depth of every tree in the segment
    int t0, t1;   // tree range [t0, t1) in evaluation order
};

struct DeviceTables {
    uint2 *nodes = nullptr;          // node records, all trees
    float *leaves = nullptr;         // kComplete leaf values, all trees
    uint32_t *node_base = nullptr;   // [T] first record of tree t
    uint32_t *leaf_base = nullptr;   // [T] first leaf of tree t (kComplete)
    int32_t *depth = nullptr;        // [T]
    double *weight = nullptr;        // [T]
};

struct HostScratch {
    float *x[2] = {nullptr, nullptr};
    double *out = nullptr;
    int32_t *status = nullptr;
    int64_t x_rows = 0, out_rows = 0;
    cudaStream_t copy = nullptr, compute = nullptr;
    cudaEvent_t copied[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
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
    std::mutex scratch_mu;
    ts::HostScratch scratch;
};

namespace ts {

void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t err, const char *what);

struct ScoreArgs {
    const float *x;
    long long n, ld;
    int F;
    const uint2 *nodes;
    const float *leaves;
    const uint32_t *node_base;
    const uint32_t *leaf_base;
    const int32_t *depth;
    const double *weight;
    int t0, t1;
    int unit_w;
    int accumulate;
    double *out;
    uint16_t *ord;
    long long ld_ord;
    int32_t *status;
};

// Launch the kernel of one segment; returns cudaSuccess or the launch error.
cudaError_t launch_segment(const Segment &seg, const ScoreArgs &args, int device,
                           cudaStream_t stream);

void count_launch();

}  // namespace ts
