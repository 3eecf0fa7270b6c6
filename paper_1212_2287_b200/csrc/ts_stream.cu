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

namespace {
using StreamFn = cudaError_t (*)(const StreamArgs &, int, cudaStream_t);
const StreamFn kStreamTable[kStreamMaxDepth + 1] = {
    launch_d<0>, launch_d<1>, launch_d<2>, launch_d<3>, launch_d<4>, launch_d<5>,
    launch_d<6>, launch_d<7>, launch_d<8>, launch_d<9>, launch_d<10>, launch_d<11>, launch_d<12>};

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
    const uint32_t tb = a->tree_bytes;
    const size_t bars = 2 * kMaxStages * 8;
    if (xs + bars + (size_t)2 * tb > (size_t)optin) return false;
    const size_t ring = (size_t)optin - xs - bars;
    const uint32_t K = chains_for_depth(D);
    const size_t group = (size_t)K * tb;
    int stages = 0;
    uint32_t tpc = 0;
    for (int s = kMaxStages; s >= 2 && !stages; s--) {
        size_t cap = ring / s;
        if (cap < group) continue;
        size_t g = cap / group;
        const size_t soft = 48 * 1024;   // small chunks keep the ring turning over
        if (g > 1 && g * group > soft) g = std::max<size_t>(1, soft / group);
        stages = s;
        tpc = (uint32_t)(g * K);
    }
    if (!stages) {
        if (cw != 8) return false;  // the 256-row shape handles it better
        stages = 2;                 // not even two K-groups fit: single trees
        tpc = (uint32_t)std::max<size_t>(1, (ring / 2) / tb);
    }
    a->cw = cw;
    a->xs_bytes = (uint32_t)xs;
    a->tpc = (int)tpc;
    a->stages = stages;
    a->chunk_cap = (tpc * tb + 127) & ~127u;
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

cudaError_t launch_stream(int D, const StreamArgs &a, int device, cudaStream_t stream) {
    if (a.n <= 0) return cudaSuccess;
    return stream_detail::kStreamTable[D](a, device, stream);
}

}  // namespace ts
