// ts_cstream.cu -- shape planning and dispatch of the irregular-tree
// streaming kernel (ts_cstream_kernel.cuh; instantiations ts_cstream_w8.cu,
// ts_cstream_w16.cu).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <cstdlib>

#include "ts_internal.h"
#include "ts_cstream_kernel.cuh"

namespace ts {

namespace cstream_detail {
cudaError_t launch_w8(const CStreamArgs &a, int device, cudaStream_t stream);
cudaError_t launch_w16(const CStreamArgs &a, int device, cudaStream_t stream);
}  // namespace cstream_detail

// Kernel shape: the most lockstep chains (W walker warps x K trees) whose
// instance tile, double-buffered leaf buffer and two ring stages of
// tpc = (W / G) * K trees (~1.2 KB per 64-leaf tree) fit the opt-in shared
// memory; ties go to the larger tile (fewer tree-stream passes), then to more
// warps.  TS_CSTREAM_PLAN=G,W,K forces one shape (A/B experiments).
bool plan_cstream(int F, int device, CStreamArgs *a) {
    using namespace cstream_detail;
    const int optin = dev_attrs(device).smem_optin;
    if (!optin) return false;
    struct Cand { int G, W, K; };
    static const Cand cands[] = {{8, 8, 8}, {8, 8, 4}, {4, 8, 8}, {4, 8, 4}, {2, 8, 8},
                                 {2, 8, 4}, {1, 8, 8}, {1, 8, 4}, {2, 16, 4}, {2, 16, 3},
                                 {1, 16, 4}, {1, 16, 3}};
    int fg = 0, fw = 0, fk = 0;
    if (const char *e = getenv("TS_CSTREAM_PLAN")) sscanf(e, "%d,%d,%d", &fg, &fw, &fk);
    bool found = false;
    CStreamArgs best{};
    int best_chains = 0;
    for (const Cand &c : cands) {
        if (fg && (c.G != fg || c.W != fw || c.K != fk)) continue;
        const int B = 32 * c.G;
        const int S = c.W / c.G;
        const int tpc = std::min(S * c.K, kCStreamMaxT);
        const size_t xs = ((size_t)(F + 1) * B * 4 + 127) & ~(size_t)127;
        const size_t lb = 2 * (size_t)tpc * B * 4;  // double-buffered
        const size_t bars = 8 * 8;
        if (xs + lb + bars >= (size_t)optin) continue;
        const size_t stage = ((((size_t)optin - xs - lb - bars) / kStagesC) & ~(size_t)127);
        if (stage < kHeadBytes + (size_t)tpc * 1200) continue;
        const int chains = c.W * c.K;
        if (found && (chains < best_chains || (chains == best_chains && B <= best.B))) continue;
        found = true;
        best_chains = chains;
        best = CStreamArgs{};
        best.B = B;
        best.w = c.W;
        best.k = c.K;
        best.tpc = tpc;
        best.xs_bytes = (uint32_t)xs;
        best.lb_bytes = (uint32_t)lb;
        best.stage_bytes = (uint32_t)std::min<size_t>(stage, (size_t)tpc * 2048 + kHeadBytes);
        best.chunk_cap = best.stage_bytes - kHeadBytes;  // tree bytes per stage
    }
    if (!found) return false;
    a->B = best.B;
    a->w = best.w;
    a->k = best.k;
    a->tpc = best.tpc;
    a->xs_bytes = best.xs_bytes;
    a->lb_bytes = best.lb_bytes;
    a->stage_bytes = best.stage_bytes;
    a->chunk_cap = best.chunk_cap;
    return true;
}

cudaError_t launch_cstream(const CStreamArgs &a, int device, cudaStream_t stream) {
    if (a.n <= 0) return cudaSuccess;
    return a.w == 16 ? cstream_detail::launch_w16(a, device, stream)
                     : cstream_detail::launch_w8(a, device, stream);
}

}  // namespace ts
