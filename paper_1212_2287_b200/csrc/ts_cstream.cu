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

// Kernel shape: the most lockstep chains that actually walk (G row groups x
// min(S*K, trees per chunk), S = W/G walker warps per group, chunks of at
// most 64 trees) whose instance tile, double-buffered leaf buffer and >= 2
// ring stages of tpc trees (~1.2 KB per 64-leaf tree) fit the opt-in shared
// memory.  Ties go to the smaller K (less lockstep padding), then more
// stages (up to 3), then two row groups, then more warps.  r1 session 2
// (tools/irregular_shapes.py, 500k rows x 2000 trees): the old key (W*K)
// picked 1x16x8 at F = 256 / 400, whose 128 slots half-idle on 64-tree
// chunks (6.41 / 6.52 ms); this one picks 2x16x4 (5.44 / 5.60 ms), and
// 2x16x8 at F = 136 (4.99 vs 5.15 ms); F = 700 (config 3) stays 1x16x3.  Two teams on alternate chunks of S*K/2 trees (smaller
// stages, more of them in flight) are only a fallback: on config 3 the
// 16x4 two-team shape ran 58.8 ms against 57.8 ms for 16x3 with one team
// (per-chunk overhead is paid per half as much work).
// TS_CSTREAM_PLAN=G,W,K[,teams] forces a shape (A/B experiments).
bool plan_cstream(int F, int device, CStreamArgs *a) {
    using namespace cstream_detail;
    const int optin = dev_attrs(device).smem_optin;
    if (!optin) return false;
    struct Cand { int G, W, K; };
    static const Cand cands[] = {{8, 8, 8}, {8, 8, 4}, {4, 8, 8}, {4, 8, 4}, {2, 8, 8},
                                 {2, 8, 4}, {1, 8, 8}, {1, 8, 4}, {4, 16, 8}, {4, 16, 4},
                                 {2, 16, 8}, {2, 16, 4}, {2, 16, 3}, {1, 16, 8}, {1, 16, 4},
                                 {1, 16, 3}, {1, 16, 2}};
    int fg = 0, fw = 0, fk = 0, ft = 0;
    if (const char *e = getenv("TS_CSTREAM_PLAN")) sscanf(e, "%d,%d,%d,%d", &fg, &fw, &fk, &ft);
    bool found = false;
    CStreamArgs best{};
    long best_key = -1;
    for (const Cand &c : cands) {
        if (fg && (c.G != fg || c.W != fw || c.K != fk)) continue;
        for (int teams = 1; teams <= 2; teams++) {
            if (ft && teams != ft) continue;
            const int B = 32 * c.G;
            const int S = c.W / c.G;
            if (S % teams) continue;
            const int tpc = std::min(S * c.K / teams, kCStreamMaxT);
            const size_t xs = ((size_t)(F + 1) * B * 4 + 127) & ~(size_t)127;
            const size_t lb = 2 * (size_t)tpc * B * 4;  // double-buffered
            const size_t bars = (2 * kMaxStagesC + 4) * 8;
            if (xs + lb + bars >= (size_t)optin) continue;
            const size_t need = kHeadBytes + (size_t)tpc * 1200;   // one chunk of trees
            const size_t room = (size_t)optin - xs - lb - bars;
            const int stages = (int)std::min<size_t>(kMaxStagesC, room / ((need + 127) & ~(size_t)127));
            if (stages < 2) continue;
            const size_t stage = std::min<size_t>((room / stages) & ~(size_t)127,
                                                  (size_t)tpc * 2048 + kHeadBytes);
            // chains that actually walk: a chunk holds tpc <= 64 trees, so S
            // warps x K of a row group only all work while S * K <= tpc
            const long eff = (long)c.G * std::min(S * c.K, teams * tpc);
            const long key = (2 - teams) * 1000000000L + eff * 1000000 + (16 - c.K) * 10000 +
                             std::min(stages, 3) * 1000 + (c.G == 2 ? 100 : 0) + c.W;
            if (found && key <= best_key) continue;
            found = true;
            best_key = key;
            best = CStreamArgs{};
            best.B = B;
            best.w = c.W;
            best.k = c.K;
            best.tpc = tpc;
            best.stages = stages;
            best.teams = teams;
            best.xs_bytes = (uint32_t)xs;
            best.lb_bytes = (uint32_t)lb;
            best.stage_bytes = (uint32_t)stage;
            best.chunk_cap = best.stage_bytes - kHeadBytes;  // tree bytes per stage
        }
    }
    if (!found) return false;
    a->B = best.B;
    a->w = best.w;
    a->k = best.k;
    a->tpc = best.tpc;
    a->stages = best.stages;
    a->teams = best.teams;
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
