// ts_trace.cu -- GPU traced prediction / feature coverage.
//
// Restates the reference's predict_ensemble_traced (ref evaluators.py:599-620)
// and measure_feature_coverage (ref bench.py:412-427) for whole batches: per
// instance, the union of feature ids on its root-to-leaf paths in every
// LOGICAL tree (dummy padding nodes never exist there), the left-to-right
// (logical) leaf ordinal per tree, and the score (f64, tree order).  This is
// an analysis path, not the hot path: one thread per instance walks the
// packed logical trees through L1 (left iff x < theta, the reference rule)
// and ORs feature bits into a per-thread bitset held in registers, written
// to its row of the output once (r2; r1 did a global read-modify-write per
// visit: profiles/r2_trace.txt has the timings).
#include <cuda_runtime.h>
#include <stdint.h>

#include "ts_internal.h"

namespace ts {
namespace {

// Rows with F <= 32 * W keep their visited-feature bitset in W registers
// (a compile-time word count; each visit ORs its bit into word fid >> 5
// through W predicated LOPs -- no memory traffic) and write it out once per
// row; wider rows OR into the output directly (W = 0).
constexpr int kTraceThreads = 256;

template <int W>
__global__ void __launch_bounds__(kTraceThreads)
    k_trace(const float *__restrict__ x, long long n, long long ld,
            const TraceNode *__restrict__ nodes, const uint32_t *__restrict__ tree_base,
            const double *__restrict__ weight, int T, int unit_w, double *out,
            uint16_t *leaf_ord, long long ld_ord, uint32_t *visited, int words) {
    for (long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x; row < n;
         row += (long long)gridDim.x * blockDim.x) {
        const float *xr = x + row * ld;
        uint32_t *bits = visited ? visited + row * words : nullptr;
        uint32_t b[W > 0 ? W : 1];
#pragma unroll
        for (int w = 0; w < (W > 0 ? W : 1); w++) b[w] = 0u;
        if (W == 0 && bits)
            for (int w = 0; w < words; w++) bits[w] = 0u;
        double acc = 0.0;
        for (int t = 0; t < T; t++) {
            const TraceNode *nd = nodes + __ldg(tree_base + t);
            TraceNode q = nd[0];
            while (q.fid >= 0) {
                if constexpr (W > 0) {
                    const uint32_t hi = (uint32_t)q.fid >> 5, bit = 1u << (q.fid & 31);
#pragma unroll
                    for (int w = 0; w < W; w++) b[w] |= hi == (uint32_t)w ? bit : 0u;
                } else if (bits) {
                    bits[q.fid >> 5] |= 1u << (q.fid & 31);
                }
                q = nd[__ldg(xr + q.fid) < q.value ? q.left : q.right];
            }
            acc = unit_w ? __dadd_rn(acc, (double)q.value)
                         : __dadd_rn(acc, __dmul_rn(__ldg(weight + t), (double)q.value));
            if (leaf_ord) leaf_ord[(long long)t * ld_ord + row] = (uint16_t)q.left;
        }
        if (W > 0 && bits)
#pragma unroll
            for (int w = 0; w < (W > 0 ? W : 1); w++)
                if (w < words) bits[w] = b[w];
        if (out) out[row] = acc;
    }
}

}  // namespace
}  // namespace ts

using namespace ts;

extern "C" int ts_trace(const ts_model *m, const float *x, int64_t n, int64_t f, int64_t ld,
                        double *out, uint16_t *leaf_ord, int64_t ld_ord, uint32_t *visited,
                        int32_t words, void *stream) {
    if (!m) return fail(TS_ERR_INVALID, "model is NULL");
    if (!m->dev.trace_nodes)
        return fail(TS_ERR_UNSUPPORTED, "model was packed without TS_PACK_TRACE");
    if (f != m->num_features || ld < f || n < 0) return fail(TS_ERR_SHAPE, "bad instance shape");
    if (visited && words < (m->num_features + 31) / 32)
        return fail(TS_ERR_SHAPE, "visited needs ceil(F/32) words per row");
    if (leaf_ord && ld_ord < n) return fail(TS_ERR_SHAPE, "ld_ord must be >= n");
    if (n == 0) return TS_OK;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != m->device) cudaSetDevice(m->device);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device);
    const long long blocks = (n + kTraceThreads - 1) / kTraceThreads;
    const int grid = (int)(blocks < 8LL * sms ? blocks : 8LL * sms);
    const int w = visited ? words : 0;
    auto go = [&](auto kern) {
        kern<<<grid, kTraceThreads, 0, (cudaStream_t)stream>>>(
            x, n, ld, m->dev.trace_nodes, m->dev.trace_base, m->dev.weight, m->num_trees,
            m->unit_weights ? 1 : 0, out, leaf_ord, ld_ord, visited, words);
    };
    if (w == 0) go(k_trace<1>);  // no bitset: one dead register word
    else if (w <= 2) go(k_trace<2>);
    else if (w <= 5) go(k_trace<5>);
    else if (w <= 8) go(k_trace<8>);
    else if (w <= 16) go(k_trace<16>);
    else if (w <= 24) go(k_trace<24>);
    else go(k_trace<0>);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (prev >= 0 && prev != m->device) cudaSetDevice(prev);
    return e == cudaSuccess ? TS_OK : cuda_fail(e, "trace kernel launch");
}
