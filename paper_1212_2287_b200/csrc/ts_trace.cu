// ts_trace.cu -- GPU traced prediction / feature coverage.
//
// Restates the reference's predict_ensemble_traced (ref evaluators.py:599-620)
// and measure_feature_coverage (ref bench.py:412-427) for whole batches: per
// instance, the union of feature ids on its root-to-leaf paths in every
// LOGICAL tree (dummy padding nodes never exist there), the left-to-right
// (logical) leaf ordinal per tree, and the score (f64, tree order).  This is
// an analysis path, not the hot path: one thread per instance walks the
// packed logical trees through L1 (left iff x < theta, the reference rule)
// and ORs feature bits into its own row of the output bitset.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ts_internal.h"

namespace ts {
namespace {

__global__ void k_trace(const float *__restrict__ x, long long n, long long ld,
                        const TraceNode *__restrict__ nodes, const uint32_t *__restrict__ tree_base,
                        const double *__restrict__ weight, int T, int unit_w, double *out,
                        uint16_t *leaf_ord, long long ld_ord, uint32_t *visited, int words) {
    for (long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x; row < n;
         row += (long long)gridDim.x * blockDim.x) {
        const float *xr = x + row * ld;
        uint32_t *bits = visited ? visited + row * words : nullptr;
        if (bits)
            for (int w = 0; w < words; w++) bits[w] = 0u;
        double acc = 0.0;
        for (int t = 0; t < T; t++) {
            const TraceNode *nd = nodes + __ldg(tree_base + t);
            TraceNode q = nd[0];
            while (q.fid >= 0) {
                if (bits) bits[q.fid >> 5] |= 1u << (q.fid & 31);
                q = nd[__ldg(xr + q.fid) < q.value ? q.left : q.right];
            }
            acc = unit_w ? __dadd_rn(acc, (double)q.value)
                         : __dadd_rn(acc, __dmul_rn(__ldg(weight + t), (double)q.value));
            if (leaf_ord) leaf_ord[(long long)t * ld_ord + row] = (uint16_t)q.left;
        }
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
    const long long blocks = (n + 255) / 256;
    k_trace<<<(int)(blocks < 8LL * sms ? blocks : 8LL * sms), 256, 0, (cudaStream_t)stream>>>(
        x, n, ld, m->dev.trace_nodes, m->dev.trace_base, m->dev.weight, m->num_trees,
        m->unit_weights ? 1 : 0, out, leaf_ord, ld_ord, visited, words);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (prev >= 0 && prev != m->device) cudaSetDevice(prev);
    return e == cudaSuccess ? TS_OK : cuda_fail(e, "trace kernel launch");
}
