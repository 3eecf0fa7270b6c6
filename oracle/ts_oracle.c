/*
 * ts_oracle.c -- CPU restatement of the reference's predicated scoring path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker (and the CPU baseline
 * timed by bench.py's cpu_baseline leg / --impl reference).  Nothing in the
 * product package links, loads or calls it.
 *
 * It restates, in plain C, the arithmetic of the reference package
 * `treescore` (pure Python + numpy, /root/reference/pkg/src/treescore):
 *
 *   orc_expand        <- expand_to_complete          model.py:315-349
 *                        dummy nodes fid=0, theta=+inf model.py:45-50
 *   orc_score         <- VPredicatedEvaluator._predict_into
 *                        evaluators.py:520-546, lockstep batch kernel
 *                        evaluators.py:90-99: i = (i<<1)+1+(x[fid[i]] >= theta[i]),
 *                        d times, ordinal = i - (2^d - 1); score
 *                        acc += weight * (double)leaf[ordinal] in tree order
 *                        (evaluators.py:529-535, f64, acc starts at +0.0)
 *   orc_score_linked  <- reference_predict / traverse_to_leaf
 *                        model.py:251-271: left iff x[fid] < threshold
 *
 * Input trees come in the flat form the product's C-ABI also takes: per tree
 * a block of nodes with tree-local ids, node 0 the root, fid == -1 for a leaf,
 * value = threshold (internal) or leaf value (leaf), already fp32.
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off, no -ffast-math: the
 * f64 sum must be IEEE round-to-nearest multiply-then-add, never an FMA).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAX_DEPTH 16

/* ---------------------------------------------------------------- expand */

static int tree_depth(const int32_t *fid, const int32_t *left,
                      const int32_t *right, int32_t node) {
    if (fid[node] < 0) return 0;
    int a = tree_depth(fid, left, right, left[node]);
    int b = tree_depth(fid, left, right, right[node]);
    return 1 + (a > b ? a : b);
}

static void fill(const int32_t *fid, const float *val, const int32_t *left,
                 const int32_t *right, int32_t node, int64_t slot,
                 int64_t n_internal, int32_t *ofid, float *otheta, float *oleaf) {
    if (slot >= n_internal) {            /* bottom level: a leaf slot */
        oleaf[slot - n_internal] = val[node];
        return;
    }
    if (fid[node] < 0) {                 /* early leaf: dummy subtree */
        ofid[slot] = 0;
        otheta[slot] = INFINITY;
        fill(fid, val, left, right, node, 2 * slot + 1, n_internal, ofid, otheta, oleaf);
        fill(fid, val, left, right, node, 2 * slot + 2, n_internal, ofid, otheta, oleaf);
    } else {
        ofid[slot] = fid[node];
        otheta[slot] = val[node];
        fill(fid, val, left, right, left[node], 2 * slot + 1, n_internal, ofid, otheta, oleaf);
        fill(fid, val, left, right, right[node], 2 * slot + 2, n_internal, ofid, otheta, oleaf);
    }
}

/* Depth of every tree; returns -1 if any exceeds ORC_MAX_DEPTH. */
int orc_depths(int32_t num_trees, const int64_t *tree_off, const int32_t *fid,
               const int32_t *left, const int32_t *right, int32_t *depth_out) {
    for (int32_t t = 0; t < num_trees; t++) {
        int64_t o = tree_off[t];
        int d = tree_depth(fid + o, left + o, right + o, 0);
        depth_out[t] = d;
        if (d > ORC_MAX_DEPTH) return -1;
    }
    return 0;
}

/* Complete tables.  int_off / leaf_off (size T+1) are computed by the caller
 * from the depths: internal block 2^d - 1 entries, leaf block 2^d entries. */
void orc_expand(int32_t num_trees, const int64_t *tree_off, const int32_t *fid,
                const float *val, const int32_t *left, const int32_t *right,
                const int32_t *depth, const int64_t *int_off, const int64_t *leaf_off,
                int32_t *cfid, float *ctheta, float *cleaf) {
    for (int32_t t = 0; t < num_trees; t++) {
        int64_t o = tree_off[t];
        int64_t n_internal = ((int64_t)1 << depth[t]) - 1;
        fill(fid + o, val + o, left + o, right + o, 0, 0, n_internal,
             cfid + int_off[t], ctheta + int_off[t], cleaf + leaf_off[t]);
    }
}

/* ----------------------------------------------------------------- score */

typedef struct {
    int32_t num_trees;
    const int32_t *depth;
    const int64_t *int_off, *leaf_off;
    const int32_t *cfid;
    const float *ctheta, *cleaf;
    const double *weight;
    const float *x;
    int64_t f, ld;
    double *out;
    uint16_t *ord;      /* nullable, layout [tree][row] with stride ld_ord */
    int64_t ld_ord;
    int64_t row_begin, row_end;
    int64_t v;          /* lockstep micro-batch (the reference's batch_size) */
} job_t;

static void *score_rows(void *arg) {
    job_t *j = (job_t *)arg;
    int64_t v = j->v > 0 ? j->v : 64;
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * v);
    double *acc = (double *)malloc(sizeof(double) * v);
    for (int64_t s = j->row_begin; s < j->row_end; s += v) {
        int64_t m = j->row_end - s < v ? j->row_end - s : v;
        for (int64_t r = 0; r < m; r++) acc[r] = 0.0;
        for (int32_t t = 0; t < j->num_trees; t++) {
            const int32_t *fd = j->cfid + j->int_off[t];
            const float *th = j->ctheta + j->int_off[t];
            const float *lf = j->cleaf + j->leaf_off[t];
            int d = j->depth[t];
            for (int64_t r = 0; r < m; r++) cur[r] = 0;
            for (int l = 0; l < d; l++) {           /* one level for the whole batch */
                for (int64_t r = 0; r < m; r++) {
                    const float *xr = j->x + (s + r) * j->ld;
                    int64_t i = cur[r];
                    cur[r] = (i << 1) + 1 + (xr[fd[i]] >= th[i]);
                }
            }
            int64_t base = ((int64_t)1 << d) - 1;
            double w = j->weight[t];
            for (int64_t r = 0; r < m; r++) {
                int64_t o = cur[r] - base;
                acc[r] = acc[r] + w * (double)lf[o];   /* built with -ffp-contract=off */
                if (j->ord) j->ord[(int64_t)t * j->ld_ord + s + r] = (uint16_t)o;
            }
        }
        for (int64_t r = 0; r < m; r++) j->out[s + r] = acc[r];
    }
    free(cur);
    free(acc);
    return NULL;
}

void orc_score(int32_t num_trees, const int32_t *depth, const int64_t *int_off,
               const int64_t *leaf_off, const int32_t *cfid, const float *ctheta,
               const float *cleaf, const double *weight, const float *x, int64_t n,
               int64_t f, int64_t ld, double *out, uint16_t *ord, int64_t ld_ord,
               int64_t v, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (n <= 0) return;
    if (nthreads > n) nthreads = (int)n;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    job_t *jobs = (job_t *)malloc(sizeof(job_t) * nthreads);
    for (int k = 0; k < nthreads; k++) {
        job_t j = {num_trees, depth, int_off, leaf_off, cfid, ctheta, cleaf, weight,
                   x, f, ld, out, ord, ld_ord, n * k / nthreads, n * (k + 1) / nthreads, v};
        jobs[k] = j;
        if (nthreads == 1) score_rows(&jobs[k]);
        else pthread_create(&th[k], NULL, score_rows, &jobs[k]);
    }
    if (nthreads > 1)
        for (int k = 0; k < nthreads; k++) pthread_join(th[k], NULL);
    free(th);
    free(jobs);
}

/* Linked traversal on the flat (unexpanded) trees: the reference oracle
 * semantics, strict `<` goes left. */
void orc_score_linked(int32_t num_trees, const int64_t *tree_off, const int32_t *fid,
                      const float *val, const int32_t *left, const int32_t *right,
                      const double *weight, const float *x, int64_t n, int64_t ld,
                      double *out) {
    for (int64_t r = 0; r < n; r++) {
        const float *xr = x + r * ld;
        double acc = 0.0;
        for (int32_t t = 0; t < num_trees; t++) {
            int64_t o = tree_off[t];
            int32_t i = 0;
            while (fid[o + i] >= 0)
                i = (xr[fid[o + i]] < val[o + i]) ? left[o + i] : right[o + i];
            acc = acc + weight[t] * (double)val[o + i];
        }
        out[r] = acc;
    }
}
