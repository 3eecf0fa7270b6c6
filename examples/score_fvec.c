/* score_fvec.c -- the C ABI end to end, no Python: parse a model file in the
 * reference's text format (ts_parse_model), pack it for GPU 0 (ts_pack),
 * read an FVEC instance file ("FVEC", u32 n, u32 f, n*f little-endian fp32;
 * ref data.py:72-96) and score it from host buffers (ts_score_host).
 * Prints one f64 score per line with 17 significant digits.
 *
 *   cc -O2 -Iinclude examples/score_fvec.c -Lpaper_1212_2287_b200 \
 *      -l:_ts_gpu.so -Wl,-rpath,$PWD/paper_1212_2287_b200 -o score_fvec
 *   ./score_fvec model.txt x.fvec > scores.txt
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "treescore_gpu.h"

static char *slurp(const char *path, long *len) {
    FILE *f = fopen(path, "rb");
    if (!f) return NULL;
    fseek(f, 0, SEEK_END);
    *len = ftell(f);
    fseek(f, 0, SEEK_SET);
    char *buf = malloc(*len + 1);
    if (buf && fread(buf, 1, *len, f) != (size_t)*len) {
        free(buf);
        buf = NULL;
    }
    fclose(f);
    return buf;
}

int main(int argc, char **argv) {
    if (argc != 3) {
        fprintf(stderr, "usage: %s model.txt x.fvec\n", argv[0]);
        return 2;
    }
    long mlen = 0, xlen = 0;
    char *text = slurp(argv[1], &mlen);
    char *fvec = slurp(argv[2], &xlen);
    if (!text || !fvec || xlen < 12 || memcmp(fvec, "FVEC", 4) != 0) {
        fprintf(stderr, "cannot read inputs\n");
        return 1;
    }
    uint32_t n, f;
    memcpy(&n, fvec + 4, 4);
    memcpy(&f, fvec + 8, 4);
    if ((long)(12 + (int64_t)n * f * 4) != xlen) {
        fprintf(stderr, "FVEC payload size mismatch\n");
        return 1;
    }
    ts_flat_model *flat = NULL;
    if (ts_parse_model(text, mlen, &flat) != TS_OK) {
        fprintf(stderr, "parse error at %d:%d: %s\n", flat ? flat->err_line : 0,
                flat ? flat->err_col : 0, ts_last_error());
        ts_flat_free(flat);
        return 1;
    }
    ts_model_desc desc = {flat->num_features, flat->num_trees, flat->tree_node_offset,
                          flat->tree_weight, flat->node_fid, flat->node_value,
                          flat->node_left, flat->node_right};
    ts_model *model = NULL;
    if (ts_pack(&desc, 0, &model) != TS_OK) {
        fprintf(stderr, "pack: %s\n", ts_last_error());
        return 1;
    }
    ts_flat_free(flat);  /* the packed model owns device copies */
    float *x = malloc((size_t)n * f * sizeof(float));
    double *out = malloc((size_t)n * sizeof(double));
    memcpy(x, fvec + 12, (size_t)n * f * sizeof(float));
    int rc = ts_score_host(model, x, n, f, out);
    if (rc != TS_OK) {
        fprintf(stderr, "score: %s\n", ts_last_error());
        return 1;
    }
    for (uint32_t i = 0; i < n; i++) printf("%.17g\n", out[i]);
    ts_free(model);
    free(x);
    free(out);
    free(text);
    free(fvec);
    return 0;
}
