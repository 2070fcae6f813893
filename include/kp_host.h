/*
 * kp_host.h -- host-side (no CUDA) native helpers of the framework
 * (libkp_host.so).
 *
 * kp_csv_load_matrix: SURVEY §8(f) item 4, faster ingestion of the sweep
 * interchange CSV.  Replaces, for well-formed input, the composition
 *   dataset.build_matrix(dataset.load_records(path))
 * of the reference (pkg/src/kernelprune/dataset.py: load_records :188-222,
 * build_matrix :239-270) with one pass of native parsing straight into the
 * dense gflops grid.  Same result by construction: problems in order of first
 * appearance, configs present in canonical (acc, row_tile, col_tile, wg_rows,
 * wg_cols) order, reals parsed with the correctly rounded strtod (== Python
 * float()).  The accepted grammar is a strict subset of what the reference
 * accepts (no quoting, no surrounding blanks, no '_' digit separators, no
 * inf/nan); anything outside it -- and every invalid input -- returns
 * KP_CSV_DEFER with the offending line, and the caller re-runs the exact
 * reference validator, which either accepts the input or raises its
 * line-numbered DataError.  So error behaviour is the reference's, always.
 */
#ifndef KP_HOST_H
#define KP_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t n_problems, n_configs;
    int64_t* problems;  /* n_problems x 3 (m, k, n), first-appearance order */
    uint32_t* configs;  /* n_configs x 5, canonical order                   */
    double* gflops;     /* n_problems x n_configs, row-major                */
} kp_csv_matrix;

enum { KP_CSV_OK = 0, KP_CSV_DEFER = 1, KP_CSV_IO = 2 };

/* Parse `path` into *out (owned by the caller: release with kp_csv_free).
 * On KP_CSV_DEFER, *bad_line is the 1-based line that left the fast grammar
 * (0 for whole-file conditions: empty, duplicates, holes). */
int32_t kp_csv_load_matrix(const char* path, kp_csv_matrix* out, int64_t* bad_line);
void kp_csv_free(kp_csv_matrix* m);

#ifdef __cplusplus
}
#endif
#endif /* KP_HOST_H */
