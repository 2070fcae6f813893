// Launcher table of the K1 family: one translation unit per (acc, row_tile)
// pair (simt_inst.cu compiled with -DKP_ACC/-DKP_RT) exports a function that
// instantiates the 4 col_tile values x 4 operand layouts.
#pragma once
#include "kp_internal.cuh"

namespace kp {
namespace simt {

// layout = trans_a * 2 + trans_b
using LaunchFn = kp_status (*)(int col_tile, int layout, const GemmProblem& g, int wg_rows,
                               int wg_cols, cudaStream_t stream);

#define KP_SIMT_FN(a, r) simt_launch_a##a##_r##r
#define KP_SIMT_DECL(a, r)                                                                \
    kp_status KP_SIMT_FN(a, r)(int col_tile, int layout, const GemmProblem& g, int wg_rows, \
                               int wg_cols, cudaStream_t stream);
KP_SIMT_DECL(1, 1) KP_SIMT_DECL(1, 2) KP_SIMT_DECL(1, 4) KP_SIMT_DECL(1, 8)
KP_SIMT_DECL(2, 1) KP_SIMT_DECL(2, 2) KP_SIMT_DECL(2, 4) KP_SIMT_DECL(2, 8)
KP_SIMT_DECL(4, 1) KP_SIMT_DECL(4, 2) KP_SIMT_DECL(4, 4) KP_SIMT_DECL(4, 8)
KP_SIMT_DECL(8, 1) KP_SIMT_DECL(8, 2) KP_SIMT_DECL(8, 4) KP_SIMT_DECL(8, 8)

}  // namespace simt
}  // namespace kp
