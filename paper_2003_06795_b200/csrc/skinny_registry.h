// Entry points of the small-M ("skinny", m <= 16) path, skinny_gemm.cu.
#pragma once
#include "kp_internal.cuh"

namespace kp {
namespace skinny {
constexpr int64_t MAX_M = 16;
// Launch the small-M kernels for any family (fp32 inputs for F32 / TF32,
// bf16 for BF16); KP_ERR_UNSUPPORTED when m > MAX_M.
kp_status launch(kp_family fam, const GemmProblem& g, cudaStream_t s);
// Whether kp_gemm_auto routes this problem to the skinny path (kp_set_skinny).
bool eligible(kp_family fam, const GemmProblem& g);
// 0 = never, 1 = auto (default), 2 = every m <= 16 problem; returns the
// previous mode or -1 for an unknown mode.
int32_t set_mode(int32_t mode);
}  // namespace skinny
}  // namespace kp
