// Entry points of the tcgen05 families (K2 TF32, K3 BF16), tc_gemm.cu.
#pragma once
#include "kp_internal.cuh"

namespace kp {
namespace tc {
int32_t num_configs(kp_family fam);
kp_status config_at(kp_family fam, int32_t index, kp_config* out);
kp_status valid(kp_family fam, const kp_config& c);
kp_status launch(kp_family fam, const kp_config& c, const GemmProblem& g, cudaStream_t s);
// split-K policy of the 1-CTA kernels (kp_set_tc_split); returns the previous mode or -1
int32_t set_split_mode(int32_t mode);
}  // namespace tc
}  // namespace kp
