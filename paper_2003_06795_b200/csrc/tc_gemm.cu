// K2/K3 tcgen05 families -- placeholder until the tensor-core path lands.
#include "tc_registry.h"

namespace kp {
namespace tc {
int32_t num_configs(kp_family) { return 0; }
kp_status config_at(kp_family, int32_t, kp_config*) {
    return fail(KP_ERR_UNSUPPORTED, "tcgen05 families not built");
}
kp_status valid(kp_family, const kp_config&) {
    return fail(KP_ERR_UNSUPPORTED, "tcgen05 families not built");
}
kp_status launch(kp_family, const kp_config&, const GemmProblem&, cudaStream_t) {
    return fail(KP_ERR_UNSUPPORTED, "tcgen05 families not built");
}
}  // namespace tc
}  // namespace kp
