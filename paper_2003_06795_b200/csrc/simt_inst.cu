// Instantiation unit of the K1 family for one (acc, row_tile) pair, selected
// with -DKP_ACC=<1|2|4|8> -DKP_RT=<1|2|4|8> (16 objects built in parallel).
#include "simt_gemm.cuh"
#include "simt_registry.h"

#if !defined(KP_ACC) || !defined(KP_RT)
#error "compile with -DKP_ACC=<acc> -DKP_RT=<row_tile>"
#endif

namespace kp {
namespace simt {

template <int CT>
static kp_status by_layout(int layout, const GemmProblem& g, int wgr, int wgc, cudaStream_t s) {
    switch (layout) {
        case 0: return launch<KP_ACC, KP_RT, CT, false, false>(g, wgr, wgc, s);
        case 1: return launch<KP_ACC, KP_RT, CT, false, true>(g, wgr, wgc, s);
        case 2: return launch<KP_ACC, KP_RT, CT, true, false>(g, wgr, wgc, s);
        case 3: return launch<KP_ACC, KP_RT, CT, true, true>(g, wgr, wgc, s);
    }
    return fail(KP_ERR_INVALID_ARG, "simt: bad operand layout");
}

#define KP_SIMT_DEF(a, r) KP_SIMT_FN(a, r)
kp_status KP_SIMT_DEF(KP_ACC, KP_RT)(int col_tile, int layout, const GemmProblem& g, int wgr,
                                      int wgc, cudaStream_t s) {
    switch (col_tile) {
        case 1: return by_layout<1>(layout, g, wgr, wgc, s);
        case 2: return by_layout<2>(layout, g, wgr, wgc, s);
        case 4: return by_layout<4>(layout, g, wgr, wgc, s);
        case 8: return by_layout<8>(layout, g, wgr, wgc, s);
    }
    return fail(KP_ERR_INVALID_CONFIG, "simt: col_tile not in {1,2,4,8}");
}

}  // namespace simt
}  // namespace kp
