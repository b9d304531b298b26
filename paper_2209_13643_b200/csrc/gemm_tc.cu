// tcgen05 int8-limb ring GEMM (sm_100a). Placeholder until the tensor-core path lands.
#include "gemm.cuh"

namespace mpcg {
bool ring_gemm_tc_try(Session&, const GemmArgs&) { return false; }
}  // namespace mpcg
