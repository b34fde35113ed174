// Placeholder until the tcgen05 kernels land: the tensor-core path is not yet
// eligible, so contexts created with a tensor-core precision fail loudly.
#include <stdexcept>

#include "tc_gemm.cuh"

namespace dasmc_b200 {

bool tc_layer1_eligible(const Ctx&) { return false; }
void tc_forward_layer1(Ctx&, const float*, int64_t, int64_t) { throw std::runtime_error("tcgen05 path not built"); }
void tc_delta_layer1(Ctx&, const float*, int64_t, int64_t) { throw std::runtime_error("tcgen05 path not built"); }
void tc_dw_layer1(Ctx&, int64_t, int64_t, const EpiParams&) { throw std::runtime_error("tcgen05 path not built"); }

}  // namespace dasmc_b200
