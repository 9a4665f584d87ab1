// Instantiates hs_pass_kernel for G = 1 lanes per pixel (see hs_kernels.cuh).
#include "hs_kernels.cuh"

namespace hs {
HS_DEFINE_SELECT(1)
}  // namespace hs
