// Instantiates hs_pass_kernel for G = 8 lanes per pixel (see hs_kernels.cuh).
#include "hs_kernels.cuh"

namespace hs {
HS_DEFINE_SELECT(8)
}  // namespace hs
