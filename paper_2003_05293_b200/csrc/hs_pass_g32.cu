// Instantiates hs_pass_kernel for G = 32 lanes per pixel (see hs_kernels.cuh);
// NL = 32 serves 513..1024 spots (one CTA per SM, 255 registers).
#include "hs_kernels.cuh"

namespace hs {
PassFn hs_select_g32(int nl, int mode)
{
    switch (nl) {
    case 4: return hs_pass_fn<32, 4>(mode);
    case 8: return hs_pass_fn<32, 8>(mode);
    case 10: return hs_pass_fn<32, 10>(mode);
    case 12: return hs_pass_fn<32, 12>(mode);
    case 14: return hs_pass_fn<32, 14>(mode);
    case 16: return hs_pass_fn<32, 16>(mode);
    case 32: return hs_pass_fn<32, 32>(mode);
    default: return nullptr;
    }
}
}  // namespace hs
