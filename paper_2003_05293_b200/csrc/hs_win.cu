// Instantiates the compressed-window kernel for NL = 1..8 (np = 16 NL <= 128 spots).
#include "hs_win.cuh"

namespace hs {

WinFn hs_select_win(int nl)
{
    switch (nl) {
    case 1: return hs_win_kernel<1>;
    case 2: return hs_win_kernel<2>;
    case 3: return hs_win_kernel<3>;
    case 4: return hs_win_kernel<4>;
    case 5: return hs_win_kernel<5>;
    case 6: return hs_win_kernel<6>;
    case 7: return hs_win_kernel<7>;
    case 8: return hs_win_kernel<8>;
    default: return nullptr;
    }
}

}  // namespace hs
