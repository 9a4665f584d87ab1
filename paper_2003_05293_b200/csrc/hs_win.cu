// Instantiates the compressed-window kernel for NL = 1..8 (np = 16 NL <= 128 spots)
// at 2, 3 or 4 resident CTAs per SM (register caps 128 / 85 / 64).
#include "hs_win.cuh"

namespace hs {

template <int MINB>
static WinFn pick(int nl)
{
    switch (nl) {
    case 1: return hs_win_kernel<1, MINB>;
    case 2: return hs_win_kernel<2, MINB>;
    case 3: return hs_win_kernel<3, MINB>;
    case 4: return hs_win_kernel<4, MINB>;
    case 5: return hs_win_kernel<5, MINB>;
    case 6: return hs_win_kernel<6, MINB>;
    case 7: return hs_win_kernel<7, MINB>;
    case 8: return hs_win_kernel<8, MINB>;
    default: return nullptr;
    }
}

WinFn hs_select_win(int nl, int minb)
{
    if (minb >= 4) return pick<4>(nl);
    if (minb == 3) return pick<3>(nl);
    return pick<2>(nl);
}

}  // namespace hs
