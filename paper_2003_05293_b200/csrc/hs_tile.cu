// Instantiates the full-range GEMM-tile kernel for SPT = 1..16 spots per
// forward thread (KP = 8 SPT >= n, n <= 128).
#include "hs_tile.cuh"

namespace hs {

template <int SPT>
static TileFn pick(bool write)
{
    return write ? hs_tile_kernel<SPT, true> : hs_tile_kernel<SPT, false>;
}

TileFn hs_select_tile(int spt, bool write)
{
    switch (spt) {
    case 1: return pick<1>(write);
    case 2: return pick<2>(write);
    case 3: return pick<3>(write);
    case 4: return pick<4>(write);
    case 5: return pick<5>(write);
    case 6: return pick<6>(write);
    case 7: return pick<7>(write);
    case 8: return pick<8>(write);
    case 9: return pick<9>(write);
    case 10: return pick<10>(write);
    case 11: return pick<11>(write);
    case 12: return pick<12>(write);
    case 13: return pick<13>(write);
    case 14: return pick<14>(write);
    case 15: return pick<15>(write);
    case 16: return pick<16>(write);
    default: return nullptr;
    }
}

}  // namespace hs
