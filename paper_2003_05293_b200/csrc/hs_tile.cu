// Instantiates the full-range GEMM-tile kernel for NS = 1..8 (np = 16 NS <= 128 spots).
#include "hs_tile.cuh"

namespace hs {

template <int NS>
static TileFn pick(bool write)
{
    return write ? hs_tile_kernel<NS, true> : hs_tile_kernel<NS, false>;
}

TileFn hs_select_tile(int ns, bool write)
{
    switch (ns) {
    case 1: return pick<1>(write);
    case 2: return pick<2>(write);
    case 3: return pick<3>(write);
    case 4: return pick<4>(write);
    case 5: return pick<5>(write);
    case 6: return pick<6>(write);
    case 7: return pick<7>(write);
    case 8: return pick<8>(write);
    default: return nullptr;
    }
}

}  // namespace hs
