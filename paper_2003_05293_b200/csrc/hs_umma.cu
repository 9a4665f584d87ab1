// Instantiates the tcgen05 full-range pass for np = 16 .. 112 (one forward
// spot chunk) and for larger np (forward spot chunks of 128).
#include "hs_umma.cuh"

namespace hs {

template <int NP>
static UmmaFn pick(int write)
{
    return write == 2 ? hs_umma_kernel<NP, 2> : write == 1 ? hs_umma_kernel<NP, 1> : hs_umma_kernel<NP, 0>;
}

UmmaFn hs_select_umma(int np, int write)
{
    switch (np) {
    case 16: return pick<16>(write);
    case 32: return pick<32>(write);
    case 48: return pick<48>(write);
    case 64: return pick<64>(write);
    case 80: return pick<80>(write);
    case 96: return pick<96>(write);
    case 112: return pick<112>(write);
    default: return np > kUNPMax ? pick<kUNPC>(write) : nullptr;  // spot-chunked forward
    }
}

}  // namespace hs
