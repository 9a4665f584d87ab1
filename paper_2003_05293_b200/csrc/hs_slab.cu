// Instantiates the slab-staged compressed-window kernel for NS = 1..8
// (np = 16 NS <= 128 spots), whole-chunk and half-chunk CTAs.
#include "hs_slab.cuh"

namespace hs {

template <bool HALF>
static SlabFn pick(int ns)
{
    switch (ns) {
    case 1: return hs_slab_kernel<1, kSlabG, HALF>;
    case 2: return hs_slab_kernel<2, kSlabG, HALF>;
    case 3: return hs_slab_kernel<3, kSlabG, HALF>;
    case 4: return hs_slab_kernel<4, kSlabG, HALF>;
    case 5: return hs_slab_kernel<5, kSlabG, HALF>;
    case 6: return hs_slab_kernel<6, kSlabG, HALF>;
    case 7: return hs_slab_kernel<7, kSlabG, HALF>;
    case 8: return hs_slab_kernel<8, kSlabG, HALF>;
    default: return nullptr;
    }
}

SlabFn hs_select_slab(int ns, bool half) { return half ? pick<true>(ns) : pick<false>(ns); }

}  // namespace hs
