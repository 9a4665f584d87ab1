// Instantiates the slab-staged compressed-window kernel for NS = 1..8
// (np = 16 NS <= 128 spots), whole-chunk and half-chunk CTAs.
#include <stdlib.h>

#include "hs_slab.cuh"

namespace hs {

template <bool HALF, bool PIPE>
static SlabFn pick(int ns)
{
    switch (ns) {
    case 1: return hs_slab_kernel<1, kSlabG, HALF, PIPE>;
    case 2: return hs_slab_kernel<2, kSlabG, HALF, PIPE>;
    case 3: return hs_slab_kernel<3, kSlabG, HALF, PIPE>;
    case 4: return hs_slab_kernel<4, kSlabG, HALF, PIPE>;
    case 5: return hs_slab_kernel<5, kSlabG, HALF, PIPE>;
    case 6: return hs_slab_kernel<6, kSlabG, HALF, PIPE>;
    case 7: return hs_slab_kernel<7, kSlabG, HALF, PIPE>;
    case 8: return hs_slab_kernel<8, kSlabG, HALF, PIPE>;
    default: return nullptr;
    }
}

SlabFn hs_select_slab(int ns, bool half, bool pipe)
{
    if (pipe) return half ? pick<true, true>(ns) : pick<false, true>(ns);
    return half ? pick<true, false>(ns) : pick<false, false>(ns);
}

// HS_SLAB_PIPE=0|1 selects the main loop (A/B experiments)
SlabFn hs_select_slab(int ns, bool half)
{
    static const bool pipe = getenv("HS_SLAB_PIPE") ? atoi(getenv("HS_SLAB_PIPE")) != 0 : false;
    return hs_select_slab(ns, half, pipe);
}

}  // namespace hs
