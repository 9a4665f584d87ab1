// Instantiates the slab-staged compressed-window kernel for NS = 1..8
// (np = 16 NS <= 128 spots).
#include "hs_slab.cuh"

namespace hs {

SlabFn hs_select_slab(int ns)
{
    switch (ns) {
    case 1: return hs_slab_kernel<1, kSlabG>;
    case 2: return hs_slab_kernel<2, kSlabG>;
    case 3: return hs_slab_kernel<3, kSlabG>;
    case 4: return hs_slab_kernel<4, kSlabG>;
    case 5: return hs_slab_kernel<5, kSlabG>;
    case 6: return hs_slab_kernel<6, kSlabG>;
    case 7: return hs_slab_kernel<7, kSlabG>;
    case 8: return hs_slab_kernel<8, kSlabG>;
    default: return nullptr;
    }
}

}  // namespace hs
