// Instantiates the spot-chunked full-range tile kernel (n > 128).
#include "hs_tilek.cuh"

namespace hs {

TileKFn hs_select_tilek(bool write) { return write ? hs_tilek_kernel<true> : hs_tilek_kernel<false>; }

}  // namespace hs
