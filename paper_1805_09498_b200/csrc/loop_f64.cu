// Instantiations of the FastFCA-AS loop kernel for double arithmetic.
#include "ffca_loop.cuh"

namespace ffca {

using LoopFn = void (*)(const LoopArgs);

// Hot (BASELINE) shapes: exact J; G = 2 lane-interleaved bins (one 32-byte
// sector of double complex) when a bin fits one CTA, G = 1 for clusters / the
// global-slab path.
template <int I, int J>
static LoopFn hot(int G, bool res, bool fast) {
  if constexpr (I == 3 && J == 3) {  // config 0 (one-bin CTAs) and the batched complex128 line
    if (fast && res && G == 2) return ffca_loop_kernel<double, I, J, 2, true, true>;
    if (fast && res && G == 1) return ffca_loop_kernel<double, I, J, 1, true, true>;
  }
  if constexpr (I <= 4) {
    if (G == 2 && res) return ffca_loop_kernel<double, I, J, 2, true>;
  }
  if (G == 1) return res ? (LoopFn)ffca_loop_kernel<double, I, J, 1, true> : (LoopFn)ffca_loop_kernel<double, I, J, 1, false>;
  return nullptr;
}

LoopFn loop_kernel_f64(int I, int J, int G, bool res, bool fast) {
  if (I == 3 && J == 3) return hot<3, 3>(G, res, fast);
  if (I == 4 && J == 4) return hot<4, 4>(G, res, false);
  if (I == 8 && J == 6) return hot<8, 6>(G, res, false);
  if (I == 2 && J == 2) return hot<2, 2>(G, res, false);
  if (J > 8 || G != 1) return nullptr;
  // runtime J (<= 8); residency decided at run time (scratch == nullptr)
  switch (I) {
    case 1: return ffca_loop_kernel<double, 1, 0, 1, false>;
    case 2: return ffca_loop_kernel<double, 2, 0, 1, false>;
    case 3: return ffca_loop_kernel<double, 3, 0, 1, false>;
    case 4: return ffca_loop_kernel<double, 4, 0, 1, false>;
    case 5: return ffca_loop_kernel<double, 5, 0, 1, false>;
    case 6: return ffca_loop_kernel<double, 6, 0, 1, false>;
    case 7: return ffca_loop_kernel<double, 7, 0, 1, false>;
    case 8: return ffca_loop_kernel<double, 8, 0, 1, false>;
  }
  return nullptr;
}

}  // namespace ffca
