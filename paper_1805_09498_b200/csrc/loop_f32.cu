// Instantiations of the FastFCA-AS loop kernel for float arithmetic.
#include "ffca_loop.cuh"

namespace ffca {

using LoopFn = void (*)(const LoopArgs);

// Hot (BASELINE) shapes: exact J; G = 4 lane-interleaved bins (one 32-byte
// sector of float complex) when a bin fits one CTA, G = 1 for clusters / the
// global-slab path.
template <int I, int J>
static LoopFn hot(int G, bool res, bool fast, bool tm) {
  if constexpr (I == 3 && J == 3)
    if (tm)
      return !(G == 4 && res) ? nullptr
             : fast           ? (LoopFn)ffca_loop_kernel<float, 3, 3, 4, true, true, true>
                              : (LoopFn)ffca_loop_kernel<float, 3, 3, 4, true, false, true>;
  if constexpr (I == 4 && J == 4)
    if (tm) return (G == 1 && res && fast) ? (LoopFn)ffca_loop_kernel<float, 4, 4, 1, true, true, true> : nullptr;
  if constexpr (I <= 4) {
    if constexpr (I == 3 && J == 3)
      if (G == 4 && res && fast) return ffca_loop_kernel<float, I, J, 4, true, true>;
    if (G == 4 && res) return ffca_loop_kernel<float, I, J, 4, true>;
    if constexpr (I == 3 && J == 3)
      if (G == 2 && res)
        return fast ? (LoopFn)ffca_loop_kernel<float, I, J, 2, true, true> : (LoopFn)ffca_loop_kernel<float, I, J, 2, true>;
  }
  if constexpr ((I == 4 && J == 4) || (I == 8 && J == 6) || (I == 3 && J == 3))  // the config-2 / config-4 cluster plans, one-bin config 3
    if (G == 1 && res && fast) return ffca_loop_kernel<float, I, J, 1, true, true>;
  if (G == 1) return res ? (LoopFn)ffca_loop_kernel<float, I, J, 1, true> : (LoopFn)ffca_loop_kernel<float, I, J, 1, false>;
  return nullptr;
}

LoopFn loop_kernel_f32(int I, int J, int G, bool res, bool fast, bool tm) {
  if (tm && !((I == 3 && J == 3) || (I == 4 && J == 4))) return nullptr;
  if (I == 3 && J == 3) return hot<3, 3>(G, res, fast, tm);
  if (I == 4 && J == 4) return hot<4, 4>(G, res, fast, tm);
  if (I == 8 && J == 6) return hot<8, 6>(G, res, fast, false);
  if (I == 2 && J == 2) return hot<2, 2>(G, res, false, false);
  if (J > 8 || G != 1) return nullptr;
  // runtime J (<= 8); residency decided at run time (scratch == nullptr) -- except the resident
  // I > 4 plans, which run one CTA per SM and get the 255-register instantiation
  if (res && I > 4) switch (I) {
      case 5: return ffca_loop_kernel<float, 5, 0, 1, true>;
      case 6: return ffca_loop_kernel<float, 6, 0, 1, true>;
      case 7: return ffca_loop_kernel<float, 7, 0, 1, true>;
      case 8: return ffca_loop_kernel<float, 8, 0, 1, true>;
    }
  switch (I) {
    case 1: return ffca_loop_kernel<float, 1, 0, 1, false>;
    case 2: return ffca_loop_kernel<float, 2, 0, 1, false>;
    case 3: return ffca_loop_kernel<float, 3, 0, 1, false>;
    case 4: return ffca_loop_kernel<float, 4, 0, 1, false>;
    case 5: return ffca_loop_kernel<float, 5, 0, 1, false>;
    case 6: return ffca_loop_kernel<float, 6, 0, 1, false>;
    case 7: return ffca_loop_kernel<float, 7, 0, 1, false>;
    case 8: return ffca_loop_kernel<float, 8, 0, 1, false>;
  }
  return nullptr;
}

}  // namespace ffca

#ifdef FFCA_PHASE_PROBE
extern "C" int ffca_debug_fixed(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, ffca::g_fixed, sizeof(unsigned long long) * 4);
  unsigned long long z[4] = {};
  cudaMemcpyToSymbol(ffca::g_fixed, z, sizeof(z));
  return 0;
}
extern "C" int ffca_debug_phase(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, ffca::g_phase, sizeof(unsigned long long) * 16);
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(ffca::g_phase, z, sizeof(z));
  return 0;
}
#endif
