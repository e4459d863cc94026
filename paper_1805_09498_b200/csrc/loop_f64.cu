// Instantiations of the FastFCA-AS loop kernel for double arithmetic.
#include "ffca_loop.cuh"

namespace ffca {

using LoopFn = void (*)(const LoopArgs);

template <int I, int JT>
static LoopFn pick(bool res) {
  return res ? (LoopFn)ffca_loop_kernel<double, I, JT, true> : (LoopFn)ffca_loop_kernel<double, I, JT, false>;
}

// Exact-J instantiations for the BASELINE shapes, runtime-J (<= 8) otherwise.
LoopFn loop_kernel_f64(int I, int J, bool res) {
  if (I == 3 && J == 3) return pick<3, 3>(res);
  if (I == 4 && J == 4) return pick<4, 4>(res);
  if (I == 8 && J == 6) return pick<8, 6>(res);
  if (I == 2 && J == 2) return pick<2, 2>(res);
  if (J > 8) return nullptr;
  switch (I) {
    case 1: return (LoopFn)ffca_loop_kernel<double, 1, 0, false>;
    case 2: return (LoopFn)ffca_loop_kernel<double, 2, 0, false>;
    case 3: return (LoopFn)ffca_loop_kernel<double, 3, 0, false>;
    case 4: return (LoopFn)ffca_loop_kernel<double, 4, 0, false>;
    case 5: return (LoopFn)ffca_loop_kernel<double, 5, 0, false>;
    case 6: return (LoopFn)ffca_loop_kernel<double, 6, 0, false>;
    case 7: return (LoopFn)ffca_loop_kernel<double, 7, 0, false>;
    case 8: return (LoopFn)ffca_loop_kernel<double, 8, 0, false>;
  }
  return nullptr;
}

}  // namespace ffca
