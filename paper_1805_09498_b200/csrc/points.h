// Per-point streaming kernels (points.cu): modes and arguments, shared with the loop's C ABI
// (abi_fastfca.cu launches the statistics refresh right after the loop kernel).
#pragma once

#include <cuda_runtime.h>

namespace ffca {

enum PointMode : int {
  PM_STATS = 0,      // y, P, lam, v -> mu_t, phi_t       (fastfca.py:373-387)
  PM_ESTEP_YT = 1,   // y_t, lam, v  -> mu_t, phi_t       (fastfca.py:144-157)
  PM_TRANSFORM = 2,  // y, P         -> y_t (N,F,I)       (fastfca.py:113-116)
  PM_WEIGHTS = 3,    // lam, v       -> w (N,F,I)         (fastfca.py:138-141)
  PM_IMAGES = 4,     // y, P, Q=P^-H, lam, v -> images    (wiener.py:38-43 on the final state)
  PM_BACK = 5,       // mu_t, Q      -> Q mu_t            (fastfca.py:258-273)
};

struct PointArgs {
  int mode, U, I, J, N, F;
  const void* y;     // (U,I,N,F) complex, or y_t (U,N,F,I) for PM_ESTEP_YT, or mu_t (U,J,N,F,I) for PM_BACK
  const void* P;     // (U,F,I,I) complex
  const void* Q;     // (U,F,I,I) complex fp64: P^-H
  const void* lam;   // (U,J,F,I) real
  const void* v;     // (U,J,N,F) real
  void* out0;        // mu_t / y_t / w / images / back
  void* out1;        // phi_t
  int images_layout; // PM_BACK: write (U,J,I,N,F)
};

// Launches the per-point kernel for a.mode (the bin-tiled kernel for statistics / images at
// I, J <= 4).  Stream-ordered on s.
int launch_points(int dtype, const PointArgs& a, cudaStream_t s);
int launch_inv_PH(int dtype, int I, const void* P, double2* Q, int* status, long long nbins, cudaStream_t s);

}  // namespace ffca
