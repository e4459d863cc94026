// Unfused diagonal M-step (fastfca.m_step_diag, fastfca.py:160-181) on device.
//
// One CTA per bin; threads stride over frames.  Per point and source
//   v'  = max(sum_i (|mu_i|^2 + phi_i) / lam_i / I, floor)
// and per bin
//   lam'_i = sum_n (|mu_i|^2 + phi_i) / v' / N, floored at 1e-12 max_i.
// The reduction over n is a fixed-order warp-shuffle + shared-memory tree.
#include "common.cuh"
#include "host_common.h"

namespace ffca {

struct MstepArgs {
  int U, I, J, N, F;
  const void* mu;   // (U,J,N,F,I) complex
  const void* phi;  // (U,J,N,F,I) real
  const void* lam;  // (U,J,F,I) real
  int vf_mode;      // FFCA_VF_SCALAR / BIN / FULL
  double vf_scalar;
  const void* vf;
  void* v_out;      // (U,J,N,F)
  void* lam_out;    // (U,J,F,I)
};

template <typename R, int I>
__global__ void __launch_bounds__(128) mstep_kernel(const MstepArgs a) {
  using C2 = typename Cpx<R>::T;
  constexpr int JM = 8;
  const long long bin = blockIdx.x;
  const int F = a.F, N = a.N, J = a.J;
  const long long u = bin / F;
  const int f = int(bin % F);
  const R* lam = (const R*)a.lam;
  const C2* mu = (const C2*)a.mu;
  const R* phi = (const R*)a.phi;
  R* vo = (R*)a.v_out;
  __shared__ double part[4][JM * I];
  R acc[JM * I];
#pragma unroll
  for (int k = 0; k < JM * I; ++k) acc[k] = R(0);
  R ilam[JM * I];
#pragma unroll
  for (int j = 0; j < JM; ++j)
#pragma unroll
    for (int i = 0; i < I; ++i) ilam[j * I + i] = j < J ? R(1) / lam[((u * J + j) * F + f) * I + i] : R(0);
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
#pragma unroll
    for (int j = 0; j < JM; ++j) {
      if (j >= J) continue;
      const long long base = (((u * J + j) * N + n) * (long long)F + f) * I;
      R m2[I];
      R s = R(0);
#pragma unroll
      for (int i = 0; i < I; ++i) {
        const C2 m = mu[base + i];
        m2[i] = m.x * m.x + m.y * m.y + phi[base + i];
        s += m2[i] * ilam[j * I + i];
      }
      R fl = R(a.vf_scalar);
      if (a.vf_mode == FFCA_VF_BIN) fl = ((const R*)a.vf)[bin];
      if (a.vf_mode == FFCA_VF_FULL) fl = ((const R*)a.vf)[((u * J + j) * N + n) * (long long)F + f];
      const R vn = fmax(s / R(I), fl);
      vo[((u * J + j) * N + n) * (long long)F + f] = vn;
      const R iv = R(1) / vn;
#pragma unroll
      for (int i = 0; i < I; ++i) acc[j * I + i] = fma(iv, m2[i], acc[j * I + i]);
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < JM * I; ++k) {
    R x = warp_sum_seg(acc[k], 1);
    if (lane == 0) part[warp][k] = double(x);
  }
  __syncthreads();
  if (threadIdx.x < J) {
    const int j = threadIdx.x;
    double ln[I];
    double mx = -1.0;
#pragma unroll
    for (int i = 0; i < I; ++i) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w][j * I + i];
      ln[i] = s / double(N);
      mx = fmax(mx, ln[i]);
    }
#pragma unroll
    for (int i = 0; i < I; ++i) ((R*)a.lam_out)[((u * J + j) * F + f) * I + i] = R(fmax(ln[i], 1e-12 * mx));
  }
}

template <typename R>
static void* mstep_fn(int I) {
  switch (I) {
    case 1: return (void*)mstep_kernel<R, 1>;
    case 2: return (void*)mstep_kernel<R, 2>;
    case 3: return (void*)mstep_kernel<R, 3>;
    case 4: return (void*)mstep_kernel<R, 4>;
    case 5: return (void*)mstep_kernel<R, 5>;
    case 6: return (void*)mstep_kernel<R, 6>;
    case 7: return (void*)mstep_kernel<R, 7>;
    case 8: return (void*)mstep_kernel<R, 8>;
  }
  return nullptr;
}

}  // namespace ffca

using namespace ffca;

extern "C" int ffca_mstep_diag(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                               const void* mu, const void* phi, const void* lam, int vf_mode, double vf_scalar,
                               const void* vf, void* v_out, void* lam_out) {
  reset_launches();
  if (!check_dims(dtype, U, I, J, N, F)) return FFCA_E_ARG;
  if (I > 8 || J > 8 || !(vf_mode == FFCA_VF_SCALAR || vf_mode == FFCA_VF_BIN || vf_mode == FFCA_VF_FULL)) {
    set_error("unsupported I=%d J=%d vf_mode=%d", I, J, vf_mode);
    return FFCA_E_UNSUPPORTED;
  }
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  const long long nb = (long long)U * F;
  if (nb == 0) return FFCA_OK;
  Staging st(mem, s);
  MstepArgs a = {};
  a.U = U; a.I = I; a.J = J; a.N = N; a.F = F;
  a.vf_mode = vf_mode; a.vf_scalar = vf_scalar;
  FFCA_TRY(st.in(mu, size_t(U) * J * N * F * I * cs, &a.mu));
  FFCA_TRY(st.in(phi, size_t(U) * J * N * F * I * rs, &a.phi));
  FFCA_TRY(st.in(lam, size_t(U) * J * F * I * rs, &a.lam));
  if (vf_mode == FFCA_VF_BIN) FFCA_TRY(st.in(vf, size_t(nb) * rs, &a.vf));
  if (vf_mode == FFCA_VF_FULL) FFCA_TRY(st.in(vf, size_t(U) * J * N * F * rs, &a.vf));
  FFCA_TRY(st.out(v_out, size_t(U) * J * N * F * rs, &a.v_out));
  FFCA_TRY(st.out(lam_out, size_t(U) * J * F * I * rs, &a.lam_out));
  void* fn = dtype == FFCA_C64 ? mstep_fn<float>(I) : mstep_fn<double>(I);
  void* args[] = {(void*)&a};
  FFCA_CK(cudaLaunchKernel(fn, dim3(unsigned(nb)), dim3(128), args, 0, s));
  count_launch();
  FFCA_TRY(st.flush());
  FFCA_CK(cudaStreamSynchronize(s));
  return FFCA_OK;
}
