// Per-bin small linear algebra of the FastFCA-AS API surface (sm_100a):
//   reconstruct_spatial_covariances  S_j = P^-H diag(lam_j) P^-1      (fastfca.py:119-135)
//   back_transform_stats (phi part)  P^-H diag(phi_t) P^-1 per point   (fastfca.py:276-287)
//   params_from_covariances          whitening init                    (fastfca.py:290-309)
// All per-bin algebra is fp64; one thread per (source, bin) or per point.
#include "common.cuh"
#include "host_common.h"

namespace ffca {

// Q = P^-H for every bin, (nb, I, I) fp64 (from points.cu).
int launch_inv_PH(int dtype, int I, const void* P, double2* Q, int* status, long long nbins, cudaStream_t s);

// S_j[a][b] = sum_i Q[a][i] lam_ji conj(Q[b][i]), hermitized (lower triangle mirrored, real diagonal).
template <typename R, int I>
__global__ void reconstruct_kernel(const double2* Q, const void* lamv, void* Sv, int U, int J, int F) {
  using C2 = typename Cpx<R>::T;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)U * J * F;
  if (t >= total) return;
  const int f = int(t % F);
  const long long uj = t / F;
  const int j = int(uj % J);
  const long long u = uj / J;
  const double2* q = Q + (u * F + f) * I * I;
  const R* lam = (const R*)lamv + ((u * J + j) * F + f) * I;
  C2* S = (C2*)Sv + ((u * J + j) * F + f) * I * I;
#pragma unroll
  for (int x = 0; x < I; ++x)
#pragma unroll
    for (int b = 0; b <= x; ++b) {
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int i = 0; i < I; ++i) {
        const double2 p = q[x * I + i], r = q[b * I + i];
        const double l = double(lam[i]);
        re += l * (p.x * r.x + p.y * r.y);
        im += l * (p.y * r.x - p.x * r.y);
      }
      if (x == b) S[x * I + x] = mk<C2, R>(R(re), R(0));
      else {
        S[x * I + b] = mk<C2, R>(R(re), R(im));
        S[b * I + x] = mk<C2, R>(R(re), R(-im));
      }
    }
}

// phi_full[u,j,n,f] = Q diag(phi_t) Q^H, hermitized, (U,J,N,F,I,I).
template <typename R, int I>
__global__ void back_phi_kernel(const double2* Q, const void* phiv, void* outv, int U, int J, int N, int F) {
  using C2 = typename Cpx<R>::T;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)U * J * N * F;
  if (t >= total) return;
  const int f = int(t % F);
  const long long ujn = t / F;
  const long long u = ujn / ((long long)J * N);
  const double2* q = Q + (u * F + f) * I * I;
  const R* ph = (const R*)phiv + t * I;
  C2* out = (C2*)outv + t * I * I;
  double d[I];
#pragma unroll
  for (int i = 0; i < I; ++i) d[i] = double(ph[i]);
#pragma unroll
  for (int x = 0; x < I; ++x)
#pragma unroll
    for (int b = 0; b <= x; ++b) {
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int i = 0; i < I; ++i) {
        const double2 p = q[x * I + i], r = q[b * I + i];
        re += d[i] * (p.x * r.x + p.y * r.y);
        im += d[i] * (p.y * r.x - p.x * r.y);
      }
      if (x == b) out[x * I + x] = mk<C2, R>(R(re), R(0));
      else {
        out[x * I + b] = mk<C2, R>(R(re), R(im));
        out[b * I + x] = mk<C2, R>(R(re), R(-im));
      }
    }
}

// Whitening init per bin: T = sum_j S_j = L L^H (Cholesky, fails -> NotPD),
// P = (L^H)^-1, lam_ji = Re (P^H S_j P)_ii floored at 1e-12 max_i.
template <typename R, int I>
__global__ void whiten_kernel(const void* Sv, void* Pv, void* lamv, int* status, int U, int J, int F) {
  using C2 = typename Cpx<R>::T;
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= (long long)U * F) return;
  const long long u = b / F;
  const int f = int(b % F);
  const C2* S = (const C2*)Sv;
  double2 Lm[I][I];
#pragma unroll
  for (int x = 0; x < I; ++x)
#pragma unroll
    for (int y = 0; y < I; ++y) Lm[x][y] = make_double2(0.0, 0.0);
  for (int j = 0; j < J; ++j) {
    const C2* Sj = S + ((u * J + j) * F + f) * I * I;
#pragma unroll
    for (int x = 0; x < I; ++x)
#pragma unroll
      for (int y = 0; y <= x; ++y) {
        Lm[x][y].x += double(Sj[x * I + y].x);
        Lm[x][y].y += double(Sj[x * I + y].y);
      }
  }
  // Cholesky (lower), LAPACK zpotrf semantics: fail on a non-positive pivot
  bool ok = true;
#pragma unroll
  for (int k = 0; k < I; ++k) {
    double dk = Lm[k][k].x;
#pragma unroll
    for (int c = 0; c < k; ++c) dk -= Lm[k][c].x * Lm[k][c].x + Lm[k][c].y * Lm[k][c].y;
    if (!(dk > 0.0)) ok = false;
    const double lk = sqrt(fmax(dk, 0.0));
    Lm[k][k] = make_double2(lk, 0.0);
    const double il = lk > 0.0 ? 1.0 / lk : 0.0;
#pragma unroll
    for (int r = k + 1; r < I; ++r) {
      double2 acc = Lm[r][k];
#pragma unroll
      for (int c = 0; c < k; ++c) {  // acc -= L[r][c] conj(L[k][c])
        acc.x -= Lm[r][c].x * Lm[k][c].x + Lm[r][c].y * Lm[k][c].y;
        acc.y -= Lm[r][c].y * Lm[k][c].x - Lm[r][c].x * Lm[k][c].y;
      }
      Lm[r][k] = make_double2(acc.x * il, acc.y * il);
    }
  }
  if (!ok) {
    status[b] |= ST_NOT_PD;
    return;
  }
  // X = L^-1 (lower), P = X^H : P[a][c] = conj(X[c][a])
  double2 X[I][I];
#pragma unroll
  for (int c = 0; c < I; ++c) {
#pragma unroll
    for (int r = 0; r < I; ++r) {
      double2 acc = make_double2(r == c ? 1.0 : 0.0, 0.0);
#pragma unroll
      for (int k = 0; k < r; ++k) {
        acc.x -= Lm[r][k].x * X[k][c].x - Lm[r][k].y * X[k][c].y;
        acc.y -= Lm[r][k].x * X[k][c].y + Lm[r][k].y * X[k][c].x;
      }
      const double il = 1.0 / Lm[r][r].x;
      X[r][c] = make_double2(acc.x * il, acc.y * il);
    }
  }
  C2* P = (C2*)Pv + b * I * I;
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int c = 0; c < I; ++c) P[a * I + c] = mk<C2, R>(R(X[c][a].x), R(-X[c][a].y));
  // lam_ji = Re sum_ab conj(P[a][i]) S_j[a][b] P[b][i] = Re (X S_j X^H)_ii
  for (int j = 0; j < J; ++j) {
    const C2* Sj = S + ((u * J + j) * F + f) * I * I;
    double l[I];
    double mx = -1.0;
#pragma unroll
    for (int i = 0; i < I; ++i) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < I; ++a) {
        double2 t = make_double2(0.0, 0.0);  // (S X^H)[a][i] = sum_b S[a][b] conj(X[i][b])
#pragma unroll
        for (int bb = 0; bb < I; ++bb) {
          const C2 sv = Sj[a * I + bb];
          const double2 xv = X[i][bb];
          t.x += double(sv.x) * xv.x + double(sv.y) * xv.y;
          t.y += double(sv.y) * xv.x - double(sv.x) * xv.y;
        }
        s += X[i][a].x * t.x - X[i][a].y * t.y;
      }
      l[i] = s;
      mx = fmax(mx, s);
    }
#pragma unroll
    for (int i = 0; i < I; ++i) ((R*)lamv)[((u * J + j) * F + f) * I + i] = R(fmax(l[i], 1e-12 * mx));
  }
}

#define FFCA_I_SWITCH(I, EXPR) \
  switch (I) {                 \
    case 1: { constexpr int II = 1; EXPR; } break; \
    case 2: { constexpr int II = 2; EXPR; } break; \
    case 3: { constexpr int II = 3; EXPR; } break; \
    case 4: { constexpr int II = 4; EXPR; } break; \
    case 5: { constexpr int II = 5; EXPR; } break; \
    case 6: { constexpr int II = 6; EXPR; } break; \
    case 7: { constexpr int II = 7; EXPR; } break; \
    case 8: { constexpr int II = 8; EXPR; } break; \
  }

}  // namespace ffca

using namespace ffca;

extern "C" int ffca_reconstruct_covariances(int device, void* stream, int mem, int dtype, int U, int I, int J,
                                            int F, const void* P, const void* lam, void* S, int* status) {
  reset_launches();
  if (!check_dims(dtype, U, I, J, 1, F) || I > 8 || !P || !lam || !S) {
    set_error("bad arguments to ffca_reconstruct_covariances");
    return FFCA_E_ARG;
  }
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const long long nb = (long long)U * F;
  if (nb == 0) return FFCA_OK;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  Staging st(mem, s);
  const void *dP, *dl;
  void *dS, *Q, *dstatus;
  FFCA_TRY(st.in(P, size_t(nb) * I * I * cs, &dP));
  FFCA_TRY(st.in(lam, size_t(U) * J * F * I * rs, &dl));
  FFCA_TRY(st.out(S, size_t(U) * J * F * I * I * cs, &dS));
  FFCA_TRY(st.scratch(size_t(nb) * I * I * 16, &Q));
  FFCA_TRY(st.scratch(size_t(nb) * 4, &dstatus));
  FFCA_CK(cudaMemsetAsync(dstatus, 0, size_t(nb) * 4, s));
  FFCA_TRY(launch_inv_PH(dtype, I, dP, (double2*)Q, (int*)dstatus, nb, s));
  const long long total = (long long)U * J * F;
  const unsigned blocks = unsigned((total + 127) / 128);
  if (dtype == FFCA_C64) {
    FFCA_I_SWITCH(I, (reconstruct_kernel<float, II><<<blocks, 128, 0, s>>>((const double2*)Q, dl, dS, U, J, F)))
  } else {
    FFCA_I_SWITCH(I, (reconstruct_kernel<double, II><<<blocks, 128, 0, s>>>((const double2*)Q, dl, dS, U, J, F)))
  }
  count_launch();
  FFCA_CK(cudaGetLastError());
  FFCA_TRY(st.flush());
  return finish_status((const int*)dstatus, status, nb, mem, s, FFCA_ST_SINGULAR_P);
}

extern "C" int ffca_back_transform_phi(int device, void* stream, int mem, int dtype, int U, int I, int J, int N,
                                       int F, const void* P, const void* phi_t, void* phi_out, int* status) {
  reset_launches();
  if (!check_dims(dtype, U, I, J, N, F) || I > 8 || !P || !phi_t || !phi_out) {
    set_error("bad arguments to ffca_back_transform_phi");
    return FFCA_E_ARG;
  }
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const long long nb = (long long)U * F;
  if (nb == 0) return FFCA_OK;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  Staging st(mem, s);
  const void *dP, *dph;
  void *dout, *Q, *dstatus;
  FFCA_TRY(st.in(P, size_t(nb) * I * I * cs, &dP));
  FFCA_TRY(st.in(phi_t, size_t(U) * J * N * F * I * rs, &dph));
  FFCA_TRY(st.out(phi_out, size_t(U) * J * N * F * I * I * cs, &dout));
  FFCA_TRY(st.scratch(size_t(nb) * I * I * 16, &Q));
  FFCA_TRY(st.scratch(size_t(nb) * 4, &dstatus));
  FFCA_CK(cudaMemsetAsync(dstatus, 0, size_t(nb) * 4, s));
  FFCA_TRY(launch_inv_PH(dtype, I, dP, (double2*)Q, (int*)dstatus, nb, s));
  const long long total = (long long)U * J * N * F;
  const unsigned blocks = unsigned((total + 127) / 128);
  if (dtype == FFCA_C64) {
    FFCA_I_SWITCH(I, (back_phi_kernel<float, II><<<blocks, 128, 0, s>>>((const double2*)Q, dph, dout, U, J, N, F)))
  } else {
    FFCA_I_SWITCH(I, (back_phi_kernel<double, II><<<blocks, 128, 0, s>>>((const double2*)Q, dph, dout, U, J, N, F)))
  }
  count_launch();
  FFCA_CK(cudaGetLastError());
  FFCA_TRY(st.flush());
  return finish_status((const int*)dstatus, status, nb, mem, s, FFCA_ST_SINGULAR_P);
}

extern "C" int ffca_params_from_covariances(int device, void* stream, int mem, int dtype, int U, int I, int J,
                                            int F, const void* S_hat, void* P_out, void* lam_out, int* status) {
  reset_launches();
  if (!check_dims(dtype, U, I, J, 1, F) || I > 8 || !S_hat || !P_out || !lam_out) {
    set_error("bad arguments to ffca_params_from_covariances");
    return FFCA_E_ARG;
  }
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const long long nb = (long long)U * F;
  if (nb == 0) return FFCA_OK;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  Staging st(mem, s);
  const void* dS;
  void *dP, *dl, *dstatus;
  FFCA_TRY(st.in(S_hat, size_t(U) * J * F * I * I * cs, &dS));
  FFCA_TRY(st.out(P_out, size_t(nb) * I * I * cs, &dP));
  FFCA_TRY(st.out(lam_out, size_t(U) * J * F * I * rs, &dl));
  FFCA_TRY(st.scratch(size_t(nb) * 4, &dstatus));
  FFCA_CK(cudaMemsetAsync(dstatus, 0, size_t(nb) * 4, s));
  const unsigned blocks = unsigned((nb + 127) / 128);
  if (dtype == FFCA_C64) {
    FFCA_I_SWITCH(I, (whiten_kernel<float, II><<<blocks, 128, 0, s>>>(dS, dP, dl, (int*)dstatus, U, J, F)))
  } else {
    FFCA_I_SWITCH(I, (whiten_kernel<double, II><<<blocks, 128, 0, s>>>(dS, dP, dl, (int*)dstatus, U, J, F)))
  }
  count_launch();
  FFCA_CK(cudaGetLastError());
  FFCA_TRY(st.flush());
  return finish_status((const int*)dstatus, status, nb, mem, s, FFCA_ST_NOT_PD);
}
