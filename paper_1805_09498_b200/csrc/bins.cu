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

// ---------------------------------------------------------------------------
// Initialisers (scene.oracle_covariances / diffuse_covariances, scene.py:207-247)
// ---------------------------------------------------------------------------
namespace ffca {

// Bins are the fastest axis of every (.., N, F) array, so a CTA owns a tile of
// INIT_FT consecutive bins (one per lane: every load is a 32-bin coalesced row)
// and INIT_NG warps split the frames; the per-bin sums are combined across
// warps in shared memory in a fixed order (deterministic).
constexpr int INIT_FT = 32, INIT_NG = 8;

// One frame of one bin: v_hat out, power-weighted outer product into acc (packed lower triangle:
// diag at a*a, (a, b<a) re/im at a*a+1+2b).
template <typename R, int I, int MODE>
__device__ __forceinline__ void init_accumulate(const typename Cpx<R>::T (&t)[I], double fl, int J, double invJ,
                                                R* __restrict__ v, long long vstride, double (&acc)[I * I]) {
  double2 z[I];
  double p = 0.0;
#pragma unroll
  for (int i = 0; i < I; ++i) {
    z[i] = make_double2(double(t[i].x), double(t[i].y));
    p += z[i].x * z[i].x + z[i].y * z[i].y;
  }
  // p / I and p / I / J as products with compile-time / per-call reciprocals (<= 2 ulp from the
  // reference's divisions); 1 / v_hat via MUFU seed + 2 Newton steps (fp64-accurate)
  constexpr double invI = 1.0 / I;
  double2 zw[I];  // MODE 0: z / v_hat; MODE 1: z
#pragma unroll
  for (int i = 0; i < I; ++i) zw[i] = z[i];
  if (MODE == 0) {
    const double vh = fmax(p * invI, fl);
    *v = R(vh);
    const double w = rcp(vh);
#pragma unroll
    for (int i = 0; i < I; ++i) zw[i] = make_double2(z[i].x * w, z[i].y * w);  // acc += z_a (w z_b)^*
  } else {
    const R vh = R(fmax(p * invI * invJ, fl));
    for (int jj = 0; jj < J; ++jj) v[jj * vstride] = vh;
  }
#pragma unroll
  for (int a = 0; a < I; ++a) {
    const double2 za = z[a];
    acc[a * a] += za.x * zw[a].x + za.y * zw[a].y;
#pragma unroll
    for (int b = 0; b < a; ++b) {
      acc[a * a + 1 + 2 * b] += za.x * zw[b].x + za.y * zw[b].y;
      acc[a * a + 2 + 2 * b] += za.y * zw[b].x - za.x * zw[b].y;
    }
  }
}

// complex64 inputs, 4 frames: the power-normalised outer products in fp32 (scale-free terms of
// magnitude <= I, ~1e-7 relative), summed over the 4 frames in fp32 and then into the fp64
// accumulators -- 2.25 fp32->fp64 conversions per point instead of 2I + 1, which otherwise
// bound the kernel on the FP64 pipe.  Frames whose v_hat is below 1e-30 (silent / floor-only
// points, where fp32 would under- or overflow) take the fp64 path of init_accumulate.
template <int I, int MODE>
__device__ __forceinline__ void init_batch_f32(const float2 (&t)[4][I], double fl, int J, double invJ,
                                               float* __restrict__ v, long long kstride, long long vstride,
                                               double (&acc)[I * I]) {
  constexpr float invI = 1.0f / I;
  const float flf = float(fl), invJf = float(invJ);
  float pa[I * I];
#pragma unroll
  for (int e = 0; e < I * I; ++e) pa[e] = 0.0f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float p = 0.0f;
#pragma unroll
    for (int i = 0; i < I; ++i) p = fmaf(t[k][i].x, t[k][i].x, fmaf(t[k][i].y, t[k][i].y, p));
    const float vh = MODE == 0 ? fmaxf(p * invI, flf) : fmaxf(p * invI * invJf, flf);
    if (!(vh >= 1e-30f)) {
      init_accumulate<float, I, MODE>(t[k], fl, J, invJ, v + k * kstride, vstride, acc);
      continue;
    }
    float w = 1.0f;
    if (MODE == 0) {
      v[k * kstride] = vh;
      w = rcp(vh);
    } else {
      for (int jj = 0; jj < J; ++jj) v[k * kstride + jj * vstride] = vh;
    }
    float2 zw[I];
#pragma unroll
    for (int i = 0; i < I; ++i) zw[i] = make_float2(t[k][i].x * w, t[k][i].y * w);
#pragma unroll
    for (int a = 0; a < I; ++a) {
      const float2 za = t[k][a];
      pa[a * a] = fmaf(za.x, zw[a].x, fmaf(za.y, zw[a].y, pa[a * a]));
#pragma unroll
      for (int b = 0; b < a; ++b) {
        pa[a * a + 1 + 2 * b] = fmaf(za.x, zw[b].x, fmaf(za.y, zw[b].y, pa[a * a + 1 + 2 * b]));
        pa[a * a + 2 + 2 * b] = fmaf(za.y, zw[b].x, fmaf(-za.x, zw[b].y, pa[a * a + 2 + 2 * b]));
      }
    }
  }
#pragma unroll
  for (int e = 0; e < I * I; ++e) acc[e] += double(pa[e]);
}

// One CTA per (mixture, source, bin tile) [oracle] or (mixture, bin tile) [diffuse]:
//   v_hat = max(sum_i |x_i|^2 / I, floor_f) per frame (diffuse: power / J),
//   S_hat = sum_n x x^H w / N (w = 1 / v_hat [oracle], 1 [diffuse]) + 0.5 scale W_j [diffuse]
//   then diagonal loading 1e-9 tr / I, identity when tr <= 0 (scene._load_pd, scene.py:200-204).
template <typename R, int I, int MODE>
__global__ void __launch_bounds__(INIT_FT* INIT_NG, (I <= 4 ? 3 : 1)) init_cov_kernel(const void* xv, const double* floor_f,
                                                                    const void* Wv, void* Sv, void* vv, int U,
                                                                    int J, int N, int F) {
  using C2 = typename Cpx<R>::T;
  const int lane = threadIdx.x & 31, ng = threadIdx.x >> 5;
  const int ftiles = (F + INIT_FT - 1) / INIT_FT;
  const long long blk = blockIdx.x;
  const int f = int(blk % ftiles) * INIT_FT + lane;
  const long long uj = blk / ftiles;
  const int j = MODE == 0 ? int(uj % J) : 0;
  const long long u = MODE == 0 ? uj / J : uj;
  const bool live = f < F;
  const double invJ = 1.0 / J;
  const C2* __restrict__ x = (const C2*)xv;
  const long long xbase = MODE == 0 ? (u * J + j) * (long long)I : u * (long long)I;  // channel-row base
  const double fl = live ? floor_f[u * F + f] : 1.0;
  R* vo = (R*)vv;
  double acc[I * I];  // packed lower triangle: diag a*a, off-diagonal (a, b<a) re/im at a*a+1+2b
#pragma unroll
  for (int e = 0; e < I * I; ++e) acc[e] = 0.0;
  if (live) {
    const C2* __restrict__ xp = x + xbase * N * (long long)F + f;
    R* __restrict__ vp = vo + ((u * J + j) * N) * (long long)F + f;
    const long long cstride = (long long)N * F, vstride = (long long)N * F;
    int n = ng;
    // 4 frames per trip: all 4*I loads are issued before the first use (memory-level parallelism)
    for (; n + 3 * INIT_NG < N; n += 4 * INIT_NG) {
      C2 t[4][I];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < I; ++i) t[k][i] = xp[i * cstride + (long long)(n + k * INIT_NG) * F];
      if constexpr (sizeof(R) == 4 && I <= 4) {
        init_batch_f32<I, MODE>(t, fl, J, invJ, vp + (long long)n * F, (long long)INIT_NG * F, vstride, acc);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          init_accumulate<R, I, MODE>(t[k], fl, J, invJ, vp + (long long)(n + k * INIT_NG) * F, vstride, acc);
      }
    }
    for (; n < N; n += INIT_NG) {
      C2 t[I];
#pragma unroll
      for (int i = 0; i < I; ++i) t[i] = xp[i * cstride + (long long)n * F];
      init_accumulate<R, I, MODE>(t, fl, J, invJ, vp + (long long)n * F, vstride, acc);
    }
  }
  __shared__ double red[INIT_NG][INIT_FT];
#pragma unroll
  for (int e = 0; e < I * I; ++e) {
    red[ng][lane] = acc[e];
    __syncthreads();
    if (ng == 0) {
      double t = red[0][lane];
#pragma unroll
      for (int g = 1; g < INIT_NG; ++g) t += red[g][lane];
      acc[e] = t / N;
    }
    __syncthreads();
  }
  if (ng != 0 || !live) return;
  const C2* W = (const C2*)Wv;
  double scale = 0.0;
  if (MODE == 1) {
#pragma unroll
    for (int a = 0; a < I; ++a) scale += acc[a * a];
    scale = fmax(scale / I, 1e-300);
  }
  const int jlo = MODE == 0 ? j : 0, jhi = MODE == 0 ? j + 1 : J;
  for (int jj = jlo; jj < jhi; ++jj) {
    double Sd[I * I];
#pragma unroll
    for (int e = 0; e < I * I; ++e) Sd[e] = acc[e];
    if (MODE == 1) {  // avg + 0.5 scale W_j, W (J, I, I) Hermitian, shared by every mixture
      const C2* Wj = W + jj * I * I;
#pragma unroll
      for (int a = 0; a < I; ++a) {
        Sd[a * a] += 0.5 * scale * double(Wj[a * I + a].x);
#pragma unroll
        for (int b = 0; b < a; ++b) {
          Sd[a * a + 1 + 2 * b] += 0.5 * scale * double(Wj[a * I + b].x);
          Sd[a * a + 2 + 2 * b] += 0.5 * scale * double(Wj[a * I + b].y);
        }
      }
    }
    double tr = 0.0;
#pragma unroll
    for (int a = 0; a < I; ++a) tr += Sd[a * a];
    const double sc = tr / I;
    const double load = sc > 0.0 ? 1e-9 * sc : 1.0;
    C2* S = (C2*)Sv + ((u * J + jj) * F + f) * I * I;
#pragma unroll
    for (int a = 0; a < I; ++a) {
      S[a * I + a] = mk<C2, R>(R(Sd[a * a] + load), R(0));
#pragma unroll
      for (int b = 0; b < a; ++b) {
        const double re = Sd[a * a + 1 + 2 * b], im = Sd[a * a + 2 + 2 * b];
        S[a * I + b] = mk<C2, R>(R(re), R(im));
        S[b * I + a] = mk<C2, R>(R(re), R(-im));
      }
    }
  }
}

template <typename R, int I>
static void launch_init(int mode, unsigned blocks, cudaStream_t s, const void* x, const double* fl, const void* W,
                        void* S, void* v, int U, int J, int N, int F) {
  if (mode == 0)
    init_cov_kernel<R, I, 0><<<blocks, INIT_FT * INIT_NG, 0, s>>>(x, fl, W, S, v, U, J, N, F);
  else
    init_cov_kernel<R, I, 1><<<blocks, INIT_FT * INIT_NG, 0, s>>>(x, fl, W, S, v, U, J, N, F);
}

}  // namespace ffca

// refs (U,J,I,N,F) -> S_hat (U,J,F,I,I), v_hat (U,J,N,F); floor (U,F) from ffca_power_floor.
extern "C" int ffca_init_covariances(int device, void* stream, int mem, int dtype, int mode, int U, int I, int J,
                                     int N, int F, const void* x, const double* floor_f, const void* W, void* S_out,
                                     void* v_out) {
  reset_launches();
  if (!check_dims(dtype, U, I, J, N, F) || I > 8 || (mode != 0 && mode != 1) || !x || !floor_f || !S_out ||
      !v_out || (mode == 1 && !W)) {
    set_error("bad arguments to ffca_init_covariances");
    return FFCA_E_ARG;
  }
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  Staging st(mem, s);
  const void *dx, *dW = nullptr, *dfl;
  void *dS, *dv;
  const size_t xcount = mode == 0 ? size_t(U) * J * I * N * F : size_t(U) * I * N * F;
  FFCA_TRY(st.in(x, xcount * cs, &dx));
  FFCA_TRY(st.in(floor_f, size_t(U) * F * 8, &dfl));
  if (mode == 1) FFCA_TRY(st.in(W, size_t(J) * I * I * cs, &dW));
  FFCA_TRY(st.out(S_out, size_t(U) * J * F * I * I * cs, &dS));
  FFCA_TRY(st.out(v_out, size_t(U) * J * N * F * rs, &dv));
  const long long ftiles = (F + INIT_FT - 1) / INIT_FT;
  const unsigned blocks = unsigned(mode == 0 ? (long long)U * J * ftiles : (long long)U * ftiles);
  if (blocks) {
    if (dtype == FFCA_C64) {
      FFCA_I_SWITCH(I, (launch_init<float, II>(mode, blocks, s, dx, (const double*)dfl, dW, dS, dv, U, J, N, F)))
    } else {
      FFCA_I_SWITCH(I, (launch_init<double, II>(mode, blocks, s, dx, (const double*)dfl, dW, dS, dv, U, J, N, F)))
    }
    count_launch();
  }
  FFCA_CK(cudaGetLastError());
  FFCA_TRY(st.flush());
  FFCA_CK(cudaStreamSynchronize(s));
  return FFCA_OK;
}
