// C-ABI: conventional FCA baseline (fca.run_fca / e_step / log_likelihood) on sm_100a.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "fca_loop.cuh"
#include "host_common.h"

namespace ffca {

using FcaFn = void (*)(const FcaArgs);

template <typename R>
static FcaFn fca_kernel(int I, int J) {
  if (I == 3 && J == 3) return fca_loop_kernel<R, 3, 3>;
  if (I == 2 && J == 2) return fca_loop_kernel<R, 2, 2>;
  if (J > 4) return nullptr;
  switch (I) {
    case 1: return fca_loop_kernel<R, 1, 0>;
    case 2: return fca_loop_kernel<R, 2, 0>;
    case 3: return fca_loop_kernel<R, 3, 0>;
    case 4: return fca_loop_kernel<R, 4, 0>;
  }
  return nullptr;
}

static int fca_jm(int I, int J) { return ((I == 3 && J == 3) || (I == 2 && J == 2)) ? J : 4; }

struct FcaPlan {
  int C = 1, NL = 0, threads = 64;
  size_t smem = 0;
  FcaSmem L;
};

static int plan_fca(int dtype, int I, int J, int N, int vf_mode, FcaPlan& p, size_t optin) {
  const int rsz = int(rsize(dtype));
  const int VMAX = fca_jm(I, J) * I * I + 1;
  for (int C = 1; C <= 8; C <<= 1) {
    if (C > 1 && C > N) break;
    p.C = C;
    p.NL = (N + C - 1) / C;
    int t = ((p.NL + 3) / 4 + 31) / 32 * 32;
    // 255-register instantiations: 128-thread CTAs keep two resident per SM
    p.threads = t < 64 ? 64 : (t > 128 ? 128 : t);
    if (const char* ft = getenv("FFCA_FCA_THREADS")) {  // tuning hook
      const int v = atoi(ft);
      if (v >= 64 && v <= 256 && v % 32 == 0) p.threads = v;
    }
    FcaSmem L(I, J, p.NL, p.threads / 32, rsz, vf_mode, VMAX);
    p.L = L;
    p.smem = L.total;
    if (L.slab <= 100 * 1024 && p.smem <= optin) return FFCA_OK;
  }
  set_error("FCA: bin of %d frames does not fit the cluster's shared memory", N);
  return FFCA_E_UNSUPPORTED;
}

static int fca_launch(int device, int dtype, const FcaArgs& a, cudaStream_t s, const FcaPlan& p) {
  FcaFn fn = dtype == FFCA_C64 ? fca_kernel<float>(a.I, a.J) : fca_kernel<double>(a.I, a.J);
  if (!fn) {
    set_error("FCA kernel supports I <= 4 with J <= 4 (and I=J=3 / I=J=2 exactly); got I=%d J=%d", a.I, a.J);
    return FFCA_E_UNSUPPORTED;
  }
  (void)device;
  FFCA_CK(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p.smem)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(a.total_bins * p.C), 1, 1);
  cfg.blockDim = dim3(unsigned(p.threads), 1, 1);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (p.C > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(p.C);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  FcaArgs b = a;
  b.L = p.L;
  FFCA_CK(cudaLaunchKernelEx(&cfg, fn, b));
  count_launch();
  return FFCA_OK;
}

// Per-point full-matrix E-step (fca.e_step, fca.py:119-144) for ffca_fca_estep.
struct FcaEstepArgs {
  int U, I, J, N, F;
  const void* y;
  const void* S;
  const void* v;
  void* mu;
  void* phi;
  int images_layout;
  int* status;
};

template <typename R, int I>
__global__ void __launch_bounds__(256) fca_estep_kernel(const FcaEstepArgs a) {
  using C2 = typename Cpx<R>::T;
  const long long npts = (long long)a.U * a.N * a.F;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= npts) return;
  const int F = a.F, N = a.N, J = a.J;
  const int f = int(t % F);
  const long long un = t / F;
  const int n = int(un % N);
  const long long u = un / N;
  const C2* y = (const C2*)a.y;
  const C2* S = (const C2*)a.S;
  const R* v = (const R*)a.v;
  C2 yv[I];
#pragma unroll
  for (int i = 0; i < I; ++i) yv[i] = y[((u * I + i) * N + n) * (long long)F + f];
  // mixture (lower) and LDL^H
  C2 L[I][I];
  R d[I], rd[I];
#pragma unroll
  for (int x = 0; x < I; ++x)
#pragma unroll
    for (int b = 0; b <= x; ++b) L[x][b] = mk<C2, R>(R(0), R(0));
  for (int j = 0; j < J; ++j) {
    const R vj = v[((u * J + j) * N + n) * (long long)F + f];
    const C2* Sj = S + ((u * J + j) * F + f) * I * I;
#pragma unroll
    for (int x = 0; x < I; ++x)
#pragma unroll
      for (int b = 0; b <= x; ++b) {
        L[x][b].x = fma(vj, Sj[x * I + b].x, L[x][b].x);
        L[x][b].y = fma(vj, Sj[x * I + b].y, L[x][b].y);
      }
  }
  bool bad = false;
#pragma unroll
  for (int k = 0; k < I; ++k) {
    R dk = L[k][k].x;
#pragma unroll
    for (int c = 0; c < k; ++c) dk -= (L[k][c].x * L[k][c].x + L[k][c].y * L[k][c].y) * d[c];
    d[k] = dk;
    bad = bad || dk == R(0);
    rd[k] = rcp(dk);
#pragma unroll
    for (int r = k + 1; r < I; ++r) {
      C2 acc = L[r][k];
#pragma unroll
      for (int c = 0; c < k; ++c) {
        const C2 lr = L[r][c], lk = L[k][c];
        acc.x -= (lr.x * lk.x + lr.y * lk.y) * d[c];
        acc.y -= (lr.y * lk.x - lr.x * lk.y) * d[c];
      }
      L[r][k] = mk<C2, R>(acc.x * rd[k], acc.y * rd[k]);
    }
  }
  if (bad && a.status) atomicOr(&a.status[u * F + f], ST_NOT_PD);
  C2 z[I];
#pragma unroll
  for (int r = 0; r < I; ++r) {
    C2 s = yv[r];
#pragma unroll
    for (int c = 0; c < r; ++c) {
      s.x -= L[r][c].x * z[c].x - L[r][c].y * z[c].y;
      s.y -= L[r][c].x * z[c].y + L[r][c].y * z[c].x;
    }
    z[r] = s;
  }
#pragma unroll
  for (int r = 0; r < I; ++r) z[r] = mk<C2, R>(z[r].x * rd[r], z[r].y * rd[r]);
#pragma unroll
  for (int r = I - 1; r >= 0; --r)
#pragma unroll
    for (int c = r + 1; c < I; ++c) {
      const C2 lv = L[c][r];
      z[r].x -= lv.x * z[c].x + lv.y * z[c].y;
      z[r].y -= lv.x * z[c].y - lv.y * z[c].x;
    }
  C2* mu = (C2*)a.mu;
  C2* phi = (C2*)a.phi;
  for (int j = 0; j < J; ++j) {
    const R vj = v[((u * J + j) * N + n) * (long long)F + f];
    const C2* Sj = S + ((u * J + j) * F + f) * I * I;
    C2 Rm[I][I];
#pragma unroll
    for (int x = 0; x < I; ++x) {
      Rm[x][x] = mk<C2, R>(vj * Sj[x * I + x].x, R(0));
#pragma unroll
      for (int b = 0; b < x; ++b) {
        const C2 s = Sj[x * I + b];
        Rm[x][b] = mk<C2, R>(vj * s.x, vj * s.y);
        Rm[b][x] = mk<C2, R>(vj * s.x, -vj * s.y);
      }
    }
    const long long base = ((u * J + j) * N + n) * (long long)F + f;
    if (mu) {
#pragma unroll
      for (int x = 0; x < I; ++x) {
        C2 s = mk<C2, R>(R(0), R(0));
#pragma unroll
        for (int c = 0; c < I; ++c) {
          s.x = fma(Rm[x][c].x, z[c].x, fma(-Rm[x][c].y, z[c].y, s.x));
          s.y = fma(Rm[x][c].x, z[c].y, fma(Rm[x][c].y, z[c].x, s.y));
        }
        if (a.images_layout)
          mu[(((u * J + j) * I + x) * (long long)N + n) * F + f] = s;
        else
          mu[base * I + x] = s;
      }
    }
    if (phi) {
      C2 Y[I][I];
#pragma unroll
      for (int b = 0; b < I; ++b)
#pragma unroll
        for (int r = 0; r < I; ++r) {
          C2 s = Rm[r][b];
#pragma unroll
          for (int c = 0; c < r; ++c) {
            s.x -= L[r][c].x * Y[c][b].x - L[r][c].y * Y[c][b].y;
            s.y -= L[r][c].x * Y[c][b].y + L[r][c].y * Y[c][b].x;
          }
          Y[r][b] = s;
        }
#pragma unroll
      for (int x = 0; x < I; ++x)
#pragma unroll
        for (int b = 0; b <= x; ++b) {
          R re = R(0), im = R(0);
#pragma unroll
          for (int k = 0; k < I; ++k) {
            const C2 p = Y[k][x], q = Y[k][b];
            re = fma(p.x * q.x + p.y * q.y, rd[k], re);
            im = fma(p.x * q.y - p.y * q.x, rd[k], im);
          }
          const R pre = Rm[x][b].x - re, pim = x == b ? R(0) : Rm[x][b].y - im;
          phi[(base * I + x) * I + b] = mk<C2, R>(pre, pim);
          if (x != b) phi[(base * I + b) * I + x] = mk<C2, R>(pre, -pim);
        }
    }
  }
}

template <typename R>
static void* estep_fn(int I) {
  switch (I) {
    case 1: return (void*)fca_estep_kernel<R, 1>;
    case 2: return (void*)fca_estep_kernel<R, 2>;
    case 3: return (void*)fca_estep_kernel<R, 3>;
    case 4: return (void*)fca_estep_kernel<R, 4>;
    case 5: return (void*)fca_estep_kernel<R, 5>;
    case 6: return (void*)fca_estep_kernel<R, 6>;
    case 7: return (void*)fca_estep_kernel<R, 7>;
    case 8: return (void*)fca_estep_kernel<R, 8>;
  }
  return nullptr;
}

static int fca_entry(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                     const void* y, const void* S0, const void* v0, int vf_mode, double vf_scalar, const void* vf,
                     int iterations, int record_likelihood, void* S_out, void* v_out, void* S_prev,
                     void* v_prev, double* ll_out, int* status) {
  reset_launches();
  if (!check_dims(dtype, U, I, J, N, F)) return FFCA_E_ARG;
  if (iterations < 0 || vf_mode < 0 || vf_mode > 3 || !y || !S0 || !v0 || !S_out || !v_out) {
    set_error("bad arguments to ffca_fca_run");
    return FFCA_E_ARG;
  }
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const long long nb = (long long)U * F;
  if (nb == 0) return FFCA_OK;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  const int nev = 1 + iterations;
  Staging st(mem, s);
  FcaArgs a = {};
  a.U = U; a.I = I; a.J = J; a.N = N; a.F = F; a.total_bins = nb; a.iters = iterations;
  a.vf_mode = vf_mode; a.vf_scalar = vf_scalar;
  FFCA_TRY(st.in(y, size_t(U) * I * N * F * cs, &a.y));
  FFCA_TRY(st.in(S0, size_t(U) * J * F * I * I * cs, &a.S0));
  FFCA_TRY(st.in(v0, size_t(U) * J * N * F * rs, &a.v0));
  if (vf_mode == 1) FFCA_TRY(st.in(vf, size_t(nb) * rs, &a.vf));
  if (vf_mode == 2) FFCA_TRY(st.in(vf, size_t(U) * J * N * F * rs, &a.vf));
  FFCA_TRY(st.out(S_out, size_t(U) * J * F * I * I * cs, &a.S_out));
  FFCA_TRY(st.out(v_out, size_t(U) * J * N * F * rs, &a.v_out));
  if (iterations > 0) {
    FFCA_TRY(st.out(S_prev, size_t(U) * J * F * I * I * cs, &a.S_prev));
    FFCA_TRY(st.out(v_prev, size_t(U) * J * N * F * rs, &a.v_prev));
  }
  void *dstatus, *dll = nullptr, *oll = nullptr;
  FFCA_TRY(st.scratch(size_t(nb) * 4, &dstatus));
  FFCA_CK(cudaMemsetAsync(dstatus, 0, size_t(nb) * 4, s));
  a.status = (int*)dstatus;
  if (record_likelihood) {
    FFCA_TRY(st.scratch(size_t(nb) * nev * 8, &dll));
    a.ll = (double*)dll;
    if (ll_out) FFCA_TRY(st.out(ll_out, size_t(U) * nev * 8, &oll));
  }
  int optin = 0;
  FFCA_CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  FcaPlan p;
  FFCA_TRY(plan_fca(dtype, I, J, N, vf_mode, p, size_t(optin)));
  a.C = p.C;
  a.NL = p.NL;
  FFCA_TRY(fca_launch(device, dtype, a, s, p));
  FFCA_CK(cudaGetLastError());
  if (oll) FFCA_TRY(reduce_ll((const double*)dll, (double*)oll, U, F, nev, -double(N) * F * I * std::log(M_PI), s));
  FFCA_TRY(st.flush());
  return finish_status((const int*)dstatus, status, nb, mem, s, FFCA_ST_NOT_PD);
}

}  // namespace ffca

using namespace ffca;

extern "C" int ffca_fca_run(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                            const void* y, const void* S0, const void* v0, int vf_mode, double vf_scalar,
                            const void* vf, int iterations, int record_likelihood, void* S_out, void* v_out,
                            void* S_prev, void* v_prev, double* ll_out, int* status) {
  return fca_entry(device, stream, mem, dtype, U, I, J, N, F, y, S0, v0, vf_mode, vf_scalar, vf, iterations,
                   record_likelihood, S_out, v_out, S_prev, v_prev, ll_out, status);
}

extern "C" int ffca_fca_loglik(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                               const void* y, const void* S, const void* v, double* ll_out, int* status) {
  if (!check_dims(dtype, U, I, J, N, F)) return FFCA_E_ARG;
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  void *So = nullptr, *vo = nullptr;
  FFCA_CK(cudaMallocAsync(&So, size_t(U) * J * F * I * I * cs + 16, s));
  FFCA_CK(cudaMallocAsync(&vo, size_t(U) * J * N * F * rs + 16, s));
  int rc;
  {
    Staging st(mem, s);
    const void *dy, *dS, *dv;
    void* dll;
    rc = st.in(y, size_t(U) * I * N * F * cs, &dy);
    if (!rc) rc = st.in(S, size_t(U) * J * F * I * I * cs, &dS);
    if (!rc) rc = st.in(v, size_t(U) * J * N * F * rs, &dv);
    if (!rc) rc = st.out(ll_out, size_t(U) * 8, &dll);
    if (!rc) {
      int* dst = (status && mem == FFCA_MEM_DEVICE) ? status : nullptr;
      rc = fca_entry(device, stream, FFCA_MEM_DEVICE, dtype, U, I, J, N, F, dy, dS, dv, FFCA_VF_SCALAR, 0.0,
                     nullptr, 0, 1, So, vo, nullptr, nullptr, (double*)dll, dst);
      if (rc == FFCA_OK) rc = st.flush();
      if (rc == FFCA_OK && cudaStreamSynchronize(s) != cudaSuccess) rc = FFCA_E_CUDA;
    }
  }
  cudaFreeAsync(So, s);
  cudaFreeAsync(vo, s);
  return rc;
}

extern "C" int ffca_fca_estep(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                              const void* y, const void* S, const void* v, void* mu, void* phi, int images_layout,
                              int* status) {
  reset_launches();
  if (!check_dims(dtype, U, I, J, N, F)) return FFCA_E_ARG;
  if (I > 8 || !y || !S || !v) {
    set_error("bad arguments to ffca_fca_estep");
    return FFCA_E_ARG;
  }
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  const long long nb = (long long)U * F;
  const long long npts = nb * N;
  if (npts == 0) return FFCA_OK;
  Staging st(mem, s);
  FcaEstepArgs a = {};
  a.U = U; a.I = I; a.J = J; a.N = N; a.F = F; a.images_layout = images_layout;
  FFCA_TRY(st.in(y, size_t(U) * I * N * F * cs, &a.y));
  FFCA_TRY(st.in(S, size_t(U) * J * F * I * I * cs, &a.S));
  FFCA_TRY(st.in(v, size_t(U) * J * N * F * rs, &a.v));
  FFCA_TRY(st.out(mu, size_t(U) * J * N * F * I * cs, &a.mu));
  FFCA_TRY(st.out(phi, size_t(U) * J * N * F * I * I * cs, &a.phi));
  void* dstatus;
  FFCA_TRY(st.scratch(size_t(nb) * 4, &dstatus));
  FFCA_CK(cudaMemsetAsync(dstatus, 0, size_t(nb) * 4, s));
  a.status = (int*)dstatus;
  void* fn = dtype == FFCA_C64 ? estep_fn<float>(I) : estep_fn<double>(I);
  void* args[] = {(void*)&a};
  FFCA_CK(cudaLaunchKernel(fn, dim3(unsigned((npts + 255) / 256)), dim3(256), args, 0, s));
  count_launch();
  FFCA_TRY(st.flush());
  return finish_status((const int*)dstatus, status, nb, mem, s, FFCA_ST_NOT_PD);
}

// ---------------------------------------------------------------------------
// fca.m_step (fca.py:161-184) from given posterior statistics, and the
// per-bin power floor (fca.power_floor, fca.py:82-89).
// ---------------------------------------------------------------------------
namespace ffca {

struct FcaMstepArgs {
  int U, I, J, N, F;
  const void* mu;   // (U,J,N,F,I) complex
  const void* phi;  // (U,J,N,F,I,I) complex
  const void* S;    // (U,J,F,I,I) complex (old S)
  int vf_mode;
  double vf_scalar;
  const void* vf;
  void* S_out;
  void* v_out;
  int* status;
};

template <typename R, int I>
__global__ void __launch_bounds__(128) fca_mstep_kernel(const FcaMstepArgs a) {
  using C2 = typename Cpx<R>::T;
  constexpr int H = I * I;
  const long long bin = blockIdx.x;
  const int F = a.F, N = a.N, J = a.J;
  const long long u = bin / F;
  const int f = int(bin % F);
  __shared__ double Sinv[8][H];
  __shared__ double part[4][H];
  const C2* S = (const C2*)a.S;
  for (int j = threadIdx.x; j < J; j += blockDim.x) {
    double Sp[H], out[H];
    const C2* Sj = S + ((u * J + j) * F + f) * I * I;
    for (int x = 0; x < I; ++x) {
      Sp[pk_diag(x)] = double(Sj[x * I + x].x);
      for (int b = 0; b < x; ++b) {
        Sp[pk_re(x, b)] = double(Sj[x * I + b].x);
        Sp[pk_re(x, b) + 1] = double(Sj[x * I + b].y);
      }
    }
    const int st = fca_inverse_spatial<I>(Sp, out);
    if (st) atomicOr(&a.status[bin], st);
    for (int e = 0; e < H; ++e) Sinv[j][e] = out[e];
  }
  __syncthreads();
  const C2* mu = (const C2*)a.mu;
  const C2* phi = (const C2*)a.phi;
  for (int j = 0; j < J; ++j) {
    R acc[H];
#pragma unroll
    for (int e = 0; e < H; ++e) acc[e] = R(0);
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      const long long base = ((u * J + j) * N + n) * (long long)F + f;
      C2 m[I];
#pragma unroll
      for (int x = 0; x < I; ++x) m[x] = mu[base * I + x];
      R T[H];
      R tr = R(0);
#pragma unroll
      for (int x = 0; x < I; ++x)
#pragma unroll
        for (int b = 0; b <= x; ++b) {
          const C2 p = phi[(base * I + x) * I + b];
          const R re = m[x].x * m[b].x + m[x].y * m[b].y + p.x;
          const R im = m[x].y * m[b].x - m[x].x * m[b].y + p.y;
          if (x == b) {
            T[pk_diag(x)] = re;
            tr += R(Sinv[j][pk_diag(x)]) * re;
          } else {
            T[pk_re(x, b)] = re;
            T[pk_re(x, b) + 1] = im;
            tr += R(2) * (R(Sinv[j][pk_re(x, b)]) * re + R(Sinv[j][pk_re(x, b) + 1]) * im);
          }
        }
      R fl = R(a.vf_scalar);
      if (a.vf_mode == FFCA_VF_BIN) fl = ((const R*)a.vf)[bin];
      if (a.vf_mode == FFCA_VF_FULL) fl = ((const R*)a.vf)[base];
      const R vn = fmax(tr / R(I), fl);
      ((R*)a.v_out)[base] = vn;
      const R iv = R(1) / vn;
#pragma unroll
      for (int e = 0; e < H; ++e) acc[e] = fma(T[e], iv, acc[e]);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int e = 0; e < H; ++e) {
      R x = warp_sum_seg(acc[e], 1);
      if (lane == 0) part[warp][e] = double(x);
    }
    __syncthreads();
    C2* So = (C2*)a.S_out + ((u * J + j) * F + f) * I * I;
    for (int t = threadIdx.x; t < I * I; t += blockDim.x) {
      const int x = t / I, b = t % I;
      const int hi = x >= b ? x : b, lo = x >= b ? b : x;
      double re = 0.0, im = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        re += hi == lo ? part[w][pk_diag(hi)] : part[w][pk_re(hi, lo)];
        im += hi == lo ? 0.0 : part[w][pk_re(hi, lo) + 1];
      }
      re /= double(N);
      im /= double(N);
      So[t] = mk<C2, R>(R(re), R(x >= b ? im : -im));
    }
    __syncthreads();
  }
}

// np.abs(y) ** 2 (fca.py:88): hypot then square for complex128; for complex64 the fp64
// x^2 + y^2 of fp32 components is exact up to one rounding (more accurate than hypot^2).
__device__ __forceinline__ double abs2_ref(double2 z) {
  const double m = hypot(z.x, z.y);
  return m * m;
}
__device__ __forceinline__ double abs2_ref(float2 z) {
  return fma(double(z.x), double(z.x), double(z.y) * double(z.y));
}

// One CTA per (mixture, tile of 32 bins): lanes own consecutive bins (coalesced rows of the
// (I, N, F) layout), 8 warps split the frames, fixed-order combine in shared memory.
template <typename R>
__global__ void __launch_bounds__(256) power_floor_kernel(const void* yv, double* out, int U, int I, int N, int F) {
  using C2 = typename Cpx<R>::T;
  const int lane = threadIdx.x & 31, ng = threadIdx.x >> 5;
  const int ftiles = (F + 31) / 32;
  const long long u = blockIdx.x / ftiles;
  const int f = int(blockIdx.x % ftiles) * 32 + lane;
  const C2* y = (const C2*)yv;
  double s = 0.0;
  if (f < F) {
    const C2* __restrict__ yp = y + u * I * (long long)N * F + f;
    const long long rows = (long long)I * N;  // (i, n) rows are contiguous: one flat frame index
    long long r = ng;
    for (; r + 24 < rows; r += 32) {  // 4 rows in flight per thread
      C2 z[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) z[k] = yp[(r + 8 * k) * F];
#pragma unroll
      for (int k = 0; k < 4; ++k) s += abs2_ref(z[k]);
    }
    for (; r < rows; r += 8) {
      s += abs2_ref(yp[r * F]);
    }
  }
  __shared__ double red[8][32];
  red[ng][lane] = s;
  __syncthreads();
  if (ng != 0 || f >= F) return;
  double t = red[0][lane];
#pragma unroll
  for (int g = 1; g < 8; ++g) t += red[g][lane];
  out[u * F + f] = fmax(1e-10 * (t / (double(I) * N)), 1e-300);
}

template <typename R>
static void* fca_mstep_fn(int I) {
  switch (I) {
    case 1: return (void*)fca_mstep_kernel<R, 1>;
    case 2: return (void*)fca_mstep_kernel<R, 2>;
    case 3: return (void*)fca_mstep_kernel<R, 3>;
    case 4: return (void*)fca_mstep_kernel<R, 4>;
    case 5: return (void*)fca_mstep_kernel<R, 5>;
    case 6: return (void*)fca_mstep_kernel<R, 6>;
    case 7: return (void*)fca_mstep_kernel<R, 7>;
    case 8: return (void*)fca_mstep_kernel<R, 8>;
  }
  return nullptr;
}

}  // namespace ffca

extern "C" int ffca_fca_mstep(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                              const void* mu, const void* phi, const void* S, int vf_mode, double vf_scalar,
                              const void* vf, void* S_out, void* v_out, int* status) {
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
  FcaMstepArgs a = {};
  a.U = U; a.I = I; a.J = J; a.N = N; a.F = F; a.vf_mode = vf_mode; a.vf_scalar = vf_scalar;
  FFCA_TRY(st.in(mu, size_t(U) * J * N * F * I * cs, &a.mu));
  FFCA_TRY(st.in(phi, size_t(U) * J * N * F * I * I * cs, &a.phi));
  FFCA_TRY(st.in(S, size_t(U) * J * F * I * I * cs, &a.S));
  if (vf_mode == FFCA_VF_BIN) FFCA_TRY(st.in(vf, size_t(nb) * rs, &a.vf));
  if (vf_mode == FFCA_VF_FULL) FFCA_TRY(st.in(vf, size_t(U) * J * N * F * rs, &a.vf));
  FFCA_TRY(st.out(S_out, size_t(U) * J * F * I * I * cs, &a.S_out));
  FFCA_TRY(st.out(v_out, size_t(U) * J * N * F * rs, &a.v_out));
  void* dstatus;
  FFCA_TRY(st.scratch(size_t(nb) * 4, &dstatus));
  FFCA_CK(cudaMemsetAsync(dstatus, 0, size_t(nb) * 4, s));
  a.status = (int*)dstatus;
  void* fn = dtype == FFCA_C64 ? fca_mstep_fn<float>(I) : fca_mstep_fn<double>(I);
  void* args[] = {(void*)&a};
  FFCA_CK(cudaLaunchKernel(fn, dim3(unsigned(nb)), dim3(128), args, 0, s));
  count_launch();
  FFCA_TRY(st.flush());
  return finish_status((const int*)dstatus, status, nb, mem, s, FFCA_ST_NOT_PD);
}

extern "C" int ffca_power_floor(int device, void* stream, int mem, int dtype, int U, int I, int N, int F,
                                const void* y, double* out) {
  reset_launches();
  if (!check_dims(dtype, U, I, 1, N, F)) return FFCA_E_ARG;
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const long long nb = (long long)U * F;
  if (nb == 0) return FFCA_OK;
  Staging st(mem, s);
  const void* dy;
  void* dout;
  FFCA_TRY(st.in(y, size_t(U) * I * N * F * csize(dtype), &dy));
  FFCA_TRY(st.out(out, size_t(nb) * 8, &dout));
  if (dtype == FFCA_C64)
    power_floor_kernel<float><<<unsigned(U * ((F + 31) / 32)), 256, 0, s>>>(dy, (double*)dout, U, I, N, F);
  else
    power_floor_kernel<double><<<unsigned(U * ((F + 31) / 32)), 256, 0, s>>>(dy, (double*)dout, U, I, N, F);
  count_launch();
  FFCA_CK(cudaGetLastError());
  FFCA_TRY(st.flush());
  FFCA_CK(cudaStreamSynchronize(s));
  return FFCA_OK;
}
