// Shared device helpers for the FastFCA-AS / FCA kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdint>

namespace ffca {

namespace cg = cooperative_groups;

constexpr unsigned FULL = 0xffffffffu;

template <typename R> struct Cpx;
template <> struct Cpx<float> { using T = float2; };
template <> struct Cpx<double> { using T = double2; };

// Numeric floors.  fp64 uses the reference constants verbatim
// (fastfca.py:45, fca.py:89); fp32 substitutes representable values
// (1e-300 underflows to 0 in fp32 -- SURVEY.md §0 finding 4).
template <typename R> struct Floors;
template <> struct Floors<double> {
  static constexpr double weight = 1e-300;
  static constexpr double vmin = 1e-300;
};
template <> struct Floors<float> {
  static constexpr float weight = 1e-30f;
  static constexpr float vmin = 1e-30f;
};

// IEEE reciprocal / quotient in the arithmetic type.
__device__ __forceinline__ double rcp(double x) { return 1.0 / x; }
__device__ __forceinline__ float rcp(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double quot(double a, double b) { return a / b; }
__device__ __forceinline__ float quot(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double flog(double x) { return log(x); }
__device__ __forceinline__ float flog(float x) { return logf(x); }

template <typename C2, typename R>
__device__ __forceinline__ C2 mk(R x, R y) {
  C2 z;
  z.x = x;
  z.y = y;
  return z;
}

// conj(p) * y, accumulated into acc
template <typename C2>
__device__ __forceinline__ void cmac_conj(C2& acc, const C2 p, const C2 y) {
  acc.x = fma(p.x, y.x, fma(p.y, y.y, acc.x));
  acc.y = fma(p.x, y.y, fma(-p.y, y.x, acc.y));
}

// Sum over lanes that share (lane mod G); G is a power of two dividing 32.
template <typename T>
__device__ __forceinline__ T warp_sum_seg(T x, int G) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1)
    if (o >= G) x += __shfl_xor_sync(FULL, x, o);
  return x;
}

// ------------------------------------------------------------------------
// Small dense complex LU in fp64, partial pivoting on |re|+|im| (LAPACK's
// izamax criterion).  One thread per system; matrices live in shared memory so
// the solver adds no register pressure to the streaming phases.
// ------------------------------------------------------------------------
__device__ __forceinline__ double cabs1(const double2 z) { return fabs(z.x) + fabs(z.y); }
__device__ __forceinline__ double2 cmul(const double2 a, const double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 crecip(const double2 z) {
  // 1/z = conj(z)/|z|^2 with a scaling step against over/underflow
  double s = fmax(fabs(z.x), fabs(z.y));
  double zr = z.x / s, zi = z.y / s;
  double d = zr * zr + zi * zi;
  return make_double2(zr / (d * s), -zi / (d * s));
}

// In-place LU with partial pivoting of one I x I complex matrix stored
// row-major in shared memory (fp64).  Returns false on an exactly zero pivot
// (LAPACK zgetrf INFO > 0, which is when numpy.linalg.inv raises).
template <int I>
__device__ bool lu_factor(double2* a, int* piv) {
  bool ok = true;
#pragma unroll 1
  for (int k = 0; k < I; ++k) {
    int p = k;
    double best = cabs1(a[k * I + k]);
    for (int r = k + 1; r < I; ++r) {
      const double m = cabs1(a[r * I + k]);
      if (m > best) { best = m; p = r; }
    }
    piv[k] = p;
    if (p != k)
      for (int c = 0; c < I; ++c) {
        const double2 t = a[k * I + c];
        a[k * I + c] = a[p * I + c];
        a[p * I + c] = t;
      }
    const double2 d = a[k * I + k];
    if (d.x == 0.0 && d.y == 0.0) { ok = false; continue; }
    const double2 inv = crecip(d);
    for (int r = k + 1; r < I; ++r) {
      const double2 l = cmul(a[r * I + k], inv);
      a[r * I + k] = l;
      for (int c = k + 1; c < I; ++c) {
        const double2 u = a[k * I + c];
        double2 x = a[r * I + c];
        x.x -= l.x * u.x - l.y * u.y;
        x.y -= l.x * u.y + l.y * u.x;
        a[r * I + c] = x;
      }
    }
  }
  return ok;
}

// Solve A x = b in place (b in shared memory) with the factors from lu_factor.
template <int I>
__device__ void lu_solve(const double2* a, const int* piv, double2* b) {
#pragma unroll 1
  for (int k = 0; k < I; ++k) {
    const int p = piv[k];
    if (p != k) {
      const double2 t = b[k];
      b[k] = b[p];
      b[p] = t;
    }
  }
#pragma unroll 1
  for (int r = 1; r < I; ++r)
    for (int c = 0; c < r; ++c) {
      const double2 l = a[r * I + c];
      b[r].x -= l.x * b[c].x - l.y * b[c].y;
      b[r].y -= l.x * b[c].y + l.y * b[c].x;
    }
#pragma unroll 1
  for (int r = I - 1; r >= 0; --r) {
    for (int c = r + 1; c < I; ++c) {
      const double2 u = a[r * I + c];
      b[r].x -= u.x * b[c].x - u.y * b[c].y;
      b[r].y -= u.x * b[c].y + u.y * b[c].x;
    }
    b[r] = cmul(b[r], crecip(a[r * I + r]));
  }
}

template <int I>
__device__ double lu_logabsdet(const double2* a) {
  double s = 0.0;
  for (int k = 0; k < I; ++k) s += log(hypot(a[k * I + k].x, a[k * I + k].y));
  return s;
}

// Status bits written per bin (mapped to the reference's exceptions on host).
enum : int {
  ST_SINGULAR_P = 1,          // errors.SingularP               (fastfca.py:360-363)
  ST_SINGULAR_B = 2,          // errors.SingularWeightedCovariance (fastfca.py:184-194)
  ST_B_LOADED = 4,            // B_i needed the trace-loading retry (informational)
  ST_NOT_PD = 8,              // errors.NotPositiveDefinite (FCA)  (fca.py:137-140,157-158)
  ST_S_LOADED = 16,           // FCA S needed Cholesky-failure loading (informational)
};

}  // namespace ffca
