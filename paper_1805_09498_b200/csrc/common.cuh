// Shared device helpers for the FastFCA-AS / FCA kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdint>
#include <type_traits>

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

// Reciprocals: hardware approximation (fp32: 1 ulp as is; fp64: refined by
// two Newton steps from MUFU.RCP64H to full double precision).  The
// operands here are floored positive weights / powers, never 0, inf or
// subnormal, so the IEEE special-case paths of 1/x are not needed.
__device__ __forceinline__ double rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  return r;
}
// Per-point reciprocal: fp64 with one Newton step (relative error ~1e-13,
// three orders inside the 1e-10 parity bound); fp32 as rcp().
__device__ __forceinline__ double rcp_pt(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return fma(r, fma(-x, r, 1.0), r);
}
__device__ __forceinline__ float rcp_pt(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp(float x) {
  // MUFU.RCP: max error 1 ulp over the full range -- no Newton step needed for
  // the complex64 path's 1e-4 tolerance (weights are >= 1e-30, never subnormal)
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
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

// Pair arithmetic: fp32 pairs lower to Blackwell's packed FFMA2 (fma.rn.f32x2,
// scalar operands become broadcast operands, swaps become operand swizzles);
// fp64 pairs are two DFMAs.
__device__ __forceinline__ unsigned long long pk64(float2 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 upk64(unsigned long long r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk64(a)), "l"(pk64(b)), "l"(pk64(c)));
  return upk64(r);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk64(a)), "l"(pk64(b)));
  return upk64(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk64(a)), "l"(pk64(b)));
  return upk64(r);
}
__device__ __forceinline__ double2 fma2(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y));
}
template <typename R>
__device__ __forceinline__ typename Cpx<R>::T bc2(R x) {
  typename Cpx<R>::T t;
  t.x = x;
  t.y = x;
  return t;
}

// conj(p) * y, accumulated into acc
template <typename C2>
__device__ __forceinline__ void cmac_conj(C2& acc, const C2 p, const C2 y) {
  acc.x = fma(p.x, y.x, fma(p.y, y.y, acc.x));
  acc.y = fma(p.x, y.y, fma(-p.y, y.x, acc.y));
}

// Dynamic shared memory actually granted to this launch (bytes).
// ---- 1-D bulk copies (TMA engine) global -> shared, completed on an mbarrier ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ unsigned dynamic_smem_bytes() {
  unsigned r;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
  return r;
}

// Asynchronous global -> shared copy of one element (cp.async, LDGSTS);
// `valid == false` zero-fills the destination without reading the source.
// ---- tensor memory (TMEM, sm_100a) used as thread-private storage -------------------------
// 512 columns x 128 lanes x 32 bit per SM.  A CTA allocates a power-of-two number of columns
// (all 128 lanes); warp w of the CTA reaches lanes 32 (w % 4) .. + 31 only, and the 32x32b
// shape gives thread t of the warp N consecutive columns of lane 32 (w % 4) + t: a per-thread
// array that costs neither registers nor shared memory.  Address = (lane << 16) | column.
__device__ __forceinline__ void tmem_alloc(unsigned* smem_dst, unsigned cols) {  // one full warp; cols = 32 .. 512, power of 2
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(smem_dst)), "r"(cols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(unsigned taddr, unsigned cols) {  // one full warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(cols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
// wait::ld that also "touches" the destination registers of the loads it completes, so the
// compiler cannot schedule a use of them before the wait
__device__ __forceinline__ void tmem_wait_ld(float (&a)[8], float (&b)[4]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+f"(a[0]), "+f"(a[1]), "+f"(a[2]), "+f"(a[3]), "+f"(a[4]), "+f"(a[5]), "+f"(a[6]), "+f"(a[7]), "+f"(b[0]),
                 "+f"(b[1]), "+f"(b[2]), "+f"(b[3])
               :
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_ld4(unsigned taddr, float (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]) : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(unsigned taddr, float (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st4(unsigned taddr, const float (&r)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(taddr), "f"(r[0]), "f"(r[1]),
               "f"(r[2]), "f"(r[3]) : "memory");
}
__device__ __forceinline__ void tmem_st8(unsigned taddr, const float (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr), "f"(r[0]),
               "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7]) : "memory");
}

// One thread-private record of W = 12 or 16 words at columns [taddr, taddr + W): load (asynchronous;
// tm_rec_wait makes r valid -- it names r so no use of it can be scheduled before the wait) / store.
template <int W>
__device__ __forceinline__ void tm_rec_ld(unsigned taddr, float (&r)[W]) {
  static_assert(W == 12 || W == 16, "records of 12 or 16 words");
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
               : "r"(taddr));
  if constexpr (W == 12)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                 : "=f"(r[8]), "=f"(r[9]), "=f"(r[10]), "=f"(r[11]) : "r"(taddr + 8));
  else
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=f"(r[8]), "=f"(r[9]), "=f"(r[10]), "=f"(r[11]), "=f"(r[12]), "=f"(r[13]), "=f"(r[14]), "=f"(r[15])
                 : "r"(taddr + 8));
}
template <int W>
__device__ __forceinline__ void tm_rec_wait(float (&r)[W]) {
  if constexpr (W == 12)
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : "+f"(r[0]), "+f"(r[1]), "+f"(r[2]), "+f"(r[3]), "+f"(r[4]), "+f"(r[5]), "+f"(r[6]), "+f"(r[7]),
                   "+f"(r[8]), "+f"(r[9]), "+f"(r[10]), "+f"(r[11])
                 :
                 : "memory");
  else
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : "+f"(r[0]), "+f"(r[1]), "+f"(r[2]), "+f"(r[3]), "+f"(r[4]), "+f"(r[5]), "+f"(r[6]), "+f"(r[7]),
                   "+f"(r[8]), "+f"(r[9]), "+f"(r[10]), "+f"(r[11]), "+f"(r[12]), "+f"(r[13]), "+f"(r[14]), "+f"(r[15])
                 :
                 : "memory");
}
template <int W>
__device__ __forceinline__ void tm_rec_st(unsigned taddr, const float (&r)[W]) {
  static_assert(W == 12 || W == 16, "records of 12 or 16 words");
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr), "f"(r[0]),
               "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7]) : "memory");
  if constexpr (W == 12)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(taddr + 8), "f"(r[8]), "f"(r[9]),
                 "f"(r[10]), "f"(r[11]) : "memory");
  else
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr + 8), "f"(r[8]),
                 "f"(r[9]), "f"(r[10]), "f"(r[11]), "f"(r[12]), "f"(r[13]), "f"(r[14]), "f"(r[15]) : "memory");
}

template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem_dst, const void* gsrc, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  const int n = valid ? BYTES : 0;
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc), "r"(n));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(d), "l"(gsrc), "n"(BYTES), "r"(n));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
// L1 prefetch of the line holding a global address (no register result)
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

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
__device__ __forceinline__ double2 cadd(const double2 a, const double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(const double2 a, const double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 crecip(const double2 z) {
  // 1/z = conj(z) / |z|^2; rescale by an exact power of two outside
  // [2^-500, 2^500] so |z|^2 neither overflows nor underflows.
  const double m = fmax(fabs(z.x), fabs(z.y));
  if (m > 0x1p-500 && m < 0x1p500) {
    const double r = rcp(z.x * z.x + z.y * z.y);
    return make_double2(z.x * r, -z.y * r);
  }
  const int e = ilogb(m);
  const double zr = scalbn(z.x, -e), zi = scalbn(z.y, -e);
  const double r = 1.0 / (zr * zr + zi * zi);
  return make_double2(scalbn(zr * r, -e), scalbn(-zi * r, -e));
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

// ------------------------------------------------------------------------
// Register-resident LDL^H of the Hermitian weighted covariance B_i (fully
// unrolled; static indexing only, so the factors stay in registers for
// I <= 4).  Reports an exactly zero pivot, when numpy.linalg.inv raises.
// ------------------------------------------------------------------------
template <int I>
struct SmallLDL {
  double2 l[I][I];  // strictly lower part used
  double rd[I];     // 1 / d_k
  bool ok;

  // B given as its lower triangle (diag real).  B = L D L^H.
  __device__ __forceinline__ void factor(double2 (&b)[I][I]) {
    ok = true;
    double d[I];
#pragma unroll
    for (int k = 0; k < I; ++k) {
      double dk = b[k][k].x;
#pragma unroll
      for (int c = 0; c < k; ++c) dk -= (l[k][c].x * l[k][c].x + l[k][c].y * l[k][c].y) * d[c];
      d[k] = dk;
      if (dk == 0.0) ok = false;
      rd[k] = (dk != 0.0) ? rcp(dk) : 0.0;
#pragma unroll
      for (int r = k + 1; r < I; ++r) {
        double2 acc = b[r][k];
#pragma unroll
        for (int c = 0; c < k; ++c) {  // acc -= l[r][c] d_c conj(l[k][c])
          const double2 lr = l[r][c], lk = l[k][c];
          acc.x -= (lr.x * lk.x + lr.y * lk.y) * d[c];
          acc.y -= (lr.y * lk.x - lr.x * lk.y) * d[c];
        }
        l[r][k] = make_double2(acc.x * rd[k], acc.y * rd[k]);
      }
    }
  }

  __device__ __forceinline__ void solve(double2 (&x)[I]) const {
#pragma unroll
    for (int r = 1; r < I; ++r)
#pragma unroll
      for (int c = 0; c < r; ++c) {
        const double2 lv = l[r][c];
        x[r].x -= lv.x * x[c].x - lv.y * x[c].y;
        x[r].y -= lv.x * x[c].y + lv.y * x[c].x;
      }
#pragma unroll
    for (int r = 0; r < I; ++r) x[r] = make_double2(x[r].x * rd[r], x[r].y * rd[r]);
#pragma unroll
    for (int r = I - 1; r >= 0; --r)
#pragma unroll
      for (int c = r + 1; c < I; ++c) {  // (L^H)_{r,c} = conj(l[c][r])
        const double2 lv = l[c][r];
        x[r].x -= lv.x * x[c].x + lv.y * x[c].y;
        x[r].y -= lv.x * x[c].y - lv.y * x[c].x;
      }
  }
};

// Hermitian I x I (I <= 3) inverse applied through the adjugate: B^-1 = adj(B) / det(B).  Same
// interface as SmallLDL (factor: B's lower triangle, diagonal real; ok = det(B) != 0, the exact
// singularity the reference's LU inverse rejects; solve: x <- B^-1 x).  Every cofactor is an
// independent 2 x 2 determinant, so the dependency chain is a few operations deep instead of the
// factorisation's pivot-by-pivot chain (the solve is on every iteration's critical path).
template <int I>
struct HermAdj {
  static_assert(I >= 1 && I <= 3, "adjugate solve for I <= 3");
  double a[I];        // real diagonal of adj(B)
  double2 c[I][I];    // lower triangle of adj(B) (c[r][q], q < r); upper = conj
  double rdet;        // 1 / det(B)
  bool ok;

  __device__ __forceinline__ void factor(const double2 (&b)[I][I]) {
    double det;
    if constexpr (I == 1) {
      a[0] = 1.0;
      det = b[0][0].x;
    } else if constexpr (I == 2) {
      a[0] = b[1][1].x;
      a[1] = b[0][0].x;
      c[1][0] = make_double2(-b[1][0].x, -b[1][0].y);
      det = b[0][0].x * b[1][1].x - (b[1][0].x * b[1][0].x + b[1][0].y * b[1][0].y);
    } else {
      const double b00 = b[0][0].x, b11 = b[1][1].x, b22 = b[2][2].x;
      const double2 b10 = b[1][0], b20 = b[2][0], b21 = b[2][1];
      a[0] = b11 * b22 - (b21.x * b21.x + b21.y * b21.y);
      a[1] = b00 * b22 - (b20.x * b20.x + b20.y * b20.y);
      a[2] = b00 * b11 - (b10.x * b10.x + b10.y * b10.y);
      // (B^-1)_10 ~ -(b10 b22 - conj(b21) b20)
      c[1][0] = make_double2(-(b10.x * b22 - (b21.x * b20.x + b21.y * b20.y)),
                             -(b10.y * b22 - (b21.x * b20.y - b21.y * b20.x)));
      // (B^-1)_20 ~ b10 b21 - b11 b20
      c[2][0] = make_double2(b10.x * b21.x - b10.y * b21.y - b11 * b20.x, b10.x * b21.y + b10.y * b21.x - b11 * b20.y);
      // (B^-1)_21 ~ -(b00 b21 - conj(b10) b20)
      c[2][1] = make_double2(-(b00 * b21.x - (b10.x * b20.x + b10.y * b20.y)),
                             -(b00 * b21.y - (b10.x * b20.y - b10.y * b20.x)));
      // det = b00 a0 + 2 Re(conj(b10) c10 ... ) written via the first column of adj
      det = b00 * a[0] + (b10.x * c[1][0].x + b10.y * c[1][0].y) + (b20.x * c[2][0].x + b20.y * c[2][0].y);
    }
    ok = det != 0.0;
    rdet = ok ? rcp(det) : 0.0;
  }

  __device__ __forceinline__ void solve(double2 (&x)[I]) const {
    double2 y[I];
#pragma unroll
    for (int r = 0; r < I; ++r) {
      double2 acc = make_double2(a[r] * x[r].x, a[r] * x[r].y);
#pragma unroll
      for (int q = 0; q < I; ++q) {
        if (q == r) continue;
        // adj[r][q] = c[r][q] (q < r) or conj(c[q][r]) (q > r)
        const double2 m = q < r ? c[r][q] : make_double2(c[q][r].x, -c[q][r].y);
        acc.x += m.x * x[q].x - m.y * x[q].y;
        acc.y += m.x * x[q].y + m.y * x[q].x;
      }
      y[r] = acc;
    }
#pragma unroll
    for (int r = 0; r < I; ++r) x[r] = make_double2(y[r].x * rdet, y[r].y * rdet);
  }
};

// L D L^H of a Hermitian positive definite matrix held by one thread as its packed lower
// triangle (row-major, b[r(r+1)/2 + c], c <= r) -- half the registers of SmallLDL's square
// arrays, for I up to 8.  In place: b[(r,c)] becomes l_rc (c < r) and b[(k,k)] = (1/d_k, d_k).
// The failure criterion is SmallLDL's (an exactly zero d_k).
template <int I>
struct PackedLDL {
  static constexpr int NP = I * (I + 1) / 2;
  __host__ __device__ static constexpr int id(int r, int c) { return r * (r + 1) / 2 + c; }
  __device__ __forceinline__ static bool factor(double2 (&b)[NP]) {
    bool ok = true;
#pragma unroll
    for (int k = 0; k < I; ++k) {
      double dk = b[id(k, k)].x;
#pragma unroll
      for (int c = 0; c < k; ++c) {
        const double2 l = b[id(k, c)];
        dk -= (l.x * l.x + l.y * l.y) * b[id(c, c)].y;
      }
      if (dk == 0.0) ok = false;
      const double rk = (dk != 0.0) ? rcp(dk) : 0.0;
      b[id(k, k)] = make_double2(rk, dk);
#pragma unroll
      for (int r = k + 1; r < I; ++r) {
        double2 acc = b[id(r, k)];
#pragma unroll
        for (int c = 0; c < k; ++c) {  // acc -= l_rc d_c conj(l_kc)
          const double2 lr = b[id(r, c)], lk = b[id(k, c)];
          const double dc = b[id(c, c)].y;
          acc.x -= (lr.x * lk.x + lr.y * lk.y) * dc;
          acc.y -= (lr.y * lk.x - lr.x * lk.y) * dc;
        }
        b[id(r, k)] = make_double2(acc.x * rk, acc.y * rk);
      }
    }
    return ok;
  }
  // x <- (L D L^H)^-1 x with the factor in (shared) memory
  __device__ __forceinline__ static void solve(const double2* L, double2 (&x)[I]) {
#pragma unroll
    for (int r = 1; r < I; ++r)
#pragma unroll
      for (int c = 0; c < r; ++c) {
        const double2 lv = L[id(r, c)];
        x[r].x -= lv.x * x[c].x - lv.y * x[c].y;
        x[r].y -= lv.x * x[c].y + lv.y * x[c].x;
      }
#pragma unroll
    for (int r = 0; r < I; ++r) {
      const double rd = L[id(r, r)].x;
      x[r] = make_double2(x[r].x * rd, x[r].y * rd);
    }
#pragma unroll
    for (int r = I - 1; r >= 0; --r)
#pragma unroll
      for (int c = r + 1; c < I; ++c) {  // (L^H)_{r,c} = conj(l_cr)
        const double2 lv = L[id(c, r)];
        x[r].x -= lv.x * x[c].x + lv.y * x[c].y;
        x[r].y -= lv.x * x[c].y - lv.y * x[c].x;
      }
  }
};

// ------------------------------------------------------------------------
// Gauss-Jordan elimination with partial pivoting on [A | E] by a group of 8
// consecutive lanes; lane r < I owns row r (fp64, registers).  The pivot at
// step k is the remaining row with the largest |re|+|im| in column k (lowest
// lane on ties) -- the same pivot sequence as LAPACK's LU with partial
// pivoting, so "exactly zero pivot" means what numpy.linalg.inv reports as
// singular.  Rows are not swapped: on return lane r holds row `k_of_row` of
// A^-1 E.  `srow` is 2*I double2 of shared scratch for this group.
// ------------------------------------------------------------------------
// Reciprocal of a complex number via rcp.approx + Newton (no IEEE division).
__device__ __forceinline__ double2 crecip_fast(const double2 z) {
  const double m = fmax(fabs(z.x), fabs(z.y));
  if (m > 0x1p-500 && m < 0x1p500) {
    const double r = rcp(z.x * z.x + z.y * z.y);
    return make_double2(z.x * r, -z.y * r);
  }
  return crecip(z);
}

// The step loop stays rolled (instruction-cache footprint); column k of the lane's row is picked
// with selects so a[] / e[] stay in registers.
template <int I, bool LOGDET>
__device__ __forceinline__ bool gj_group(double2 (&a)[I], double2 (&e)[I], int r, unsigned gmask, double2* srow,
                                         int& k_of_row, double& logabsdet) {
  bool used = r >= I;
  bool ok = true;
  logabsdet = 0.0;
  k_of_row = -1;
#pragma unroll 1
  for (int k = 0; k < I; ++k) {
    double2 ak = a[0];
#pragma unroll
    for (int c = 1; c < I; ++c)
      if (c == k) ak = a[c];
    // max of |re|+|im| over the unused rows, lowest lane on ties, as three group-wide integer
    // reductions on the (non-negative) double's bit pattern: high word (+1, so an unused row
    // with an exactly zero entry still beats the used rows' 0), then low word, then lane
    const double best = cabs1(ak);
    const unsigned hi = used ? 0u : unsigned(__double2hiint(best)) + 1u;
    const unsigned lo = unsigned(__double2loint(best));
    const unsigned mh = __reduce_max_sync(gmask, hi);
    const unsigned ml = __reduce_max_sync(gmask, hi == mh ? lo : 0u);
    const int who = int(__reduce_min_sync(gmask, (hi == mh && lo == ml) ? unsigned(r) : 8u));
    if (mh <= 1u && ml == 0u) ok = false;  // exactly zero (or no) pivot
    const bool piv = (who == r);
    if (piv) {
#pragma unroll
      for (int c = 0; c < I; ++c) {
        srow[c] = a[c];
        srow[I + c] = e[c];
      }
    }
    __syncwarp(gmask);
    // every lane reads the unscaled pivot row and forms the same reciprocal; the pivot lane
    // scales its row, the others subtract (a_k / pivot) times it -- one uniform update
    const double2 d = srow[k];
    const double2 inv = crecip_fast(d);
    if (LOGDET && piv) logabsdet += log(hypot(d.x, d.y));
    const double2 f = cmul(ak, inv);
    const double2 coef = piv ? inv : make_double2(-f.x, -f.y);
#pragma unroll
    for (int c = 0; c < I; ++c) {
      const double2 ta = cmul(coef, srow[c]), te = cmul(coef, srow[I + c]);
      a[c] = piv ? ta : make_double2(a[c].x + ta.x, a[c].y + ta.y);
      e[c] = piv ? te : make_double2(e[c].x + te.x, e[c].y + te.y);
    }
    if (piv) {
      used = true;
      k_of_row = k;
    }
    __syncwarp(gmask);
  }
  // the pivot lanes' log|pivot| terms sum to log|det A|
  if (LOGDET)
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) logabsdet += __shfl_xor_sync(gmask, logabsdet, o);
  return ok;
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
