// Bin-resident conventional FCA EM (fca.run_fca, fca.py:187-215) on sm_100a.
//
// Same residency scheme as the FastFCA-AS loop (ffca_loop.cuh): a CTA (or a
// cluster) owns one bin for the whole run with y and v in shared memory.  One
// pass over the frames per iteration does the full-matrix E-step and the v
// update; a per-bin fixed-order reduction then gives S' and its inverse.
//
// Per point (n, f), with R_j = v_j S_j and M = sum_j R_j (fca.py:119-144):
//   M = L D L^H (registers), z = M^-1 y
//   mu_j  = R_j z                       (= gain_j y)
//   Y_j   = L^-1 R_j,  R_j M^-1 R_j = Y_j^H D^-1 Y_j
//   Phi_j = R_j - R_j M^-1 R_j          (lower triangle = hermitize)
//   T_j   = mu_j mu_j^H + Phi_j
//   v'_j  = max(Re tr(S_j^-1 T_j) / I, floor)     (fca.py:176-179, old S)
//   acc_j += T_j / v'_j                           (fca.py:181-183)
// Hermitian matrices are kept as packed lower triangles: per row a the
// diagonal (real) then (a, b<a) as complex.
#pragma once

#include "ffca_loop.cuh"

namespace ffca {



__host__ __device__ constexpr int herm_reals(int I) { return I * I; }

struct FcaSmem {
  size_t y, v0, v1, vf, S, Sd, Si, wpart, cpart, tot, vfl, total, slab;
  FcaSmem() = default;
  __host__ __device__ FcaSmem(int I, int J, int NL, int W, int rsz, int vf_mode, int VMAX) {
    size_t o = 0;
    const size_t csz = 2 * size_t(rsz);
    y = o;  o += align16(size_t(NL) * odd_up(I) * csz);
    v0 = o; o += align16(size_t(NL) * odd_up(J) * rsz);
    v1 = o; o += align16(size_t(NL) * odd_up(J) * rsz);
    vf = o; o += vf_mode == 2 ? align16(size_t(NL) * odd_up(J) * rsz) : 0;
    slab = o;
    S = o;  o += align16(size_t(J) * I * I * rsz);   // packed lower, compute type
    Sd = o; o += align16(size_t(J) * I * I * 8);     // packed lower, fp64 master
    Si = o; o += align16(size_t(J) * I * I * rsz);   // packed lower of S^-1, compute type
    wpart = o; o += align16(size_t(W) * VMAX * 8);
    cpart = o; o += align16(size_t(2) * VMAX * 8);
    tot = o;   o += align16(size_t(VMAX) * 8);
    vfl = o;   o += 16;
    total = o;
  }
};

struct FcaArgs {
  int U, I, J, N, F;
  long long total_bins;
  int C, NL;
  int iters;
  int vf_mode;  // 0 scalar, 1 per-bin, 2 full, 3 auto
  double vf_scalar;
  const void* vf;
  const void* y;   // (U,I,N,F)
  const void* S0;  // (U,J,F,I,I)
  const void* v0;  // (U,J,N,F)
  void* S_out;
  void* v_out;
  void* S_prev;    // optional: S of the last E-step
  void* v_prev;    // optional: v of the last E-step
  double* ll;      // optional (total_bins, 1 + iters)
  int* status;
  FcaSmem L;  // shared-memory carve-up from the host (read from the kernel parameters)
};

// Packed-lower index helpers: row a starts at a*a; diag first, then (a,b<a) pairs.
__host__ __device__ constexpr int pk_diag(int a) { return a * a; }
__host__ __device__ constexpr int pk_re(int a, int b) { return a * a + 1 + 2 * b; }

// LDL^H of a packed-lower Hermitian matrix in fp64 with one relative trace
// loading retry on a non-positive pivot (fca._invert_spatial, fca.py:147-158),
// then the packed lower triangle of the inverse.  Returns status bits.
template <int I>
__device__ int fca_inverse_spatial(const double* Sp, double* out) {
  double2 B[I][I];
  double tr = 0.0;
  for (int a = 0; a < I; ++a) {
    B[a][a] = make_double2(Sp[pk_diag(a)], 0.0);
    tr += Sp[pk_diag(a)];
    for (int b = 0; b < a; ++b) B[a][b] = make_double2(Sp[pk_re(a, b)], Sp[pk_re(a, b) + 1]);
  }
  int st = 0;
  SmallLDL<I> ldl;
  ldl.factor(B);
  bool pd = ldl.ok;
  for (int k = 0; k < I; ++k) pd = pd && (ldl.rd[k] > 0.0);
  if (!pd) {
    st |= ST_S_LOADED;
    for (int a = 0; a < I; ++a) B[a][a].x += 1e-10 * tr / I;
    ldl.factor(B);
    if (!ldl.ok) return st | ST_NOT_PD;
  }
  // columns of the inverse: solve with e_c, keep a >= c
  for (int c = 0; c < I; ++c) {
    double2 x[I];
    for (int a = 0; a < I; ++a) x[a] = make_double2(a == c ? 1.0 : 0.0, 0.0);
    ldl.solve(x);
    for (int a = c; a < I; ++a) {
      if (a == c) out[pk_diag(a)] = x[a].x;
      else {
        out[pk_re(a, c)] = x[a].x;
        out[pk_re(a, c) + 1] = x[a].y;
      }
    }
  }
  return st;
}

template <typename R, int I, int JM>
struct FcaPoint {
  using C2 = typename Cpx<R>::T;
  static constexpr int RS = odd_up(I);
  static constexpr int H = herm_reals(I);
  static constexpr int V = JM * H + 1;

  const C2* ys;
  const R* vin;
  R* vout;
  const R* vfs;
  const R* S;   // packed lower per source
  const R* Si;  // packed lower of S^-1 per source
  int J, JS, rec0, rstep, npts;
  R invI;

  template <bool REC, bool VF2>
  __device__ __forceinline__ int run(R (&acc)[V], R vfl_b, R* vprev) const {
    int bad = 0;
    const C2* yp = ys + rec0 * RS;
    const R* vp = vin + rec0 * JS;
    R* wp = vout + rec0 * JS;
    const R* fp = vfs + rec0 * JS;
#pragma unroll 1
    for (int k = 0; k < npts; ++k, yp += rstep * RS, vp += rstep * JS, wp += rstep * JS, fp += rstep * JS) {
      C2 yv[I];
      R vj[JM];
#pragma unroll
      for (int i = 0; i < I; ++i) yv[i] = yp[i];
#pragma unroll
      for (int j = 0; j < JM; ++j) vj[j] = (j < J) ? vp[j] : R(0);
      (void)vprev;
      // mixture covariance (lower) and its LDL^H
      C2 L[I][I];
      R d[I], rd[I];
#pragma unroll
      for (int a = 0; a < I; ++a) {
#pragma unroll
        for (int b = 0; b <= a; ++b) {
          C2 m = mk<C2, R>(R(0), R(0));
#pragma unroll
          for (int j = 0; j < JM; ++j) {
            if (j < J) {
              if (a == b) m.x = fma(vj[j], S[j * H + pk_diag(a)], m.x);
              else {
                m.x = fma(vj[j], S[j * H + pk_re(a, b)], m.x);
                m.y = fma(vj[j], S[j * H + pk_re(a, b) + 1], m.y);
              }
            }
          }
          L[a][b] = m;
        }
      }
#pragma unroll
      for (int kk = 0; kk < I; ++kk) {
        R dk = L[kk][kk].x;
#pragma unroll
        for (int c = 0; c < kk; ++c) dk -= (L[kk][c].x * L[kk][c].x + L[kk][c].y * L[kk][c].y) * d[c];
        d[kk] = dk;
        if (dk == R(0)) bad = 1;
        rd[kk] = rcp(dk);
#pragma unroll
        for (int r = kk + 1; r < I; ++r) {
          C2 acc2 = L[r][kk];
#pragma unroll
          for (int c = 0; c < kk; ++c) {
            const C2 lr = L[r][c], lk = L[kk][c];
            acc2.x -= (lr.x * lk.x + lr.y * lk.y) * d[c];
            acc2.y -= (lr.y * lk.x - lr.x * lk.y) * d[c];
          }
          L[r][kk] = mk<C2, R>(acc2.x * rd[kk], acc2.y * rd[kk]);
        }
      }
      // z = M^-1 y
      C2 z[I];
#pragma unroll
      for (int r = 0; r < I; ++r) {
        C2 t = yv[r];
#pragma unroll
        for (int c = 0; c < r; ++c) {
          t.x -= L[r][c].x * z[c].x - L[r][c].y * z[c].y;
          t.y -= L[r][c].x * z[c].y + L[r][c].y * z[c].x;
        }
        z[r] = t;
      }
#pragma unroll
      for (int r = 0; r < I; ++r) z[r] = mk<C2, R>(z[r].x * rd[r], z[r].y * rd[r]);
#pragma unroll
      for (int r = I - 1; r >= 0; --r)
#pragma unroll
        for (int c = r + 1; c < I; ++c) {
          const C2 lv = L[c][r];  // conj
          z[r].x -= lv.x * z[c].x + lv.y * z[c].y;
          z[r].y -= lv.x * z[c].y - lv.y * z[c].x;
        }
      if constexpr (REC) {
        // ln det M + y^H M^-1 y (fca.py:108-116)
        R l = R(0);
#pragma unroll
        for (int r = 0; r < I; ++r) l += flog(d[r]) + (yv[r].x * z[r].x + yv[r].y * z[r].y);
        acc[V - 1] += l;
      }
#pragma unroll
      for (int j = 0; j < JM; ++j) {
        if (j >= J) continue;
        const R vjj = vj[j];
        // full R_j from the packed lower triangle
        C2 Rm[I][I];
#pragma unroll
        for (int a = 0; a < I; ++a) {
          Rm[a][a] = mk<C2, R>(vjj * S[j * H + pk_diag(a)], R(0));
#pragma unroll
          for (int b = 0; b < a; ++b) {
            const R re = vjj * S[j * H + pk_re(a, b)], im = vjj * S[j * H + pk_re(a, b) + 1];
            Rm[a][b] = mk<C2, R>(re, im);
            Rm[b][a] = mk<C2, R>(re, -im);
          }
        }
        // mu = R z
        C2 mu[I];
#pragma unroll
        for (int a = 0; a < I; ++a) {
          C2 t = mk<C2, R>(R(0), R(0));
#pragma unroll
          for (int c = 0; c < I; ++c) {
            t.x = fma(Rm[a][c].x, z[c].x, fma(-Rm[a][c].y, z[c].y, t.x));
            t.y = fma(Rm[a][c].x, z[c].y, fma(Rm[a][c].y, z[c].x, t.y));
          }
          mu[a] = t;
        }
        // Y = L^-1 R (forward substitution per column)
        C2 Y[I][I];
#pragma unroll
        for (int b = 0; b < I; ++b)
#pragma unroll
          for (int r = 0; r < I; ++r) {
            C2 t = Rm[r][b];
#pragma unroll
            for (int c = 0; c < r; ++c) {
              t.x -= L[r][c].x * Y[c][b].x - L[r][c].y * Y[c][b].y;
              t.y -= L[r][c].x * Y[c][b].y + L[r][c].y * Y[c][b].x;
            }
            Y[r][b] = t;
          }
        // T lower = mu mu^H + R - Y^H D^-1 Y ; trace with S^-1 ; accumulate
        R Tl[H];
#pragma unroll
        for (int a = 0; a < I; ++a)
#pragma unroll
          for (int b = 0; b <= a; ++b) {
            R re = R(0), im = R(0);
#pragma unroll
            for (int kk = 0; kk < I; ++kk) {  // conj(Y[kk][a]) rd_kk Y[kk][b]
              const C2 p = Y[kk][a], q = Y[kk][b];
              re = fma((p.x * q.x + p.y * q.y), rd[kk], re);
              im = fma((p.x * q.y - p.y * q.x), rd[kk], im);
            }
            const R tre = mu[a].x * mu[b].x + mu[a].y * mu[b].y + Rm[a][b].x - re;
            const R tim = mu[a].y * mu[b].x - mu[a].x * mu[b].y + Rm[a][b].y - im;
            if (a == b) Tl[pk_diag(a)] = tre;
            else {
              Tl[pk_re(a, b)] = tre;
              Tl[pk_re(a, b) + 1] = tim;
            }
          }
        R tr = R(0);
#pragma unroll
        for (int a = 0; a < I; ++a) {
          tr = fma(Si[j * H + pk_diag(a)], Tl[pk_diag(a)], tr);
#pragma unroll
          for (int b = 0; b < a; ++b)  // 2 Re(Si_ab conj(T_ab))
            tr = fma(R(2), Si[j * H + pk_re(a, b)] * Tl[pk_re(a, b)] + Si[j * H + pk_re(a, b) + 1] * Tl[pk_re(a, b) + 1], tr);
        }
        R fl = vfl_b;
        if constexpr (VF2) fl = fp[j];
        const R vn = fmax(tr * invI, fl);
        wp[j] = vn;
        const R iv = rcp(vn);
#pragma unroll
        for (int e = 0; e < H; ++e) acc[j * H + e] = fma(Tl[e], iv, acc[j * H + e]);
      }
    }
    return bad;
  }

  // log-likelihood partial at (S, v) without updating (final evaluation)
  __device__ __forceinline__ int loglik(R (&acc)[1]) const {
    int bad = 0;
    const C2* yp = ys + rec0 * RS;
    const R* vp = vin + rec0 * JS;
#pragma unroll 1
    for (int k = 0; k < npts; ++k, yp += rstep * RS, vp += rstep * JS) {
      C2 yv[I];
      R vj[JM];
#pragma unroll
      for (int i = 0; i < I; ++i) yv[i] = yp[i];
#pragma unroll
      for (int j = 0; j < JM; ++j) vj[j] = (j < J) ? vp[j] : R(0);
      C2 L[I][I];
      R d[I], rd[I];
#pragma unroll
      for (int a = 0; a < I; ++a)
#pragma unroll
        for (int b = 0; b <= a; ++b) {
          C2 m = mk<C2, R>(R(0), R(0));
#pragma unroll
          for (int j = 0; j < JM; ++j) {
            if (j < J) {
              if (a == b) m.x = fma(vj[j], S[j * H + pk_diag(a)], m.x);
              else {
                m.x = fma(vj[j], S[j * H + pk_re(a, b)], m.x);
                m.y = fma(vj[j], S[j * H + pk_re(a, b) + 1], m.y);
              }
            }
          }
          L[a][b] = m;
        }
#pragma unroll
      for (int kk = 0; kk < I; ++kk) {
        R dk = L[kk][kk].x;
#pragma unroll
        for (int c = 0; c < kk; ++c) dk -= (L[kk][c].x * L[kk][c].x + L[kk][c].y * L[kk][c].y) * d[c];
        d[kk] = dk;
        if (dk == R(0)) bad = 1;
        rd[kk] = rcp(dk);
#pragma unroll
        for (int r = kk + 1; r < I; ++r) {
          C2 acc2 = L[r][kk];
#pragma unroll
          for (int c = 0; c < kk; ++c) {
            const C2 lr = L[r][c], lk = L[kk][c];
            acc2.x -= (lr.x * lk.x + lr.y * lk.y) * d[c];
            acc2.y -= (lr.y * lk.x - lr.x * lk.y) * d[c];
          }
          L[r][kk] = mk<C2, R>(acc2.x * rd[kk], acc2.y * rd[kk]);
        }
      }
      // y^H M^-1 y = sum_k |(L^-1 y)_k|^2 / d_k
      C2 t[I];
      R l = R(0);
#pragma unroll
      for (int r = 0; r < I; ++r) {
        C2 s = yv[r];
#pragma unroll
        for (int c = 0; c < r; ++c) {
          s.x -= L[r][c].x * t[c].x - L[r][c].y * t[c].y;
          s.y -= L[r][c].x * t[c].y + L[r][c].y * t[c].x;
        }
        t[r] = s;
        l += flog(d[r]) + (s.x * s.x + s.y * s.y) * rd[r];
      }
      acc[0] += l;
    }
    return bad;
  }
};

template <typename R, int I, int JT>
__global__ void __launch_bounds__(256) fca_loop_kernel(const FcaArgs a) {
  using C2 = typename Cpx<R>::T;
  constexpr int JM = JT > 0 ? JT : 4;  // runtime J <= 4 for the generic instantiations
  constexpr int H = herm_reals(I);
  constexpr int RS = odd_up(I);
  constexpr int V = JM * H + 1;
  constexpr int VMAX = V;
  const int J = JT > 0 ? JT : a.J;
  const int JS = odd_up(J);
  const int C = a.C;
  const int tid = threadIdx.x;
  extern __shared__ __align__(16) unsigned char smem[];
  const int W = blockDim.x >> 5;
  const FcaSmem& L = a.L;
  if (L.total > dynamic_smem_bytes()) __trap();
  int crank = 0;
  if (C > 1) crank = int(cg::this_cluster().block_rank());
  int parity = 0;
  const long long bin = blockIdx.x / C;
  const int N = a.N, F = a.F, NL = a.NL;
  const int n0 = int((long long)crank * N / C);
  const int n1 = int((long long)(crank + 1) * N / C);
  const int NLr = n1 - n0;
  const long long u = bin / F;
  const int f = int(bin % F);

  C2* ys = (C2*)(smem + L.y);
  R* vb[2] = {(R*)(smem + L.v0), (R*)(smem + L.v1)};
  R* vfs = (R*)(smem + L.vf);
  R* Sc = (R*)(smem + L.S);
  double* Sd = (double*)(smem + L.Sd);
  R* Sic = (R*)(smem + L.Si);
  double* wpart = (double*)(smem + L.wpart);
  double* cpart = (double*)(smem + L.cpart);
  double* tot = (double*)(smem + L.tot);
  double* vfl = (double*)(smem + L.vfl);
  __shared__ int sflag;

  // ---------------- load ----------------
  R psum = R(0);
  const C2* yg = (const C2*)a.y;
  for (int e = tid; e < I * NL; e += blockDim.x) {
    const int n = e % NL, i = e / NL;
    C2 val = mk<C2, R>(R(0), R(0));
    if (n < NLr) {
      val = yg[((u * I + i) * (long long)N + n0 + n) * F + f];
      psum += val.x * val.x + val.y * val.y;
    }
    ys[n * RS + i] = val;
  }
  for (int e = tid; e < J * NL; e += blockDim.x) {
    const int n = e % NL, j = e / NL;
    R val = R(0);
    if (n < NLr) val = ((const R*)a.v0)[((u * J + j) * (long long)N + n0 + n) * F + f];
    vb[0][n * JS + j] = val;
  }
  if (a.vf_mode == 2)
    for (int e = tid; e < J * NL; e += blockDim.x) {
      const int n = e % NL, j = e / NL;
      R val = R(0);
      if (n < NLr) val = ((const R*)a.vf)[((u * J + j) * (long long)N + n0 + n) * F + f];
      vfs[n * JS + j] = val;
    }
  for (int t = tid; t < J * H; t += blockDim.x) {
    const int j = t / H, e = t % H;
    int ra = 0;
    while ((ra + 1) * (ra + 1) <= e) ++ra;
    const int off = e - ra * ra;
    const C2 s = ((const C2*)a.S0)[(((u * J + j) * F + f) * I + ra) * I + (off == 0 ? ra : (off - 1) / 2)];
    const double val = off == 0 ? double(s.x) : ((off - 1) % 2 == 0 ? double(s.x) : double(s.y));
    Sd[t] = val;
    Sc[t] = R(val);
  }
  if (tid == 0) sflag = 0;
  __syncthreads();
  if (a.vf_mode == 3) {
    const R pv[1] = {psum};
    bin_reduce<R, 1, 1>(pv, wpart, cpart, tot, C, VMAX, parity);
    if (tid == 0) vfl[0] = fmax(1e-10 * tot[0] / (double(I) * N), double(Floors<R>::vmin));
  } else if (tid == 0) {
    vfl[0] = a.vf_mode == 1 ? double(((const R*)a.vf)[bin]) : a.vf_scalar;
  }
  // S^-1 of the initial S (one thread per source)
  auto invert_all = [&]() {
    for (int j = tid; j < J; j += blockDim.x) {
      double out[H];
      const int st = fca_inverse_spatial<I>(Sd + j * H, out);
      for (int e = 0; e < H; ++e) Sic[j * H + e] = R(out[e]);
      if (st && crank == 0) atomicOr(&a.status[bin], st);
    }
  };
  invert_all();
  __syncthreads();

  FcaPoint<R, I, JM> pw;
  pw.ys = ys; pw.vfs = vfs; pw.S = Sc; pw.Si = Sic;
  pw.J = J; pw.JS = JS; pw.rec0 = tid; pw.rstep = blockDim.x;
  pw.npts = NLr > tid ? (NLr - tid + blockDim.x - 1) / blockDim.x : 0;
  pw.invI = R(1) / R(I);
  const bool rec = a.ll != nullptr;
  const int nev = 1 + a.iters;

  for (int it = 0; it < a.iters; ++it) {
    pw.vin = vb[it & 1];
    pw.vout = vb[(it + 1) & 1];
    if (it == a.iters - 1) {
      // parameters of the last E-step (fca.py:211)
      if (a.v_prev)
        for (int e = tid; e < J * NL; e += blockDim.x) {
          const int n = e % NL, j = e / NL;
          if (n < NLr) ((R*)a.v_prev)[((u * J + j) * (long long)N + n0 + n) * F + f] = pw.vin[n * JS + j];
        }
      if (a.S_prev && crank == 0)
        for (int t = tid; t < J * I * I; t += blockDim.x) {
          const int j = t / (I * I), ab = t % (I * I), ra = ab / I, cb = ab % I;
          const int hi = ra >= cb ? ra : cb, lo = ra >= cb ? cb : ra;
          double re = hi == lo ? Sd[j * H + pk_diag(hi)] : Sd[j * H + pk_re(hi, lo)];
          double im = hi == lo ? 0.0 : Sd[j * H + pk_re(hi, lo) + 1] * (ra >= cb ? 1.0 : -1.0);
          ((C2*)a.S_prev)[((u * J + j) * F + f) * I * I + ab] = mk<C2, R>(R(re), R(im));
        }
    }
    R acc[V];
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] = R(0);
    const R vfl_b = R(vfl[0]);
    int bad;
    if (rec) bad = a.vf_mode == 2 ? pw.template run<true, true>(acc, vfl_b, nullptr)
                                  : pw.template run<true, false>(acc, vfl_b, nullptr);
    else bad = a.vf_mode == 2 ? pw.template run<false, true>(acc, vfl_b, nullptr)
                              : pw.template run<false, false>(acc, vfl_b, nullptr);
    if (bad) sflag = 1;
    bin_reduce<R, V, 1>(acc, wpart, cpart, tot, C, VMAX, parity);
    if (rec && tid == 0 && crank == 0) a.ll[bin * nev + it] = -tot[V - 1];
    // S' = herm(sum T / v' / N) and its inverse for the next M-step
    for (int t = tid; t < J * H; t += blockDim.x) {
      const int j = t / H, e = t % H;
      (void)j;
      const double val = tot[(t / H) * H + e] / double(N);
      Sd[t] = val;
      Sc[t] = R(val);
    }
    __syncthreads();
    invert_all();
    __syncthreads();
  }
  if (rec) {
    pw.vin = vb[a.iters & 1];
    R acc[1] = {R(0)};
    if (pw.loglik(acc)) sflag = 1;
    bin_reduce<R, 1, 1>(acc, wpart, cpart, tot, C, VMAX, parity);
    if (tid == 0 && crank == 0) a.ll[bin * nev + a.iters] = -tot[0];
  }
  __syncthreads();
  if (sflag && crank == 0 && tid == 0) atomicOr(&a.status[bin], ST_NOT_PD);

  // ---------------- write back ----------------
  const R* vfin = vb[a.iters & 1];
  for (int e = tid; e < J * NL; e += blockDim.x) {
    const int n = e % NL, j = e / NL;
    if (n < NLr) ((R*)a.v_out)[((u * J + j) * (long long)N + n0 + n) * F + f] = vfin[n * JS + j];
  }
  if (crank == 0)
    for (int t = tid; t < J * I * I; t += blockDim.x) {
      const int j = t / (I * I), ab = t % (I * I), ra = ab / I, cb = ab % I;
      const int hi = ra >= cb ? ra : cb, lo = ra >= cb ? cb : ra;
      double re = hi == lo ? Sd[j * H + pk_diag(hi)] : Sd[j * H + pk_re(hi, lo)];
      double im = hi == lo ? 0.0 : Sd[j * H + pk_re(hi, lo) + 1] * (ra >= cb ? 1.0 : -1.0);
      ((C2*)a.S_out)[((u * J + j) * F + f) * I * I + ab] = mk<C2, R>(R(re), R(im));
    }
  if (C > 1) cg::this_cluster().sync();
}

}  // namespace ffca
