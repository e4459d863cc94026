// Bin-resident FastFCA-AS estimation loop (sm_100a).
//
// One thread-block cluster owns G frequency bins (a "bin group") for the
// whole run.  Each CTA of the cluster holds a contiguous frame range of those
// bins -- y (I complex) and v (J real) per point -- in shared memory (or, when
// a bin is too long for the cluster's shared memory, in a global scratch
// slab), so the observations are read from HBM once per run instead of twice
// per iteration.  Per outer iteration the CTA runs
//   phase A  fused E/M sweep + per-bin sums s0, s1        (fastfca.py:323-346)
//   reduce   warp shuffle -> smem -> DSMEM across the cluster, fixed order
//   lambda'  per (bin, source)                            (fastfca.py:341-345)
//   phase B  weighted covariances B_i = sum_n y y^H / w_i  (fastfca.py:352-358)
//   reduce
//   solve    P^-1, B_i^-1 [P^-H]_i per bin, fp64          (fastfca.py:359-370)
// separated only by __syncthreads / cluster barriers.  Bins of a group are
// interleaved lane-wise (bin = lane % G) so the one-time gather from the
// reference's (I, N, F) layout reads whole 32-byte sectors and the compute
// loops read shared memory conflict-free.
#pragma once

#include "common.cuh"

namespace ffca {

struct LoopArgs {
  int U, I, J, N, F;
  long long total_bins;
  int G;         // bins per cluster (lane-interleaved), power of two <= 4
  int C;         // cluster size (CTAs sharing one bin group, split over n)
  int NL;        // max frames held by one CTA (ceil(N / C))
  int iters, K;
  int p_only;     // skip the EM sweep: fixed_point_update_P (fastfca.py:197-237)
  int vf_mode;   // 0 scalar, 1 per-bin (U,F), 2 full (U,J,N,F), 3 auto (power floor)
  double vf_scalar;
  const void* vf;      // real array for modes 1, 2
  const void* y;       // (U, I, N, F) complex
  const void* P_in;    // (U, F, I, I) complex
  const void* lam_in;  // (U, J, F, I) real
  const void* v_in;    // (U, J, N, F) real
  void* P_out;
  void* lam_out;
  void* v_out;
  double* vf_out;      // optional (U, F): the floor actually used
  double* ll;          // optional (total_bins, 1 + 2*iters): per-bin likelihood parts
  int* status;         // (total_bins)
  void* scratch;       // non-resident slab storage (slab_bytes per CTA)
  long long slab_bytes;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

template <int I>
struct Shape {
  // i-chunking of the B accumulation: <= 64 accumulators per thread
  static constexpr int IC = (I * I * I <= 64) ? I : ((64 / (I * I)) > 0 ? (64 / (I * I)) : 1);
  static constexpr int NCH = (I + IC - 1) / IC;
  static constexpr int NB = IC * I * I;  // reals per chunk
  static constexpr bool PREG = I <= 4;   // keep P / lambda in registers
};

template <int I, int JM>
__host__ __device__ constexpr int loop_vmax() {
  return (JM * (1 + I) + 1) > (Shape<I>::NB + 1) ? (JM * (1 + I) + 1) : (Shape<I>::NB + 1);
}

// Shared-memory carve-up; identical on host (sizing) and device.
struct LoopSmem {
  size_t y, v, vf, Pc, Pd, Pinv, lamc, lamd, vfl, ldet, wpart, cpart, tot, bst, M, piv, rhs, total, slab;
  size_t ybytes, vbytes;
  __host__ __device__ LoopSmem(int I, int J, int G, int NL, int W, int rsz, int vf_mode, bool resident,
                               int VMAX) {
    size_t o = 0;
    const size_t csz = 2 * size_t(rsz);
    ybytes = align16(size_t(I) * NL * G * csz);
    vbytes = align16(size_t(J) * NL * G * rsz);
    const size_t fs = vf_mode == 2 ? vbytes : 0;
    slab = ybytes + vbytes + fs;
    if (resident) {
      y = o; o += ybytes;
      v = o; o += vbytes;
      vf = o; o += fs;
    } else {
      y = 0;
      v = ybytes;
      vf = ybytes + vbytes;
    }
    Pc = o;    o += align16(size_t(G) * I * I * csz);
    Pd = o;    o += align16(size_t(G) * I * I * 16);
    Pinv = o;  o += align16(size_t(G) * I * I * 16);
    lamc = o;  o += align16(size_t(G) * J * I * rsz);
    lamd = o;  o += align16(size_t(G) * J * I * 8);
    vfl = o;   o += align16(size_t(G) * 8);
    ldet = o;  o += align16(size_t(G) * 8);
    wpart = o; o += align16(size_t(W) * G * VMAX * 8);
    cpart = o; o += align16(size_t(2) * G * VMAX * 8);
    tot = o;   o += align16(size_t(G) * VMAX * 8);
    bst = o;   o += align16(size_t(G) * I * I * I * 8);
    M = o;     o += align16(size_t(G) * (I + 1) * I * I * 16);
    rhs = o;   o += align16(size_t(G) * (I + 1) * I * 16);
    piv = o;   o += align16(size_t(G) * (I + 1) * I * 4);
    total = o;
  }
};

// ------------------------------------------------------------------------
// Sum V per-thread values over all threads of one bin in the cluster.
// Result lands in tot[g*VMAX + k] (fp64) and is visible after return.
// Deterministic: shuffle butterfly, warps in index order, cluster ranks in
// rank order.  cpart is double-buffered (parity) so a fast CTA cannot
// overwrite partials a slower CTA is still reading over DSMEM.
// ------------------------------------------------------------------------
template <typename R, int V>
__device__ __forceinline__ void bin_reduce(const R (&vals)[V], int nv, double* wpart, double* cpart,
                                           double* tot, int G, int C, int VMAX, int& parity) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, W = blockDim.x >> 5;
  const int g = tid % G;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    if (k < nv) {
      R s = warp_sum_seg(vals[k], G);
      if (lane < G) wpart[(warp * G + g) * VMAX + k] = double(s);
    }
  }
  __syncthreads();
  double* cp = cpart + parity * G * VMAX;
  double* dst = (C > 1) ? cp : tot;
  for (int t = tid; t < G * nv; t += blockDim.x) {
    const int gg = t / nv, k = t % nv;
    double s = 0.0;
    for (int w = 0; w < W; ++w) s += wpart[(w * G + gg) * VMAX + k];
    dst[gg * VMAX + k] = s;
  }
  if (C > 1) {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    for (int t = tid; t < G * nv; t += blockDim.x) {
      const int gg = t / nv, k = t % nv;
      double s = 0.0;
      for (int r = 0; r < C; ++r) s += cl.map_shared_rank(cp, r)[gg * VMAX + k];
      tot[gg * VMAX + k] = s;
    }
    parity ^= 1;
  }
  __syncthreads();
}

template <typename R, int I, int JT, bool RES>
__global__ void __launch_bounds__(256) ffca_loop_kernel(const LoopArgs a) {
  using C2 = typename Cpx<R>::T;
  constexpr int JM = JT > 0 ? JT : 8;
  constexpr int IC = Shape<I>::IC, NCH = Shape<I>::NCH, NB = Shape<I>::NB;
  constexpr bool PREG = Shape<I>::PREG;
  constexpr int VMAX = loop_vmax<I, JM>();
  constexpr int VA = JM * (1 + I) + 1;
  const int J = JT > 0 ? JT : a.J;
  const int G = a.G, C = a.C;
  const int tid = threadIdx.x;
  const int g = tid % G;
  const int slot = tid / G, nslots = blockDim.x / G;

  extern __shared__ __align__(16) unsigned char smem[];
  const int W = blockDim.x >> 5;
  const bool resident = RES || a.scratch == nullptr;
  const LoopSmem L(I, J, G, a.NL, W, sizeof(R), a.vf_mode, resident, VMAX);

  int crank = 0;
  if (C > 1) crank = int(cg::this_cluster().block_rank());
  int parity = 0;
  const long long group = blockIdx.x / C;
  const int N = a.N, F = a.F;
  const int n0 = int((long long)crank * N / C);
  const int n1 = int((long long)(crank + 1) * N / C);
  const int NLr = n1 - n0;
  const int NL = a.NL;

  unsigned char* slab = resident ? smem : (unsigned char*)a.scratch + (long long)blockIdx.x * a.slab_bytes;
  C2* ys = (C2*)(slab + L.y);
  R* vs = (R*)(slab + L.v);
  R* vfs = (R*)(slab + L.vf);
  C2* Pc = (C2*)(smem + L.Pc);
  double2* Pd = (double2*)(smem + L.Pd);
  double2* Pinv = (double2*)(smem + L.Pinv);
  R* lamc = (R*)(smem + L.lamc);
  double* lamd = (double*)(smem + L.lamd);
  double* vfl = (double*)(smem + L.vfl);
  double* ldet = (double*)(smem + L.ldet);
  double* wpart = (double*)(smem + L.wpart);
  double* cpart = (double*)(smem + L.cpart);
  double* tot = (double*)(smem + L.tot);
  double* bst = (double*)(smem + L.bst);
  double2* Msys = (double2*)(smem + L.M);
  double2* rhsv = (double2*)(smem + L.rhs);
  int* pivs = (int*)(smem + L.piv);

  const long long bin = group * G + g;
  const bool active = bin < a.total_bins;
  const long long u = active ? bin / F : 0;
  const int f = active ? int(bin % F) : 0;

  const C2* __restrict__ yg = (const C2*)a.y;
  const R* __restrict__ vg = (const R*)a.v_in;

  // ---------------- load: gather (I,N,F) -> slab [i][n][g] ----------------
  // idx % G == tid % G == g because blockDim is a multiple of G.
  R psum = R(0);
  for (int idx = tid; idx < I * NL * G; idx += blockDim.x) {
    const int rest = idx / G;
    const int n = rest % NL, i = rest / NL;
    C2 val = mk<C2, R>(R(0), R(0));
    if (active && n < NLr) {
      val = yg[((u * I + i) * (long long)N + n0 + n) * F + f];
      psum += val.x * val.x + val.y * val.y;
    }
    ys[idx] = val;
  }
  for (int idx = tid; idx < J * NL * G; idx += blockDim.x) {
    const int rest = idx / G;
    const int n = rest % NL, j = rest / NL;
    R val = R(0);
    if (active && n < NLr) val = vg[((u * J + j) * (long long)N + n0 + n) * F + f];
    vs[idx] = val;
  }
  if (a.vf_mode == 2) {
    const R* vfg = (const R*)a.vf;
    for (int idx = tid; idx < J * NL * G; idx += blockDim.x) {
      const int rest = idx / G;
      const int n = rest % NL, j = rest / NL;
      R val = R(0);
      if (active && n < NLr) val = vfg[((u * J + j) * (long long)N + n0 + n) * F + f];
      vfs[idx] = val;
    }
  }
  for (int t = tid; t < G * I * I; t += blockDim.x) {
    const long long b = group * G + t / (I * I);
    double2 p = make_double2(0.0, 0.0);
    if (b < a.total_bins) {
      const C2 q = ((const C2*)a.P_in)[b * I * I + t % (I * I)];
      p = make_double2(double(q.x), double(q.y));
    }
    Pd[t] = p;
    Pc[t] = mk<C2, R>(R(p.x), R(p.y));
  }
  for (int t = tid; t < G * J * I; t += blockDim.x) {
    const int gg = t / (J * I), e = t % (J * I);
    const int j = e / I, i = e % I;
    const long long b = group * G + gg;
    double l = 0.0;
    if (b < a.total_bins) {
      const long long ub = b / F, fb = b % F;
      l = double(((const R*)a.lam_in)[((ub * J + j) * F + fb) * I + i]);
    }
    lamd[t] = l;
    lamc[t] = R(l);
  }
  __syncthreads();

  // ---------------- v floor per bin (fca.py:82-89 when auto) ----------------
  if (a.vf_mode == 3) {
    const R pv[1] = {psum};
    bin_reduce<R, 1>(pv, 1, wpart, cpart, tot, G, C, VMAX, parity);
    if (tid < G) {
      const double mean = tot[tid * VMAX] / (double(I) * double(N));
      const double fl = fmax(1e-10 * mean, double(Floors<R>::vmin));
      vfl[tid] = fl;
      const long long b = group * G + tid;
      if (a.vf_out && crank == 0 && b < a.total_bins) a.vf_out[b] = fl;
    }
  } else if (tid < G) {
    const long long b = group * G + tid;
    double fl = a.vf_scalar;
    if (a.vf_mode == 1 && b < a.total_bins) fl = double(((const R*)a.vf)[b]);
    vfl[tid] = fl;
  }
  __syncthreads();

  const bool rec = a.ll != nullptr;
  const int nev = 1 + 2 * a.iters;
  const R wfl = Floors<R>::weight;
  const R rI = R(I);
  const double invN = 1.0 / double(N);

  C2 Pr[PREG ? I : 1][PREG ? I : 1];
  R Lr[PREG ? JM : 1][PREG ? I : 1];
#define FFCA_LOAD_PL()                                                            \
  if constexpr (PREG) {                                                           \
    _Pragma("unroll") for (int x_ = 0; x_ < I; ++x_)                              \
    _Pragma("unroll") for (int y_ = 0; y_ < I; ++y_) Pr[x_][y_] = Pc[(g * I + x_) * I + y_]; \
    _Pragma("unroll") for (int j_ = 0; j_ < JM; ++j_)                             \
    _Pragma("unroll") for (int i_ = 0; i_ < I; ++i_)                              \
      Lr[j_][i_] = (j_ < J) ? lamc[(g * J + j_) * I + i_] : R(0);                  \
  }
#define FFCA_P(x_, y_) (PREG ? Pr[PREG ? (x_) : 0][PREG ? (y_) : 0] : Pc[(g * I + (x_)) * I + (y_)])
#define FFCA_L(j_, i_) (PREG ? Lr[PREG ? (j_) : 0][PREG ? (i_) : 0] : lamc[(g * J + (j_)) * I + (i_)])
  // y_t = P^H y ; q = |y_t|^2   (fastfca.py:442-446)
#define FFCA_TRANSFORM_Q(yv_, q_)                                                 \
  _Pragma("unroll") for (int b_ = 0; b_ < I; ++b_) {                              \
    C2 acc_ = mk<C2, R>(R(0), R(0));                                              \
    _Pragma("unroll") for (int a_ = 0; a_ < I; ++a_) cmac_conj(acc_, FFCA_P(a_, b_), yv_[a_]); \
    q_[b_] = acc_.x * acc_.x + acc_.y * acc_.y;                                   \
  }
  // w_i = max(sum_j v_j lambda_ji, floor)   (fastfca.py:324)
#define FFCA_WEIGHTS(vj_, w_)                                                     \
  _Pragma("unroll") for (int i_ = 0; i_ < I; ++i_) {                              \
    R s_ = R(0);                                                                  \
    _Pragma("unroll") for (int j_ = 0; j_ < JM; ++j_) if (j_ < J) s_ = fma(vj_[j_], FFCA_L(j_, i_), s_); \
    w_[i_] = fmax(s_, wfl);                                                       \
  }
#define FFCA_LOAD_POINT(n_, yv_, vj_)                                             \
  _Pragma("unroll") for (int i_ = 0; i_ < I; ++i_) yv_[i_] = ys[(i_ * NL + (n_)) * G + g]; \
  _Pragma("unroll") for (int j_ = 0; j_ < JM; ++j_) vj_[j_] = (j_ < J) ? vs[(j_ * NL + (n_)) * G + g] : R(0);

  // ======================= outer iterations =======================
  for (int it = 0; it < a.iters; ++it) {
    // ---------------- phase A: fused E/M sweep ----------------
    FFCA_LOAD_PL();
    double llA = 0.0;
    if (!a.p_only) {
      R acc[VA];
#pragma unroll
      for (int k = 0; k < VA; ++k) acc[k] = R(0);
      const R vfl_b = R(vfl[g]);
      if (active) {
        for (int n = slot; n < NLr; n += nslots) {
          C2 yv[I];
          R vj[JM], q[I], w[I], iw[I], qiw2[I];
          FFCA_LOAD_POINT(n, yv, vj);
          FFCA_TRANSFORM_Q(yv, q);
          FFCA_WEIGHTS(vj, w);
#pragma unroll
          for (int i = 0; i < I; ++i) {
            iw[i] = rcp(w[i]);
            qiw2[i] = (q[i] * iw[i]) * iw[i];
          }
          if (rec) {
            R l = R(0);
#pragma unroll
            for (int i = 0; i < I; ++i) l += flog(w[i]) + q[i] * iw[i];
            acc[VA - 1] += l;
          }
#pragma unroll
          for (int j = 0; j < JM; ++j) {
            if (j < J) {
              R r1 = R(0), r2 = R(0);
#pragma unroll
              for (int i = 0; i < I; ++i) {
                r1 = fma(iw[i], FFCA_L(j, i), r1);
                r2 = fma(qiw2[i], FFCA_L(j, i), r2);
              }
              const R v = vj[j];
              const R step = quot(((r1 - r2) * v) * v, rI);
              const R fl = (a.vf_mode == 2) ? vfs[(j * NL + n) * G + g] : vfl_b;
              const R vn = fmax(v - step, fl);
              const R ratio = quot(v, vn);
              acc[j] += ratio;
              const R rv = ratio * v;
#pragma unroll
              for (int i = 0; i < I; ++i) acc[JM + j * I + i] = fma(rv, qiw2[i] - iw[i], acc[JM + j * I + i]);
              vs[(j * NL + n) * G + g] = vn;
            }
          }
        }
      }
      bin_reduce<R, VA>(acc, rec ? VA : VA - 1, wpart, cpart, tot, G, C, VMAX, parity);
      if (rec && tid < G) llA = tot[tid * VMAX + VA - 1];
    }
    // ---------------- lambda' per (bin, source) ----------------
    for (int t = tid; t < (a.p_only ? 0 : G * J); t += blockDim.x) {
      const int gg = t / J, j = t % J;
      const double* T = tot + gg * VMAX;
      const double s0 = T[j] * invN;
      double mx = -1.0;
      double ln[I];
#pragma unroll
      for (int i = 0; i < I; ++i) {
        const double l = lamd[(gg * J + j) * I + i];
        ln[i] = l * s0 + l * l * (T[JM + j * I + i] * invN);
        mx = fmax(mx, ln[i]);
      }
#pragma unroll
      for (int i = 0; i < I; ++i) {
        const double x = fmax(ln[i], 1e-12 * mx);
        lamd[(gg * J + j) * I + i] = x;
        lamc[(gg * J + j) * I + i] = R(x);
      }
    }
    __syncthreads();

    // ---------------- phase B: weighted covariances ----------------
    FFCA_LOAD_PL();
    double llB = 0.0;
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
      R acc[NB + 1];
#pragma unroll
      for (int k = 0; k < NB + 1; ++k) acc[k] = R(0);
      const bool rl = rec && ch == 0;
      if (active) {
        for (int n = slot; n < NLr; n += nslots) {
          C2 yv[I];
          R vj[JM], w[I];
          FFCA_LOAD_POINT(n, yv, vj);
          FFCA_WEIGHTS(vj, w);
          if (rl) {
            R q[I];
            FFCA_TRANSFORM_Q(yv, q);
            R l = R(0);
#pragma unroll
            for (int i = 0; i < I; ++i) l += flog(w[i]) + q[i] * rcp(w[i]);
            acc[NB] += l;
          }
          // lower-triangle outer product: per row x: diag, then (x, y<x) re, im
          R O[I * I];
          {
            int k = 0;
#pragma unroll
            for (int x = 0; x < I; ++x) {
              O[k++] = yv[x].x * yv[x].x + yv[x].y * yv[x].y;
#pragma unroll
              for (int y2 = 0; y2 < x; ++y2) {
                O[k++] = yv[x].x * yv[y2].x + yv[x].y * yv[y2].y;
                O[k++] = yv[x].y * yv[y2].x - yv[x].x * yv[y2].y;
              }
            }
          }
#pragma unroll
          for (int ii = 0; ii < IC; ++ii) {
            const int i = ch * IC + ii;
            if (i < I) {
              const R iwv = rcp(w[i]);
#pragma unroll
              for (int k = 0; k < I * I; ++k) acc[ii * I * I + k] = fma(O[k], iwv, acc[ii * I * I + k]);
            }
          }
        }
      }
      bin_reduce<R, NB + 1>(acc, rl ? NB + 1 : NB, wpart, cpart, tot, G, C, VMAX, parity);
      if (rl && tid < G) llB = tot[tid * VMAX + NB];
      // keep this chunk of B in fp64 for the solve
      const int nbc = (ch == NCH - 1) ? (I - ch * IC) * I * I : NB;
      for (int t = tid; t < G * nbc; t += blockDim.x) {
        const int gg = t / nbc, k = t % nbc;
        bst[gg * I * I * I + ch * NB + k] = tot[gg * VMAX + k];
      }
    }
    __syncthreads();

    // ---------------- solve: P^-1 and new columns (fastfca.py:359-370) --------
    {
      const int s = tid % (I + 1);
      const int gg = tid / (I + 1);
      const long long b = group * G + gg;
      const bool bact = gg < G && b < a.total_bins;
      double2* Ms = Msys + (gg * (I + 1) + s) * I * I;
      int* pv = pivs + (gg * (I + 1) + s) * I;
      double2* rv = rhsv + (gg * (I + 1) + s) * I;
      if (bact && s > 0) {
        const int i = s - 1;
        const double* T = bst + gg * I * I * I + i * I * I;
        double tr = 0.0;
        for (int pass = 0; pass < 2; ++pass) {
          // full Hermitian B_i from the packed lower triangle, / N
          int k = 0;
          for (int x = 0; x < I; ++x) {
            const double d = T[k++] * invN;
            Ms[x * I + x] = make_double2(d + (pass ? 1e-10 * tr : 0.0), 0.0);
            if (!pass) tr += d;
            for (int y2 = 0; y2 < x; ++y2) {
              const double re = T[k++] * invN, im = T[k++] * invN;
              Ms[x * I + y2] = make_double2(re, im);
              Ms[y2 * I + x] = make_double2(re, -im);
            }
          }
          const bool okB = lu_factor<I>(Ms, pv);
          if (okB && pass == 0) break;
          // one trace-loaded retry (fastfca.py:184-194)
          if (pass == 1 && crank == 0) atomicOr(&a.status[b], okB ? ST_B_LOADED : ST_SINGULAR_B);
        }
      }
#pragma unroll 1
      for (int k = 0; k < a.K; ++k) {
        if (bact && s == 0) {
          for (int e = 0; e < I * I; ++e) Ms[e] = Pd[gg * I * I + e];
          const bool okP = lu_factor<I>(Ms, pv);
          if (!okP && crank == 0) atomicOr(&a.status[b], ST_SINGULAR_P);
          if (k == 0) ldet[gg] = lu_logabsdet<I>(Ms);
          for (int c = 0; c < I; ++c) {
            for (int x = 0; x < I; ++x) rv[x] = make_double2(x == c ? 1.0 : 0.0, 0.0);
            lu_solve<I>(Ms, pv, rv);
            for (int x = 0; x < I; ++x) Pinv[(gg * I + x) * I + c] = rv[x];
          }
        }
        __syncthreads();
        if (bact && s > 0) {
          const int i = s - 1;
          for (int x = 0; x < I; ++x) {
            const double2 z = Pinv[(gg * I + i) * I + x];
            rv[x] = make_double2(z.x, -z.y);  // [P^-H]_{x,i} = conj(P^-1_{i,x})
          }
          lu_solve<I>(Ms, pv, rv);
          for (int x = 0; x < I; ++x) {
            Pd[(gg * I + x) * I + i] = rv[x];
            Pc[(gg * I + x) * I + i] = mk<C2, R>(R(rv[x].x), R(rv[x].y));
          }
        }
        __syncthreads();
      }
    }
    if (rec && tid < G) {
      const long long b = group * G + tid;
      if (crank == 0 && b < a.total_bins) {
        const double ld = 2.0 * double(N) * ldet[tid];
        a.ll[b * nev + 2 * it] = -llA + ld;
        a.ll[b * nev + 2 * it + 1] = -llB + ld;
      }
    }
  }

  // ---------------- final likelihood evaluation (after the last P update) ----
  if (rec) {
    FFCA_LOAD_PL();
    R acc[1] = {R(0)};
    if (active) {
      for (int n = slot; n < NLr; n += nslots) {
        C2 yv[I];
        R vj[JM], q[I], w[I];
        FFCA_LOAD_POINT(n, yv, vj);
        FFCA_TRANSFORM_Q(yv, q);
        FFCA_WEIGHTS(vj, w);
#pragma unroll
        for (int i = 0; i < I; ++i) acc[0] += flog(w[i]) + q[i] * rcp(w[i]);
      }
    }
    bin_reduce<R, 1>(acc, 1, wpart, cpart, tot, G, C, VMAX, parity);
    if (tid < G) {
      const long long b = group * G + tid;
      double2* Ms = Msys + (tid * (I + 1)) * I * I;
      int* pv = pivs + (tid * (I + 1)) * I;
      for (int e = 0; e < I * I; ++e) Ms[e] = Pd[tid * I * I + e];
      lu_factor<I>(Ms, pv);
      if (crank == 0 && b < a.total_bins)
        a.ll[b * nev + 2 * a.iters] = -tot[tid * VMAX] + 2.0 * double(N) * lu_logabsdet<I>(Ms);
    }
  }
#undef FFCA_LOAD_PL
#undef FFCA_P
#undef FFCA_L
#undef FFCA_TRANSFORM_Q
#undef FFCA_WEIGHTS
#undef FFCA_LOAD_POINT

  // ---------------- write back ----------------
  R* vo = (R*)a.v_out;
  for (int idx = tid; idx < J * NL * G; idx += blockDim.x) {
    const int rest = idx / G;
    const int n = rest % NL, j = rest / NL;
    if (active && n < NLr) vo[((u * J + j) * (long long)N + n0 + n) * F + f] = vs[idx];
  }
  if (crank == 0) {
    for (int t = tid; t < G * I * I; t += blockDim.x) {
      const long long b = group * G + t / (I * I);
      if (b < a.total_bins) {
        const double2 p = Pd[t];
        ((C2*)a.P_out)[b * I * I + t % (I * I)] = mk<C2, R>(R(p.x), R(p.y));
      }
    }
    for (int t = tid; t < G * J * I; t += blockDim.x) {
      const int gg = t / (J * I), e = t % (J * I);
      const int j = e / I, i = e % I;
      const long long b = group * G + gg;
      if (b < a.total_bins) {
        const long long ub = b / F, fb = b % F;
        ((R*)a.lam_out)[((ub * J + j) * F + fb) * I + i] = R(lamd[t]);
      }
    }
  }
  // no CTA may exit while a peer can still read its shared memory
  if (C > 1) cg::this_cluster().sync();
}

}  // namespace ffca
