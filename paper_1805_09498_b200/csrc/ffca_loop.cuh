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
// separated only by __syncthreads / cluster barriers.
//
// Slab layout: one record per (frame n, bin g) at index n*G + g, holding the
// I complex observations (padded to an odd count RS) or the J powers (odd
// JS).  Lane l of a warp touches record (slot*G + g) = l + const, so record
// strides are odd and every LDS is bank-conflict free; a thread walks its
// frames with one pointer increment and immediate offsets.  Bins are
// interleaved lane-wise (g = lane % G) so the one-time gather from the
// reference's (I, N, F) layout reads whole 32-byte sectors.
#pragma once

#include "common.cuh"

namespace ffca {

// Development probe (build with -DFFCA_PHASE_PROBE): per-phase clock64 cycle sums of threads 0
// and 1 of the middle CTA, read back with ffca_debug_phase (loop_f32.cu).  Compiled out otherwise.
#ifdef FFCA_PHASE_PROBE
#ifndef FFCA_PROBE_T1
#define FFCA_PROBE_T1 1  // second probed thread (e.g. 64: the P group of the I > 4 solve)
#endif
__device__ unsigned long long g_phase[16];
__device__ unsigned long long g_fixed[4];  // thread 0 of the middle CTA: gather, floor, write-back cycles
#define FFCA_PROBE_INIT                                                       \
  long long _pt = clock64();                                                  \
  const bool _pr = (blockIdx.x == gridDim.x / 2) && (threadIdx.x == 0 || threadIdx.x == FFCA_PROBE_T1);
#define FFCA_PROBE(k)                                                                            \
  if (_pr) {                                                                                     \
    const long long _n = clock64();                                                              \
    atomicAdd(&g_phase[(k) + 8 * (threadIdx.x != 0)], (unsigned long long)(_n - _pt));           \
    _pt = _n;                                                                                    \
  }
#define FFCA_FIXED_T0 const long long _ft0 = clock64();
#define FFCA_FIXED(k)                                                                   \
  if (blockIdx.x == gridDim.x / 2 && threadIdx.x == 0) g_fixed[k] += clock64() - _ft0;
#else
#define FFCA_PROBE_INIT
#define FFCA_PROBE(k)
#define FFCA_FIXED_T0
#define FFCA_FIXED(k)
#endif



__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ constexpr int odd_up(int x) { return (x & 1) ? x : x + 1; }

// Slab record layout.  I <= 4: y records of odd(I) complex and separate v records of odd(J)
// reals.  I > 4: one interleaved record per frame, I complex observations followed by the J
// powers, odd(I + ceil(JM/2)) complex units long -- the odd stride keeps every lane-strided
// access conflict free, and one record per frame lets a slab of 2 x 2000 frames of an 8-channel
// bin fit the shared memory of a CTA pair (config 4).
__host__ __device__ constexpr bool loop_interleaved(int I) { return I > 4; }
__host__ __device__ constexpr int loop_rs(int I, int JM) {
  return loop_interleaved(I) ? odd_up(I + (JM + 1) / 2) : odd_up(I);
}
__host__ __device__ constexpr int loop_js(int I, int JM, int J) { return loop_interleaved(I) ? 2 * loop_rs(I, JM) : odd_up(J); }
// I > 4 solve: the 8-lane group that inverts P is the first group of the warp after the I
// groups of the B_i (so it never shares a warp with them); the CTA needs 8 (mP + 1) threads.
__host__ __device__ constexpr int loop_pgroup(int I) { return (I + 3) / 4 * 4; }
// complex64, I <= 4: frame-pair records.  Frames 2m and 2m + 1 of a bin share one record (twice the
// per-frame record): channel i's two observations are adjacent (one 16-byte load gives y_i of both
// frames) and the powers are stored as (v_j(2m), v_j(2m + 1)) pairs, so the per-point arithmetic
// runs on packed frame pairs (FFMA2) -- weights, reciprocals, the v update and the sums over frames
// all operate on both frames at once.  Strides stay odd multiples of 16 / 8 bytes: conflict free.
__host__ __device__ constexpr bool loop_pairs(int I, int rsz) { return !loop_interleaved(I) && rsz == 4; }
// Slab element offsets of frame n, bin g: y channel i in complex units, v source j in reals
// (RS complex / JS reals per frame record).
template <bool PAIRS>
__host__ __device__ __forceinline__ int slab_y(int n, int g, int i, int G, int RS) {
  return PAIRS ? ((n >> 1) * G + g) * 2 * RS + 2 * i + (n & 1) : (n * G + g) * RS + i;
}
template <bool PAIRS>
__host__ __device__ __forceinline__ int slab_v(int n, int g, int j, int G, int JS) {
  return PAIRS ? ((n >> 1) * G + g) * 2 * JS + 2 * j + (n & 1) : (n * G + g) * JS + j;
}

template <int I, int JM>
struct Shape {
  // i-chunking of the B accumulation: <= 64 accumulators per thread
  static constexpr int IC = (I * I * I <= 64) ? I : ((64 / (I * I)) > 0 ? (64 / (I * I)) : 1);
  static constexpr int NCH = (I + IC - 1) / IC;
  static constexpr int NB = IC * I * I;  // reals per chunk
  static constexpr bool PREG = I <= 4;   // keep P / lambda in registers
  static constexpr bool ILV = loop_interleaved(I);
  static constexpr int RS = loop_rs(I, JM);  // complex units per slab record
  // I > 4: phase B as a skinny GEMM, one accumulator unit (a complex off-diagonal entry or a
  // pair of diagonal entries of B, for every i) per lane of a warp
  static constexpr bool GROUPB = I > 4;
  static constexpr int NCX = I * (I - 1) / 2;   // complex off-diagonal entries
  static constexpr int NU = NCX + (I + 1) / 2;  // accumulator units (<= 32 for I <= 8)
  static constexpr int IWS = (I + 3) & ~3;      // reciprocal weights per frame in the warp buffer
};

template <int I, int JM>
__host__ __device__ constexpr int loop_vmax() {
  return Shape<I, JM>::GROUPB
             ? ((JM * (1 + I) + 1) > (I * I * I + 1) ? (JM * (1 + I) + 1) : (I * I * I + 1))
             : ((JM * (1 + I) + 1) > (Shape<I, JM>::NB + 1) ? (JM * (1 + I) + 1) : (Shape<I, JM>::NB + 1));
}

// Shared-memory carve-up; identical on host (sizing) and device.  The warp partials of the
// reductions (wpart) and the solver workspace (M) are never live at the same time and share
// one region.
struct LoopSmem {
  size_t y, v, vf, Pc, Pd, Pinv, lamc, lamd, vfl, ldet, wpart, cpart, tot, bst, M, piv, rhs, total, slab;
  size_t ybytes, vbytes;
  LoopSmem() = default;
  __host__ __device__ LoopSmem(int I, int J, int JM, int G, int NL, int W, int rsz, int vf_mode, bool resident,
                               int VMAX, bool tmem = false) {  // tmem: the y records live in tensor memory
    size_t o = 0;
    const size_t csz = 2 * size_t(rsz);
    const bool ilv = loop_interleaved(I);
    const int JS = loop_js(I, JM, J);
    const size_t NLs = loop_pairs(I, rsz) ? size_t((NL + 1) & ~1) : size_t(NL);  // frame-pair records
    ybytes = tmem ? 0 : align16(NLs * G * loop_rs(I, JM) * csz);
    vbytes = ilv ? 0 : align16(NLs * G * JS * rsz);
    const size_t fs = vf_mode == 2 ? align16(NLs * G * JS * rsz) : 0;
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
    cpart = o; o += align16(size_t(2) * G * VMAX * 8);
    tot = o;   o += align16(size_t(G) * VMAX * 8);
    bst = o;   // unused (the solves read the reduced sums in tot)
    {  // solver workspace: per-system matrices (I <= 4) or B_i^-1 + group rows (I > 4)
      const size_t m1 = size_t(G) * (I + 1) * I * I * 16, m2 = (size_t(I) * I * I + 2 * I * (loop_pgroup(I) + 1)) * 16;
      const int nseg = (G == 1 && !ilv && (rsz == 8 || I == 3)) ? 2 : 1;  // 16-lane segments (bin_reduce SEG)
      size_t wp = align16(size_t(W) * nseg * G * VMAX * rsz);  // warp partials in the compute type
      const size_t ms = align16(m1 > m2 ? m1 : m2);
      if (ilv) {  // I > 4 phase B: per-warp buffers of 32 frames' reciprocal weights
        const size_t wb = size_t(W) * 32 * ((I + 3) & ~3) * rsz;
        wp = wp > wb ? wp : wb;
      }
      wpart = M = o;
      o += wp > ms ? wp : ms;
    }
    rhs = o;   o += align16(size_t(G) * (I + 1) * I * 16);
    piv = o;   o += align16(size_t(G) * (I + 1) * I * 4);
    total = o;
  }
};

// Sum over the lanes of one bin (lanes sharing lane % G).
struct LoopArgs {
  int U, I, J, N, F;
  long long total_bins;
  int G;         // bins per cluster (lane-interleaved), power of two <= 4
  int C;         // cluster size (CTAs sharing one bin group, split over n)
  int NL;        // max frames held by one CTA (ceil(N / C))
  int iters, K;
  int p_only;    // skip the EM sweep: fixed_point_update_P (fastfca.py:197-237)
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
  const void* packed;  // optional: slab images (slab_bytes per CTA, in blockIdx order) written by
                       // slab_pack_kernel; resident CTAs then fill their slab with bulk copies
  void* scratch;       // non-resident slab storage (slab_bytes per CTA)
  long long slab_bytes;
  LoopSmem L;          // shared-memory carve-up, computed once on the host (kernel reads it from
                       // the constant bank instead of re-deriving offsets in registers)
};

template <int G, typename T>
__device__ __forceinline__ T bin_warp_sum(T x) {
#pragma unroll
  for (int o = 16; o >= G; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
  return x;
}

// ------------------------------------------------------------------------
// Sum V per-thread values over all threads of one bin in the cluster.
// Result lands in tot[g*VMAX + k] (fp64) and is visible after return.
// Deterministic: shuffle butterfly, warps in index order, cluster ranks in
// rank order.  cpart is double-buffered (parity) so a fast CTA cannot
// overwrite partials a slower CTA is still reading over DSMEM.
// ------------------------------------------------------------------------
// Block / cluster half of the reduction: wpart[(warp*G + g)*VMAX + k] holds each
// warp's partial for k < nv; sums over warps in index order, then cluster
// ranks in rank order, into tot[g*VMAX + k].
template <int G, typename T>
__device__ __forceinline__ void bin_reduce_tail(int nv, const T* wpart, double* cpart, double* tot, int C, int VMAX,
                                                int& parity, int W = -1) {
  const int tid = threadIdx.x;
  if (W < 0) W = blockDim.x >> 5;  // rows of warp partials per bin
  __syncthreads();
  double* cp = cpart + parity * G * VMAX;
  double* dst = (C > 1) ? cp : tot;
  for (int t = tid; t < G * nv; t += blockDim.x) {
    const int gg = t / nv, k = t % nv;
    double s = 0.0;
    for (int w = 0; w < W; ++w) s += double(wpart[(w * G + gg) * VMAX + k]);
    dst[gg * VMAX + k] = s;
  }
  if (C > 1) {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    for (int t = tid; t < G * nv; t += blockDim.x) {
      const int gg = t / nv, k = t % nv;
      double s = 0.0;
#pragma unroll 8
      for (int r = 0; r < C; ++r) s += cl.map_shared_rank(cp, r)[gg * VMAX + k];
      tot[gg * VMAX + k] = s;
    }
    parity ^= 1;
  }
  __syncthreads();
}

// One level of the halving butterfly (offset O, M live values), recursing to O/2.
template <typename R, int M, int O, int G, int N>
__device__ __forceinline__ void halving_step(R (&buf)[N], int lane, int& base) {
  if constexpr (O >= G) {
    const bool hi = (lane & O) != 0;
#pragma unroll
    for (int k = 0; k < M / 2; ++k) {
      const R keep = hi ? buf[k + M / 2] : buf[k];
      const R send = hi ? buf[k] : buf[k + M / 2];
      buf[k] = keep + __shfl_xor_sync(FULL, send, O);
    }
    if (hi) base += M / 2;
    halving_step<R, M / 2, O / 2, G>(buf, lane, base);
  }
}

// Warp half of the reduction as a transposed (halving) butterfly over the
// L = SEG lanes of a bin segment: at each step a lane keeps one half of its
// current values and receives the partner's copy of that half, so the V values
// take ~V shuffles instead of V*log2(L).  Lane with in-bin bits (b..bG) ends up
// owning values [base, base + V2/L), base = sum_s b_s * V2 / 2^(s+1).
// SEG = 32/G is one segment per warp and bin.  SEG = 16 at G = 1 splits every
// warp into two "virtual warps" of 16 frame slots: the sum tree is then exactly
// that of the G = 2 plan with twice the threads (16 lanes per bin, warps in
// slot order), so a bin's results do not depend on which of the two plans a
// batch size selects (complex128, abi_fastfca.cu plan_loop).
template <typename R, int V, int G, int SEG = 32 / G, typename T>
__device__ __forceinline__ void bin_reduce(const R (&vals)[V], T* wpart, double* cpart, double* tot, int C,
                                           int VMAX, int& parity) {
  constexpr int L = SEG;
  constexpr int NSEG = 32 / (G * SEG);  // segments per warp and bin
  static_assert(NSEG >= 1 && NSEG * G * SEG == 32, "segments tile the warp");
  constexpr int V2 = (V + L - 1) / L * L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane % G;
  R buf[V2];
#pragma unroll
  for (int k = 0; k < V2; ++k) buf[k] = k < V ? vals[k] : R(0);
  int base = 0;
#ifdef FFCA_EXP_SKIP_BUTTERFLY  // timing experiment only: no cross-lane sums (results are wrong)
  base = (lane / G) % L * (V2 / L);
#else
  halving_step<R, V2, G * SEG / 2, G>(buf, lane, base);
#endif
  const int vw = warp * NSEG + lane / (G * SEG);  // (virtual) warp row in slot order
  T* row = wpart + (vw * G + g) * VMAX;  // warp partials (the loop kernel keeps them in its compute type)
#pragma unroll
  for (int k = 0; k < V2 / L; ++k)
    if (base + k < V) row[base + k] = T(buf[k]);
  bin_reduce_tail<G>(V, wpart, cpart, tot, C, VMAX, parity, (int(blockDim.x) >> 5) * NSEG);
}

// 3 x 3 determinant of the rows r0 < r1 < r2 and columns c0 < c1 < c2 of a row-major 4 x 4 matrix.
__device__ __forceinline__ double2 det3_of4(const double2* A, int r0, int r1, int r2, int c0, int c1, int c2) {
  const double2 m0 = csub(cmul(A[r1 * 4 + c1], A[r2 * 4 + c2]), cmul(A[r1 * 4 + c2], A[r2 * 4 + c1]));
  const double2 m1 = csub(cmul(A[r1 * 4 + c0], A[r2 * 4 + c2]), cmul(A[r1 * 4 + c2], A[r2 * 4 + c0]));
  const double2 m2 = csub(cmul(A[r1 * 4 + c0], A[r2 * 4 + c1]), cmul(A[r1 * 4 + c1], A[r2 * 4 + c0]));
  return cadd(csub(cmul(A[r0 * 4 + c0], m0), cmul(A[r0 * 4 + c1], m1)), cmul(A[r0 * 4 + c2], m2));
}

// Column c of the cofactor matrix of an I x I complex matrix A (row-major in shared memory,
// I <= 4): out[x] = (-1)^(x+c) * minor(x, c), so that row c of A^-1 is out / det(A).  Elements are
// read from shared memory as needed (no register copy of A).
template <int I>
__device__ __forceinline__ void adjugate_column(const double2* A, int c, double2 (&out)[I]) {
  if constexpr (I == 1) {
    out[0] = make_double2(1.0, 0.0);
  } else if constexpr (I == 2) {
    const double sg = (c == 0) ? 1.0 : -1.0;
    const double2 a1 = A[2 + (1 - c)], a0 = A[1 - c];
    out[0] = make_double2(sg * a1.x, sg * a1.y);
    out[1] = make_double2(-sg * a0.x, -sg * a0.y);
  } else if constexpr (I == 3) {
    const int c1 = c == 0 ? 1 : 0, c2 = c == 2 ? 1 : 2;
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      const int r1 = x == 0 ? 1 : 0, r2 = x == 2 ? 1 : 2;
      const double2 p = cmul(A[r1 * 3 + c1], A[r2 * 3 + c2]), q = cmul(A[r1 * 3 + c2], A[r2 * 3 + c1]);
      const double2 m = make_double2(p.x - q.x, p.y - q.y);
      out[x] = ((x + c) & 1) ? make_double2(-m.x, -m.y) : m;
    }
  } else {
    static_assert(I == 4, "cofactors for I <= 4");
    const int c0 = c == 0 ? 1 : 0, c1 = c <= 1 ? 2 : 1, c2 = c <= 2 ? 3 : 2;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int r0 = x == 0 ? 1 : 0, r1 = x <= 1 ? 2 : 1, r2 = x <= 2 ? 3 : 2;
      const double2 m = det3_of4(A, r0, r1, r2, c0, c1, c2);
      out[x] = ((x + c) & 1) ? make_double2(-m.x, -m.y) : m;
    }
  }
}

// N consecutive reals from 16-byte aligned shared memory as 16-byte vector loads.
template <int N>
__device__ __forceinline__ void load_vec(const float* p, float (&o)[N]) {
#pragma unroll
  for (int i = 0; i < N; i += 4) {
    const float4 t = *(const float4*)(p + i);
    o[i] = t.x; o[i + 1] = t.y; o[i + 2] = t.z; o[i + 3] = t.w;
  }
}
template <int N>
__device__ __forceinline__ void load_vec(const double* p, double (&o)[N]) {
#pragma unroll
  for (int i = 0; i < N; i += 2) {
    const double2 t = *(const double2*)(p + i);
    o[i] = t.x; o[i + 1] = t.y;
  }
}

// Per-point work of one thread over its frames of one bin (registers only).
template <typename R, int I, int JM, int G, bool TM = false>
struct PointWork {
  using C2 = typename Cpx<R>::T;
  static constexpr int IC = Shape<I, JM>::IC, NB = Shape<I, JM>::NB, RS = Shape<I, JM>::RS;
  static constexpr int NCXP = I * (I - 1) / 2 > 0 ? I * (I - 1) / 2 : 1;  // complex off-diagonal entries
  static constexpr bool PREG = Shape<I, JM>::PREG;
  static constexpr int VA = JM * (1 + I) + 1;

  C2* ys;
  R* vs;
  const R* vfs;
  const C2* Pc;
  const R* lamc;
  int g, J, JS, rec0, rstep, npts;
  bool gslab;  // slab in global scratch: prefetch upcoming frames into L1
  R wfl, invI;
  static constexpr int IP2 = (I + 1) / 2;  // lambda stored as (i, i+1) pairs for FFMA2
  static constexpr int PFD = 2;            // prefetch distance (frames of this thread) on a global slab
  static constexpr bool PAIRS = loop_pairs(I, int(sizeof(R)));  // frame-pair records (complex64, I <= 4)
  C2 Pr[PREG ? I : 1][PREG ? I : 1];
  C2 Lp[PREG && !PAIRS ? JM : 1][PREG && !PAIRS ? IP2 : 1];  // lambda as (i, i+1) pairs (FFMA2 over i)
  R Ls[PAIRS ? JM : 1][PAIRS ? I : 1];                        // PAIRS: lambda as scalars (broadcast operands)
  int nfull;  // PAIRS: full frame pairs of this thread
  unsigned tmy;  // TM: tensor-memory address of this thread's y records (lane quadrant of its warp, column 0)
  int nrec;      // TM: records per thread (uniform over the CTA: the tcgen05.ld are warp-collective)
  static constexpr int TMW = 4 * I;  // TM: 32-bit columns per frame-pair record
  bool part;  // PAIRS: this thread also owns the bin's last, half-filled pair (odd frame count)

  __device__ __forceinline__ void load_PL() {
    if constexpr (PREG) {
#pragma unroll
      for (int x = 0; x < I; ++x)
#pragma unroll
        for (int y2 = 0; y2 < I; ++y2) Pr[x][y2] = Pc[(g * I + x) * I + y2];
      if constexpr (PAIRS) {
#pragma unroll
        for (int j = 0; j < JM; ++j)
#pragma unroll
          for (int i = 0; i < I; ++i) Ls[j][i] = (j < J) ? lamc[(g * J + j) * I + i] : R(0);
      } else {
#pragma unroll
        for (int j = 0; j < JM; ++j)
#pragma unroll
          for (int ip = 0; ip < IP2; ++ip) {
            const R l0 = (j < J) ? lamc[(g * J + j) * I + 2 * ip] : R(0);
            const R l1 = (j < J && 2 * ip + 1 < I) ? lamc[(g * J + j) * I + 2 * ip + 1] : R(0);
            Lp[j][ip] = mk<C2, R>(l0, l1);
          }
      }
    }
  }
  __device__ __forceinline__ C2 P(int x, int y2) const {
    if constexpr (PREG) return Pr[x][y2];
    else return Pc[(g * I + x) * I + y2];
  }
  __device__ __forceinline__ R Lam(int j, int i) const {
    if constexpr (PAIRS) return Ls[j][i];
    else if constexpr (PREG) return (i & 1) ? Lp[j][i >> 1].y : Lp[j][i >> 1].x;
    else return lamc[(g * J + j) * I + i];
  }
  // y_t = P^H y ; q = |y_t|^2   (fastfca.py:442-446)
  __device__ __forceinline__ void transform_q(const C2 (&yv)[I], R (&q)[I]) const {
#pragma unroll
    for (int b = 0; b < I; ++b) {
      C2 acc = mk<C2, R>(R(0), R(0));
#pragma unroll
      for (int x = 0; x < I; ++x) cmac_conj(acc, P(x, b), yv[x]);
      q[b] = acc.x * acc.x + acc.y * acc.y;
    }
  }
  // w_i = max(sum_j v_j lambda_ji, floor)   (fastfca.py:324)
  __device__ __forceinline__ void weights(const R (&vj)[JM], R (&w)[I]) const {
    if constexpr (PREG) {  // (w_i, w_i+1) pairs: one FFMA2 per source and pair
      C2 s2[IP2];
#pragma unroll
      for (int ip = 0; ip < IP2; ++ip) s2[ip] = mk<C2, R>(R(0), R(0));
#pragma unroll
      for (int j = 0; j < JM; ++j)
        if (j < J)
#pragma unroll
          for (int ip = 0; ip < IP2; ++ip) s2[ip] = fma2(bc2<R>(vj[j]), Lp[j][ip], s2[ip]);
#pragma unroll
      for (int i = 0; i < I; ++i) w[i] = fmax((i & 1) ? s2[i >> 1].y : s2[i >> 1].x, wfl);
    } else {
#pragma unroll
      for (int i = 0; i < I; ++i) {
        R s = R(0);
#pragma unroll
        for (int j = 0; j < JM; ++j)
          if (j < J) s = fma(vj[j], Lam(j, i), s);
        w[i] = fmax(s, wfl);
      }
    }
  }
  __device__ __forceinline__ void load_point(const C2* yp, const R* vp, C2 (&yv)[I], R (&vj)[JM]) const {
#pragma unroll
    for (int i = 0; i < I; ++i) yv[i] = yp[i];
#pragma unroll
    for (int j = 0; j < JM; ++j) vj[j] = (j < J) ? vp[j] : R(0);
  }

  // Phase A: fused E/M sweep over this thread's frames (fastfca.py:323-340).
  // Arithmetic is written on value pairs (fma2 -> FFMA2 for fp32): the
  // transform as 2 packed MACs per complex term, (r1_j, r2_j) against pairs
  // (1/w_i, q_i/w_i^2), and s1_j over pairs of i.
  template <bool REC, bool VF2>
  __device__ __forceinline__ void phaseA(R (&acc)[VA], const R vfl_b) {
    using P2 = C2;
    constexpr int IP = I / 2;           // i-pairs
    constexpr bool IODD = (I & 1) != 0;
    const C2* yp = ys + rec0 * RS;
    R* vp = vs + rec0 * JS;
    const R* fp = vfs + rec0 * JS;
    R s0[JM];
    P2 s1p[JM][IP > 0 ? IP : 1];
    R s1s[JM];
    R lacc = R(0);
#pragma unroll
    for (int j = 0; j < JM; ++j) {
      s0[j] = R(0);
      s1s[j] = R(0);
#pragma unroll
      for (int ip = 0; ip < (IP > 0 ? IP : 1); ++ip) s1p[j][ip] = mk<C2, R>(R(0), R(0));
    }
#pragma unroll 1
    for (int k = 0; k < npts; ++k, yp += rstep * RS, vp += rstep * JS, fp += rstep * JS) {
      if (gslab && k + PFD < npts) {  // the global slab is L2-latency-bound: fetch PFD frames ahead
        prefetch_l1(yp + PFD * rstep * RS);
        prefetch_l1(vp + PFD * rstep * JS);
      }
      C2 yv[I];
      R vj[JM];
      load_point(yp, vp, yv, vj);
      // y_t = P^H y, q = |y_t|^2
      R q[I];
#pragma unroll
      for (int b = 0; b < I; ++b) {
        P2 t = mk<C2, R>(R(0), R(0));
#pragma unroll
        for (int x = 0; x < I; ++x) {
          const C2 pp = P(x, b);
          t = fma2(yv[x], bc2<R>(pp.x), t);                                  // p.x (y.x, y.y)
          t = fma2(mk<C2, R>(yv[x].y, -yv[x].x), bc2<R>(pp.y), t);          // p.y (y.y, -y.x)
        }
        q[b] = t.x * t.x + t.y * t.y;
      }
      R w[I];
      weights(vj, w);
      // d_i = q_i / w_i^2 - 1 / w_i, so that r2_j - r1_j = sum_i lambda_ji d_i
      R iw[I], d[I];
#pragma unroll
      for (int i = 0; i < I; ++i) {
        iw[i] = rcp_pt(w[i]);
        d[i] = fma(q[i], iw[i], R(-1)) * iw[i];
      }
      if constexpr (REC) {
#pragma unroll
        for (int i = 0; i < I; ++i) lacc += flog(w[i]) + q[i] * iw[i];
      }
#pragma unroll
      for (int j = 0; j < JM; ++j) {
        if (j < J) {
          R sd = R(0);  // r2_j - r1_j
#pragma unroll
          for (int i = 0; i < I; ++i) sd = fma(Lam(j, i), d[i], sd);
          const R v = vj[j];
          R fl = vfl_b;
          if constexpr (VF2) fl = fp[j];
          // v' = v - v^2 (r1 - r2) / I   (fastfca.py:336-337)
          const R vn = fmax(fma(sd, (v * v) * invI, v), fl);
          const R ratio = v * rcp_pt(vn);
          s0[j] += ratio;
          const R rv = ratio * v;
#pragma unroll
          for (int ip = 0; ip < IP; ++ip) s1p[j][ip] = fma2(bc2<R>(rv), mk<C2, R>(d[2 * ip], d[2 * ip + 1]), s1p[j][ip]);
          if constexpr (IODD) s1s[j] = fma(rv, d[I - 1], s1s[j]);
          vp[j] = vn;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < JM; ++j) {
      acc[j] = s0[j];
#pragma unroll
      for (int ip = 0; ip < IP; ++ip) {
        acc[JM + j * I + 2 * ip] = s1p[j][ip].x;
        acc[JM + j * I + 2 * ip + 1] = s1p[j][ip].y;
      }
      if constexpr (IODD) acc[JM + j * I + I - 1] = s1s[j];
    }
    acc[VA - 1] = lacc;
  }

  // Phase A for I > 4 (P stays in shared memory): two frames per step, so every P element
  // read from shared memory feeds two points and the two points' dependent chains interleave;
  // lambda is held in registers for the whole sweep.  Same arithmetic per point as phaseA.
  template <bool REC, bool VF2>
  __device__ __forceinline__ void phaseA2(R (&acc)[VA], const R vfl_b) {
    R lam[JM][I];
#pragma unroll
    for (int j = 0; j < JM; ++j)
#pragma unroll
      for (int i = 0; i < I; ++i) lam[j][i] = (j < J) ? lamc[(g * J + j) * I + i] : R(0);
    constexpr int IP = I / 2;
    constexpr bool IODD = (I & 1) != 0;
    R s0[JM], s1s[JM];
    C2 s1p[JM][IP];  // (s1_j,2ip, s1_j,2ip+1) pairs: FFMA2
    R lacc = R(0);
#pragma unroll
    for (int j = 0; j < JM; ++j) {
      s0[j] = R(0);
      s1s[j] = R(0);
#pragma unroll
      for (int ip = 0; ip < IP; ++ip) s1p[j][ip] = mk<C2, R>(R(0), R(0));
    }
    const int st = rstep;
    const C2* yp = ys + rec0 * RS;
    R* vp = vs + rec0 * JS;
    const R* fp = vfs + rec0 * JS;
#pragma unroll 2
    for (int k = 0; k < npts; k += 2, yp += 2 * st * RS, vp += 2 * st * JS, fp += 2 * st * JS) {
      const bool two = k + 1 < npts;
      const int o1 = two ? st : 0;  // a lone last frame is computed twice, used once
      C2 yv[2][I];
      R vj[2][JM];
      load_point(yp, vp, yv[0], vj[0]);
      load_point(yp + o1 * RS, vp + o1 * JS, yv[1], vj[1]);
      R q[2][I];
      {
        // y_t = P^H y for both frames, row x of P at a time (contiguous in shared memory: vector
        // loads, every P element read once per frame pair)
        C2 t0[I], t1[I];
#pragma unroll
        for (int b = 0; b < I; ++b) t0[b] = t1[b] = mk<C2, R>(R(0), R(0));
#pragma unroll
        for (int x = 0; x < I; ++x) {
          C2 prow[I];
          if constexpr (sizeof(R) == 4 && (I % 2) == 0) {
#pragma unroll
            for (int b = 0; b < I; b += 2) {
              const float4 t = *(const float4*)(Pc + (g * I + x) * I + b);
              prow[b] = mk<C2, R>(t.x, t.y);
              prow[b + 1] = mk<C2, R>(t.z, t.w);
            }
          } else {
#pragma unroll
            for (int b = 0; b < I; ++b) prow[b] = P(x, b);
          }
          const C2 s0 = mk<C2, R>(yv[0][x].y, -yv[0][x].x), s1 = mk<C2, R>(yv[1][x].y, -yv[1][x].x);
#pragma unroll
          for (int b = 0; b < I; ++b) {
            t0[b] = fma2(yv[0][x], bc2<R>(prow[b].x), t0[b]);
            t0[b] = fma2(s0, bc2<R>(prow[b].y), t0[b]);
            t1[b] = fma2(yv[1][x], bc2<R>(prow[b].x), t1[b]);
            t1[b] = fma2(s1, bc2<R>(prow[b].y), t1[b]);
          }
        }
#pragma unroll
        for (int b = 0; b < I; ++b) {
          q[0][b] = t0[b].x * t0[b].x + t0[b].y * t0[b].y;
          q[1][b] = t1[b].x * t1[b].x + t1[b].y * t1[b].y;
        }
      }
      R iw[2][I], d[2][I];
#pragma unroll
      for (int i = 0; i < I; ++i) {
        C2 w2 = mk<C2, R>(R(0), R(0));  // (w of frame 0, w of frame 1)
#pragma unroll
        for (int j = 0; j < JM; ++j)
          if (j < J) w2 = fma2(mk<C2, R>(vj[0][j], vj[1][j]), bc2<R>(lam[j][i]), w2);
        const R w0 = fmax(w2.x, wfl), w1 = fmax(w2.y, wfl);
        iw[0][i] = rcp_pt(w0);
        iw[1][i] = rcp_pt(w1);
        d[0][i] = fma(q[0][i], iw[0][i], R(-1)) * iw[0][i];
        d[1][i] = fma(q[1][i], iw[1][i], R(-1)) * iw[1][i];
        if constexpr (REC) {
          lacc += flog(w0) + q[0][i] * iw[0][i];
          if (two) lacc += flog(w1) + q[1][i] * iw[1][i];
        }
      }
#pragma unroll
      for (int j = 0; j < JM; ++j) {
        if (j < J) {
          C2 sd = mk<C2, R>(R(0), R(0));
#pragma unroll
          for (int i = 0; i < I; ++i) sd = fma2(bc2<R>(lam[j][i]), mk<C2, R>(d[0][i], d[1][i]), sd);
          R fl0 = vfl_b, fl1 = vfl_b;
          if constexpr (VF2) {
            fl0 = fp[j];
            fl1 = fp[o1 * JS + j];
          }
          const R v0 = vj[0][j], v1 = vj[1][j];
          const R vn0 = fmax(fma(sd.x, (v0 * v0) * invI, v0), fl0);
          const R vn1 = fmax(fma(sd.y, (v1 * v1) * invI, v1), fl1);
          const R r0 = v0 * rcp_pt(vn0);
          const R r1 = two ? v1 * rcp_pt(vn1) : R(0);
          s0[j] += r0 + r1;
          const R rv0 = r0 * v0, rv1 = r1 * v1;
#pragma unroll
          for (int ip = 0; ip < IP; ++ip) {
            s1p[j][ip] = fma2(bc2<R>(rv0), mk<C2, R>(d[0][2 * ip], d[0][2 * ip + 1]), s1p[j][ip]);
            s1p[j][ip] = fma2(bc2<R>(rv1), mk<C2, R>(d[1][2 * ip], d[1][2 * ip + 1]), s1p[j][ip]);
          }
          if constexpr (IODD) s1s[j] = fma(rv1, d[1][I - 1], fma(rv0, d[0][I - 1], s1s[j]));
          vp[j] = vn0;
          if (two) vp[o1 * JS + j] = vn1;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < JM; ++j) {
      acc[j] = s0[j];
#pragma unroll
      for (int ip = 0; ip < IP; ++ip) {
        acc[JM + j * I + 2 * ip] = s1p[j][ip].x;
        acc[JM + j * I + 2 * ip + 1] = s1p[j][ip].y;
      }
      if constexpr (IODD) acc[JM + j * I + I - 1] = s1s[j];
    }
    acc[VA - 1] = lacc;
  }

  // Phase B: weighted covariances (fastfca.py:352-358), I <= 4 (all i in one
  // pass); with REC also the likelihood at (P, v', lambda') (after-EM).
  // Off-diagonal outer-product entries y_x conj(y_y) are (re, im) pairs and
  // the diagonal |y_x|^2 terms are paired up, so every accumulation is FFMA2.
  template <bool REC>
  __device__ __forceinline__ void phaseB(R (&acc)[NB + 1], int ch) const {
    using P2 = C2;
    constexpr int NCXs = I * (I - 1) / 2;  // complex entries
    constexpr int DP = I / 2;              // diagonal pairs
    constexpr bool IODD = (I & 1) != 0;
    (void)ch;
    const C2* yp = ys + rec0 * RS;
    const R* vp = vs + rec0 * JS;
    P2 ac[I][NCXs > 0 ? NCXs : 1];
    P2 ad[I][DP > 0 ? DP : 1];
    R as[I];
    R lacc = R(0);
#pragma unroll
    for (int i = 0; i < I; ++i) {
      as[i] = R(0);
#pragma unroll
      for (int c = 0; c < (NCXs > 0 ? NCXs : 1); ++c) ac[i][c] = mk<C2, R>(R(0), R(0));
#pragma unroll
      for (int c = 0; c < (DP > 0 ? DP : 1); ++c) ad[i][c] = mk<C2, R>(R(0), R(0));
    }
#pragma unroll 1
    for (int k = 0; k < npts; ++k, yp += rstep * RS, vp += rstep * JS) {
      C2 yv[I];
      R vj[JM], w[I];
      load_point(yp, vp, yv, vj);
      weights(vj, w);
      R iw[I];
#pragma unroll
      for (int i = 0; i < I; ++i) iw[i] = rcp_pt(w[i]);
      if constexpr (REC) {
        R q[I];
        transform_q(yv, q);
#pragma unroll
        for (int i = 0; i < I; ++i) lacc += flog(w[i]) + q[i] * iw[i];
      }
      R dg[I];
#pragma unroll
      for (int x = 0; x < I; ++x) dg[x] = yv[x].x * yv[x].x + yv[x].y * yv[x].y;
      P2 oc[NCXs > 0 ? NCXs : 1];
      {
        int c = 0;
#pragma unroll
        for (int x = 1; x < I; ++x)
#pragma unroll
          for (int y2 = 0; y2 < x; ++y2, ++c) {  // y_x conj(y_y) = y_y.x (y_x) + y_y.y (y_x.y, -y_x.x)
            P2 t = fma2(yv[x], bc2<R>(yv[y2].x), mk<C2, R>(R(0), R(0)));
            oc[c] = fma2(mk<C2, R>(yv[x].y, -yv[x].x), bc2<R>(yv[y2].y), t);
          }
      }
#pragma unroll
      for (int i = 0; i < I; ++i) {
        const P2 b = bc2<R>(iw[i]);
#pragma unroll
        for (int c = 0; c < NCXs; ++c) ac[i][c] = fma2(oc[c], b, ac[i][c]);
#pragma unroll
        for (int c = 0; c < DP; ++c) ad[i][c] = fma2(mk<C2, R>(dg[2 * c], dg[2 * c + 1]), b, ad[i][c]);
        if constexpr (IODD) as[i] = fma(dg[I - 1], iw[i], as[i]);
      }
    }
    // flatten into the packed lower-triangle order: per row x, diag then (x, y<x)
#pragma unroll
    for (int i = 0; i < I; ++i) {
      R* o = acc + i * I * I;
#pragma unroll
      for (int x = 0; x < I; ++x) {
        if (IODD && x == I - 1) o[x * x] = as[i];
        else o[x * x] = (x & 1) ? ad[i][x / 2].y : ad[i][x / 2].x;
      }
      int c = 0;
#pragma unroll
      for (int x = 1; x < I; ++x)
#pragma unroll
        for (int y2 = 0; y2 < x; ++y2, ++c) {
          o[x * x + 1 + 2 * y2] = ac[i][c].x;
          o[x * x + 2 + 2 * y2] = ac[i][c].y;
        }
    }
    acc[NB] = lacc;
  }

  // Phase B for I > 4 with two accumulator units per lane: lanes l and l + 16 own units l and
  // l + 16 (of the 32) and walk alternate frames of each 32-frame chunk (half h = l / 16 takes
  // frames h, h + 2, ...), so every weight load and loop step feeds 16 FFMA2 instead of 8; the two
  // halves' sums are folded with one shuffle at the end.  Same per-unit arithmetic as the one-unit
  // form (measured at config 4: 14.91 -> 14.56 ms).
  __device__ __forceinline__ C2 unit_z(const C2* rec, int ua, int ub, bool diag) const {
    // z = U V + X Z:
    // complex unit  ya conj(yb):  U = (ya.x, ya.y), V = (yb.x, yb.x), X = (ya.y, -ya.x), Z = (yb.y, yb.y)
    // diagonal pair (|ya|^2, |yb|^2): U = V = (ya.x, yb.x), X = Z = (ya.y, yb.y)
    const C2 ya = rec[ua], yb = rec[ub];
    const C2 U = mk<C2, R>(ya.x, diag ? yb.x : ya.y);
    const C2 V = mk<C2, R>(diag ? ya.x : yb.x, yb.x);
    const C2 X = mk<C2, R>(ya.y, diag ? yb.y : -ya.x);
    const C2 Z = mk<C2, R>(diag ? ya.y : yb.y, yb.y);
    return fma2(U, V, fma2(X, Z, mk<C2, R>(R(0), R(0))));
  }
  template <bool REC>
  __device__ __forceinline__ void phaseB_entry(C2 (&ac)[2][I], R& lacc, int NLr, bool active, R* wbuf,
                                               const int (&ua)[2], const int (&ub)[2], const bool (&dg)[2], int c0,
                                               int cstep) const {
    constexpr int IWS = Shape<I, JM>::IWS;
    const int lane = threadIdx.x & 31, h = lane >> 4;
    R lam[JM][I];
#pragma unroll
    for (int j = 0; j < JM; ++j)
#pragma unroll
      for (int i = 0; i < I; ++i) lam[j][i] = (j < J) ? lamc[j * I + i] : R(0);
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int i = 0; i < I; ++i) ac[k][i] = mk<C2, R>(R(0), R(0));
    const int nch = active ? (NLr + 31) / 32 : 0;
#pragma unroll 1
    for (int c = c0; c < nch; c += cstep) {
      {  // reciprocal weights of frame 32c + lane
        const int n = 32 * c + lane;
        const bool ok = n < NLr;
        const int nn = ok ? n : 0;
        const R* vp = vs + nn * JS;
        R vj[JM];
#pragma unroll
        for (int j = 0; j < JM; ++j) vj[j] = (j < J) ? vp[j] : R(0);
        R iw[IWS];
#pragma unroll
        for (int i = 0; i < IWS; ++i) iw[i] = R(0);
#pragma unroll
        for (int ip = 0; ip < I / 2; ++ip) {  // (w_2ip, w_2ip+1) pairs: FFMA2
          C2 s2 = mk<C2, R>(R(0), R(0));
#pragma unroll
          for (int j = 0; j < JM; ++j)
            if (j < J) s2 = fma2(bc2<R>(vj[j]), mk<C2, R>(lam[j][2 * ip], lam[j][2 * ip + 1]), s2);
          iw[2 * ip] = ok ? rcp_pt(fmax(s2.x, wfl)) : R(0);
          iw[2 * ip + 1] = ok ? rcp_pt(fmax(s2.y, wfl)) : R(0);
        }
        if constexpr (I & 1) {
          R s = R(0);
#pragma unroll
          for (int j = 0; j < JM; ++j)
            if (j < J) s = fma(vj[j], lam[j][I - 1], s);
          iw[I - 1] = ok ? rcp_pt(fmax(s, wfl)) : R(0);
        }
        if constexpr (REC) {
          if (ok) {
            C2 yv[I];
#pragma unroll
            for (int i = 0; i < I; ++i) yv[i] = ys[nn * RS + i];
            R q[I];
            transform_q(yv, q);
#pragma unroll
            for (int i = 0; i < I; ++i) lacc += flog(R(1) / iw[i]) + q[i] * iw[i];
          }
        }
        R* wr = wbuf + lane * IWS;
#pragma unroll
        for (int i = 0; i < IWS; i += 2) *(C2*)(wr + i) = mk<C2, R>(iw[i], iw[i + 1]);
      }
      __syncwarp();
      const int nf = min(32, NLr - 32 * c);
      const C2* rec = ys + (32 * c + h) * RS;
      const R* wq = wbuf + h * IWS;
#pragma unroll 8
      for (int f = h; f < nf; f += 2, rec += 2 * RS, wq += 2 * IWS) {
        // units 0..15 are complex entries whenever I >= 7 (NCX >= 16): no diagonal selects
        const C2 z0 = unit_z(rec, ua[0], ub[0], Shape<I, JM>::NCX >= 16 ? false : dg[0]);
        const C2 z1 = unit_z(rec, ua[1], ub[1], dg[1]);
        R wv[IWS];
        load_vec<IWS>(wq, wv);
#pragma unroll
        for (int i = 0; i < I; ++i) {
          ac[0][i] = fma2(z0, bc2<R>(wv[i]), ac[0][i]);
          ac[1][i] = fma2(z1, bc2<R>(wv[i]), ac[1][i]);
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int i = 0; i < I; ++i) {
        ac[k][i].x += __shfl_xor_sync(FULL, ac[k][i].x, 16);
        ac[k][i].y += __shfl_xor_sync(FULL, ac[k][i].y, 16);
      }
  }

  // ---------------- frame-pair point work (PAIRS: complex64, I <= 4) ----------------
  // One record holds frames a = 2m and b = 2m + 1.  Quantities of one point are frame pairs
  // (x = frame a, y = frame b), so every scalar step of the per-point algebra of phaseA / phaseB
  // becomes one packed FFMA2 for both frames; sums over frames are kept as (even, odd) pairs and
  // added at the end.  PART: frame b is the zero padding after an odd frame count -- its power
  // stays 0 and it contributes nothing (its floor is replaced by 1 so 0 / v' is 0, never 0 / 0).
  __device__ __forceinline__ void load_y_pair(const C2* yp, C2 (&ya)[I], C2 (&yb)[I]) const {
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const float4 t = *(const float4*)(yp + 2 * i);
      ya[i] = mk<C2, R>(t.x, t.y);
      yb[i] = mk<C2, R>(t.z, t.w);
    }
  }
  __device__ __forceinline__ void load_v_pair(const R* vp, C2 (&v2)[JM]) const {
#pragma unroll
    for (int j = 0; j < JM; ++j) v2[j] = (j < J) ? *(const C2*)(vp + 2 * j) : mk<C2, R>(R(0), R(0));
  }
  __device__ __forceinline__ void load_pair(const C2* yp, const R* vp, C2 (&ya)[I], C2 (&yb)[I], C2 (&v2)[JM]) const {
    load_y_pair(yp, ya, yb);
    load_v_pair(vp, v2);
  }
  // TM: record k of this thread from tensor memory (warp-collective: every lane of the warp calls it)
  __device__ __forceinline__ void tm_load_pair(int k, C2 (&ya)[I], C2 (&yb)[I]) const {
    static_assert(!TM || ((I == 3 || I == 4) && sizeof(R) == 4), "tensor-memory records: complex64, I = 3 or 4");
    if constexpr (TM) {
      float r[TMW];
      tm_rec_ld<TMW>(tmy + k * TMW, r);
      tm_rec_wait<TMW>(r);
#pragma unroll
      for (int i = 0; i < I; ++i) {
        ya[i] = mk<C2, R>(r[4 * i], r[4 * i + 1]);
        yb[i] = mk<C2, R>(r[4 * i + 2], r[4 * i + 3]);
      }
    }
  }
  // q_b = |(P^H y)_b|^2 for both frames, as a pair
  __device__ __forceinline__ void q_pair(const C2 (&ya)[I], const C2 (&yb)[I], C2 (&q2)[I]) const {
#pragma unroll
    for (int b = 0; b < I; ++b) {
      C2 ta = mk<C2, R>(R(0), R(0)), tb = ta;
#pragma unroll
      for (int x = 0; x < I; ++x) {
        const C2 pp = P(x, b);
        ta = fma2(ya[x], bc2<R>(pp.x), ta);
        ta = fma2(mk<C2, R>(ya[x].y, -ya[x].x), bc2<R>(pp.y), ta);
        tb = fma2(yb[x], bc2<R>(pp.x), tb);
        tb = fma2(mk<C2, R>(yb[x].y, -yb[x].x), bc2<R>(pp.y), tb);
      }
      q2[b] = mk<C2, R>(ta.x * ta.x + ta.y * ta.y, tb.x * tb.x + tb.y * tb.y);
    }
  }
  // floored weights w_i = max(sum_j v_j lambda_ji, floor) of both frames; returns 1 / w
  __device__ __forceinline__ void iw_pair(const C2 (&v2)[JM], C2 (&iw2)[I], C2 (&w2)[I]) const {
#pragma unroll
    for (int i = 0; i < I; ++i) {
      C2 w = mk<C2, R>(R(0), R(0));
#pragma unroll
      for (int j = 0; j < JM; ++j)
        if (j < J) w = fma2(v2[j], bc2<R>(Lam(j, i)), w);
      w = mk<C2, R>(fmax(w.x, wfl), fmax(w.y, wfl));
      w2[i] = w;
      iw2[i] = mk<C2, R>(rcp_pt(w.x), rcp_pt(w.y));
    }
  }

  template <bool REC, bool VF2, int PART>
  __device__ __forceinline__ void pairA(const C2* yp, R* vp, const R* fp, C2 (&s0)[JM], C2 (&s1)[JM][I], C2& lacc,
                                        const R vfl_b) const {
    C2 ya[I], yb[I];
    load_y_pair(yp, ya, yb);
    pairA_core<REC, VF2, PART>(ya, yb, vp, fp, s0, s1, lacc, vfl_b);
  }
  // PART: 0 full pair, 1 half pair (frame b is padding), 2 decided at run time by `half`
  template <bool REC, bool VF2, int PART>
  __device__ __forceinline__ void pairA_core(const C2 (&ya)[I], const C2 (&yb)[I], R* vp, const R* fp, C2 (&s0)[JM],
                                             C2 (&s1)[JM][I], C2& lacc, const R vfl_b, bool half = false) const {
    const bool isp = PART == 2 ? half : (PART == 1);
    C2 v2[JM];
    load_v_pair(vp, v2);
    C2 q2[I], iw2[I], w2[I], d2[I];
    q_pair(ya, yb, q2);
    iw_pair(v2, iw2, w2);
#pragma unroll
    for (int i = 0; i < I; ++i) {
      d2[i] = mul2(fma2(q2[i], iw2[i], bc2<R>(R(-1))), iw2[i]);  // d = q / w^2 - 1 / w
      if constexpr (REC)
        lacc = add2(lacc, mk<C2, R>(flog(w2[i].x) + q2[i].x * iw2[i].x,
                                    isp ? R(0) : flog(w2[i].y) + q2[i].y * iw2[i].y));
    }
#pragma unroll
    for (int j = 0; j < JM; ++j) {
      if (j < J) {
        C2 sd = mk<C2, R>(R(0), R(0));  // r2 - r1
#pragma unroll
        for (int i = 0; i < I; ++i) sd = fma2(bc2<R>(Lam(j, i)), d2[i], sd);
        C2 fl = bc2<R>(vfl_b);
        if constexpr (VF2) fl = *(const C2*)(fp + 2 * j);
        // v' = max(v - v^2 (r1 - r2) / I, floor)   (fastfca.py:336-337)
        C2 vn = fma2(sd, mul2(mul2(v2[j], v2[j]), bc2<R>(invI)), v2[j]);
        vn = mk<C2, R>(fmax(vn.x, fl.x), fmax(vn.y, fl.y));
        if constexpr (PART == 1) {
          *(C2*)(vp + 2 * j) = mk<C2, R>(vn.x, R(0));  // the padding frame keeps v = 0
          vn.y = R(1);
        } else if constexpr (PART == 2) {
          *(C2*)(vp + 2 * j) = mk<C2, R>(vn.x, isp ? R(0) : vn.y);
          vn.y = isp ? R(1) : vn.y;
        } else {
          *(C2*)(vp + 2 * j) = vn;
        }
        const C2 ratio = mul2(v2[j], mk<C2, R>(rcp_pt(vn.x), rcp_pt(vn.y)));
        s0[j] = add2(s0[j], ratio);
        const C2 rv = mul2(ratio, v2[j]);
#pragma unroll
        for (int i = 0; i < I; ++i) s1[j][i] = fma2(rv, d2[i], s1[j][i]);
      }
    }
  }

  template <bool REC, bool VF2>
  __device__ __forceinline__ void phaseA_pairs(R (&acc)[VA], const R vfl_b) const {
    C2 s0[JM], s1[JM][I], lacc = mk<C2, R>(R(0), R(0));
#pragma unroll
    for (int j = 0; j < JM; ++j) {
      s0[j] = lacc;
#pragma unroll
      for (int i = 0; i < I; ++i) s1[j][i] = lacc;
    }
    const C2* yp = ys + rec0 * 2 * RS;
    R* vp = vs + rec0 * 2 * JS;
    const R* fp = vfs + rec0 * 2 * JS;
    const int sy = rstep * 2 * RS, sv = rstep * 2 * JS;
    if constexpr (TM) {
#pragma unroll 1
      for (int k = 0; k < nrec; ++k, vp += sv, fp += sv) {
        C2 ya[I], yb[I];
        tm_load_pair(k, ya, yb);
        // one body for full and half pairs (the half pair selects at run time): half the loop's code
        if (k < nfull + (part ? 1 : 0)) pairA_core<REC, VF2, 2>(ya, yb, vp, fp, s0, s1, lacc, vfl_b, k == nfull);
      }
    } else {
#pragma unroll 1
    for (int k = 0; k < nfull; ++k, yp += sy, vp += sv, fp += sv) pairA<REC, VF2, false>(yp, vp, fp, s0, s1, lacc, vfl_b);
    if (part) pairA<REC, VF2, true>(yp, vp, fp, s0, s1, lacc, vfl_b);
    }
#pragma unroll
    for (int j = 0; j < JM; ++j) {
      acc[j] = s0[j].x + s0[j].y;
#pragma unroll
      for (int i = 0; i < I; ++i) acc[JM + j * I + i] = s1[j][i].x + s1[j][i].y;
    }
    acc[VA - 1] = lacc.x + lacc.y;
  }

  template <bool REC, bool PART>
  __device__ __forceinline__ void pairB(const C2* yp, const R* vp, C2 (&ac)[I][NCXP], C2 (&ad)[I][I], C2& lacc) const {
    C2 ya[I], yb[I];
    load_y_pair(yp, ya, yb);
    pairB_core<REC, PART>(ya, yb, vp, ac, ad, lacc);
  }
  template <bool REC, bool PART>
  __device__ __forceinline__ void pairB_core(const C2 (&ya)[I], const C2 (&yb)[I], const R* vp, C2 (&ac)[I][NCXP],
                                             C2 (&ad)[I][I], C2& lacc) const {
    C2 v2[JM];
    load_v_pair(vp, v2);
    C2 iw2[I], w2[I];
    iw_pair(v2, iw2, w2);
    if constexpr (REC) {
      C2 q2[I];
      q_pair(ya, yb, q2);
#pragma unroll
      for (int i = 0; i < I; ++i)
        lacc = add2(lacc, mk<C2, R>(flog(w2[i].x) + q2[i].x * iw2[i].x,
                                    PART ? R(0) : flog(w2[i].y) + q2[i].y * iw2[i].y));
    }
    C2 dg[I];
#pragma unroll
    for (int x = 0; x < I; ++x)
      dg[x] = mk<C2, R>(ya[x].x * ya[x].x + ya[x].y * ya[x].y, yb[x].x * yb[x].x + yb[x].y * yb[x].y);
    C2 za[NCXP], zb[NCXP];
    {
      int c = 0;
#pragma unroll
      for (int x = 1; x < I; ++x)
#pragma unroll
        for (int y2 = 0; y2 < x; ++y2, ++c) {  // y_x conj(y_y) = y_y.x (y_x) + y_y.y (y_x.y, -y_x.x)
          za[c] = fma2(mk<C2, R>(ya[x].y, -ya[x].x), bc2<R>(ya[y2].y), fma2(ya[x], bc2<R>(ya[y2].x), mk<C2, R>(R(0), R(0))));
          zb[c] = fma2(mk<C2, R>(yb[x].y, -yb[x].x), bc2<R>(yb[y2].y), fma2(yb[x], bc2<R>(yb[y2].x), mk<C2, R>(R(0), R(0))));
        }
    }
#pragma unroll
    for (int i = 0; i < I; ++i) {
#pragma unroll
      for (int c = 0; c < NCXP; ++c) {
        if (c < I * (I - 1) / 2) {
          ac[i][c] = fma2(za[c], bc2<R>(iw2[i].x), ac[i][c]);
          ac[i][c] = fma2(zb[c], bc2<R>(iw2[i].y), ac[i][c]);
        }
      }
#pragma unroll
      for (int x = 0; x < I; ++x) ad[i][x] = fma2(dg[x], iw2[i], ad[i][x]);
    }
  }

  // Phase B on frame pairs: B_i = sum_n y y^H / w_i (fastfca.py:352-358), packed lower triangle.
  template <bool REC>
  __device__ __forceinline__ void phaseB_pairs(R (&acc)[NB + 1]) const {
    C2 ac[I][NCXP], ad[I][I], lacc = mk<C2, R>(R(0), R(0));
#pragma unroll
    for (int i = 0; i < I; ++i) {
#pragma unroll
      for (int c = 0; c < NCXP; ++c) ac[i][c] = lacc;
#pragma unroll
      for (int x = 0; x < I; ++x) ad[i][x] = lacc;
    }
    const C2* yp = ys + rec0 * 2 * RS;
    const R* vp = vs + rec0 * 2 * JS;
    const int sy = rstep * 2 * RS, sv = rstep * 2 * JS;
    if constexpr (TM) {
#pragma unroll 1
      for (int k = 0; k < nrec; ++k, vp += sv) {
        C2 ya[I], yb[I];
        tm_load_pair(k, ya, yb);
        if constexpr (REC) {
          if (k < nfull) pairB_core<REC, false>(ya, yb, vp, ac, ad, lacc);
          else if (part && k == nfull) pairB_core<REC, true>(ya, yb, vp, ac, ad, lacc);
        } else {  // without the likelihood a half pair's zero padding frame adds nothing: one body
          if (k < nfull + (part ? 1 : 0)) pairB_core<REC, false>(ya, yb, vp, ac, ad, lacc);
        }
      }
    } else {
#pragma unroll 1
    for (int k = 0; k < nfull; ++k, yp += sy, vp += sv) pairB<REC, false>(yp, vp, ac, ad, lacc);
    if (part) pairB<REC, true>(yp, vp, ac, ad, lacc);
    }
#pragma unroll
    for (int i = 0; i < I; ++i) {
      R* o = acc + i * I * I;
      int c = 0;
#pragma unroll
      for (int x = 0; x < I; ++x) {
        o[x * x] = ad[i][x].x + ad[i][x].y;
#pragma unroll
        for (int y2 = 0; y2 < x; ++y2, ++c) {
          o[x * x + 1 + 2 * y2] = ac[i][c].x;
          o[x * x + 2 + 2 * y2] = ac[i][c].y;
        }
      }
    }
    acc[NB] = lacc.x + lacc.y;
  }

  // Likelihood partial on frame pairs (after the last P update).
  __device__ __forceinline__ void phaseL_pairs(R (&acc)[1]) const {
    C2 lacc = mk<C2, R>(R(0), R(0));
    const C2* yp = ys + rec0 * 2 * RS;
    const R* vp = vs + rec0 * 2 * JS;
    const int sy = rstep * 2 * RS, sv = rstep * 2 * JS;
    const int n = nfull + (part ? 1 : 0);
#pragma unroll 1
    for (int k = 0; k < (TM ? nrec : n); ++k, yp += sy, vp += sv) {
      const bool half = part && k == n - 1;
      C2 ya[I], yb[I], v2[JM], q2[I], iw2[I], w2[I];
      if constexpr (TM) {
        tm_load_pair(k, ya, yb);  // warp-collective: every lane, every record
        if (k >= n) continue;
        load_v_pair(vp, v2);
      } else {
        load_pair(yp, vp, ya, yb, v2);
      }
      q_pair(ya, yb, q2);
      iw_pair(v2, iw2, w2);
#pragma unroll
      for (int i = 0; i < I; ++i)
        lacc = add2(lacc, mk<C2, R>(flog(w2[i].x) + q2[i].x * iw2[i].x,
                                    half ? R(0) : flog(w2[i].y) + q2[i].y * iw2[i].y));
    }
    acc[0] += lacc.x + lacc.y;
  }

  // Likelihood partial sum_n,i ln w + q / w at the current state.
  __device__ __forceinline__ void phaseL(R (&acc)[1]) const {
    const C2* yp = ys + rec0 * RS;
    const R* vp = vs + rec0 * JS;
#pragma unroll 1
    for (int k = 0; k < npts; ++k, yp += rstep * RS, vp += rstep * JS) {
      C2 yv[I];
      R vj[JM], q[I], w[I];
      load_point(yp, vp, yv, vj);
      transform_q(yv, q);
      weights(vj, w);
#pragma unroll
      for (int i = 0; i < I; ++i) acc[0] += flog(w[i]) + q[i] * rcp_pt(w[i]);
    }
  }
};

// P^-1 by the 8 lanes r = 0..7 of one group (row per lane, Gauss-Jordan with partial pivoting,
// numpy.linalg.inv's pivot order) into Pinv (row-major); with rec, log|det P| into ldet[0].
template <int I>
__device__ __forceinline__ void invert_P_group(const double2* Pd, double2* Pinv, double2* srow, int r, bool rec,
                                               double* ldet, int* status, long long group, bool report) {
  const unsigned gmask = 0xFFu << (8 * ((threadIdx.x >> 3) & 3));
  double2 ar[I], er[I];
#pragma unroll
  for (int c = 0; c < I; ++c) {
    er[c] = make_double2(c == r ? 1.0 : 0.0, 0.0);
    ar[c] = r < I ? Pd[r * I + c] : make_double2(0.0, 0.0);
  }
  int krow;
  double ld = 0.0;
  const bool ok = rec ? gj_group<I, true>(ar, er, r, gmask, srow, krow, ld)
                      : gj_group<I, false>(ar, er, r, gmask, srow, krow, ld);
  if (!ok && r == 0 && report) atomicOr(&status[group], ST_SINGULAR_P);
  if (rec && r == 0) ldet[0] = ld;
  if (r < I)
#pragma unroll
    for (int c = 0; c < I; ++c) Pinv[krow * I + c] = er[c];
}

// [P^-H]_i (i < I <= 4) of every bin of the group from the adjugate of P (cofactors / det),
// written row-wise into Pinv[(g * I + i) * I + x]; lane t = g * I + i of warp 1 handles bin g,
// column i.  Flags an exactly singular P (zero determinant) and records log|det P| with rec.
template <int I, int G>
__device__ __forceinline__ void pinvh_columns(const double2* Pd, double2* Pinv, double* ldet, int* status,
                                              long long group, long long total_bins, int crank, bool rec) {
  if ((threadIdx.x >> 5) != 1) return;
  const int t = threadIdx.x & 31;
  const int gg = t / I, i = t % I;
  const long long b = group * G + gg;
  const bool act = gg < G && b < total_bins;
  double2 z[I], det = make_double2(0.0, 0.0);
  const double2* Pb = Pd + (act ? gg : 0) * I * I;
  if constexpr (I == 4) {
    // det along column 0 from the i = 0 lane's cofactors, shuffled to the bin's other lanes
    adjugate_column<I>(Pb, i, z);
#pragma unroll
    for (int x = 0; x < I; ++x) det = cadd(det, cmul(Pb[x * I], z[x]));
    const int src = (t / I) * I;
    det.x = __shfl_sync(FULL, det.x, src);
    det.y = __shfl_sync(FULL, det.y, src);
  } else {
    double2 c0[I];
    adjugate_column<I>(Pb, i, z);
    adjugate_column<I>(Pb, 0, c0);
#pragma unroll
    for (int x = 0; x < I; ++x) det = cadd(det, cmul(Pb[x * I], c0[x]));
  }
  if (!act) return;
  if (det.x == 0.0 && det.y == 0.0 && i == 0 && crank == 0) atomicOr(&status[b], ST_SINGULAR_P);
  if (rec && i == 0) ldet[gg] = log(hypot(det.x, det.y));
  const double2 rd = crecip(det);
#pragma unroll
  for (int x = 0; x < I; ++x) {  // [P^-H]_{x,i} = conj(P^-1_{i,x}) = conj(C[x][i] / det)
    const double2 q = cmul(z[x], rd);
    Pinv[(gg * I + i) * I + x] = make_double2(q.x, -q.y);
  }
}

// Slab images for the bulk gather: a 256-thread CTA reads a tile of 32 consecutive bins x FT
// frames of y (U, I, N, F) and v (U, J, N, F) with bin-contiguous (coalesced) loads into shared
// memory, then writes each group's records in the loop kernel's slab order -- consecutive lanes
// write consecutive record words of one image.  Records past a bin's channels / sources are zero
// padding; bins past the end are zero.  Frames are mapped to the cluster rank that owns them.
struct PackArgs {
  const void* y;
  const void* v;
  void* packed;
  int I, J, N, F, G, C, RS, JS, FT;
  int ilv;
  int pairs;  // frame-pair records (loop_pairs)
  long long total_bins, ngroups, slab_bytes;
  long long Ly, Lv;  // record regions inside an image
};

template <typename R>
__global__ void __launch_bounds__(256) slab_pack_kernel(const PackArgs a) {
  using C2 = typename Cpx<R>::T;
  extern __shared__ __align__(16) unsigned char psm[];
  __shared__ int rk[32], nlk[32];  // cluster rank / local frame of each tile frame
  const int I = a.I, J = a.J, N = a.N, F = a.F, G = a.G, C = a.C, RS = a.RS, JS = a.JS, FT = a.FT;
  C2* yt = (C2*)psm;               // [FT][32][I]
  R* vt = (R*)(yt + FT * 32 * I);  // [FT][32][J]
  const int tid = threadIdx.x;
  const long long b0 = (long long)blockIdx.x * 32;
  const int m0 = blockIdx.y * FT;
  const int nf = min(FT, N - m0);
  const C2* yg = (const C2*)a.y;
  const R* vg = (const R*)a.v;
  if (tid < FT) {
    const int n = m0 + tid;
    int r = int((long long)n * C / N);
    while (r + 1 < C && (long long)(r + 1) * N / C <= n) ++r;
    while (r > 0 && (long long)r * N / C > n) --r;
    rk[tid] = r;
    nlk[tid] = n - int((long long)r * N / C);
  }
  // this lane's bin (the same for every pass: 256 threads = 8 rows of 32 bins)
  const int bl = tid & 31, row0 = tid >> 5;
  const long long bin = b0 + bl;
  const bool bok = bin < a.total_bins;
  const long long u = bok ? bin / F : 0, f = bok ? bin % F : 0;
  const C2* yb = yg + (u * I * (long long)N + m0) * F + f;
  const R* vb = vg + (u * J * (long long)N + m0) * F + f;
  for (int t = row0; t < I * FT; t += 8) {  // t = i * FT + nt
    const int nt = t % FT, i = t / FT;
    yt[(nt * 32 + bl) * I + i] = (bok && nt < nf) ? yb[((long long)i * N + nt) * F] : mk<C2, R>(R(0), R(0));
  }
  for (int t = row0; t < J * FT; t += 8) {
    const int nt = t % FT, j = t / FT;
    vt[(nt * 32 + bl) * J + j] = (bok && nt < nf) ? vb[((long long)j * N + nt) * F] : R(0);
  }
  __syncthreads();
  // one record per thread and pass: (frame nt, group qi, bin g); records of one group and frame
  // are adjacent in the image, so a warp writes a few contiguous runs
  for (int t = tid; t < nf * 32; t += blockDim.x) {
    const int nt = t >> 5, col = t & 31, qi = col / G, g = col % G;
    const long long q = b0 / G + qi;
    if (q >= a.ngroups) continue;
    unsigned char* img = (unsigned char*)a.packed + (q * C + rk[nt]) * a.slab_bytes;
    const int nl = nlk[nt];
    C2* yr = (C2*)(img + a.Ly);
    const C2* src = yt + (nt * 32 + col) * I;
    const R* vsrc = vt + (nt * 32 + col) * J;
    for (int s = 0; s < RS; ++s) {
      C2 val = mk<C2, R>(R(0), R(0));
      if (s < I) {
        val = src[s];
      } else if (a.ilv) {  // interleaved record: the J powers follow the I observations
        const int j = 2 * (s - I);
        val = mk<C2, R>(j < J ? vsrc[j] : R(0), j + 1 < J ? vsrc[j + 1] : R(0));
      }
      yr[a.pairs ? slab_y<true>(nl, g, s, G, RS) : slab_y<false>(nl, g, s, G, RS)] = val;
    }
    if (!a.ilv) {
      R* vr = (R*)(img + a.Lv);
      for (int j = 0; j < JS; ++j)
        vr[a.pairs ? slab_v<true>(nl, g, j, G, JS) : slab_v<false>(nl, g, j, G, JS)] = j < J ? vsrc[j] : R(0);
    }
  }
}

// FAST: the plain estimation loop (no likelihood recording, no full floor array, no P-only pass,
// one inner iteration) -- those paths compile out, which keeps the hot instantiations smaller
// (instruction cache) and lighter on registers.  The launcher picks it when a call allows.
template <typename R, int I, int JT, int G, bool RES, bool FAST = false, bool TM = false>
__global__ void __launch_bounds__(TM ? 128 : 256, (TM && I == 3) ? 4 : ((I == 4 || (I > 4 && RES)) ? 1 : 2)) ffca_loop_kernel(const LoopArgs a) {
  static_assert(!TM || (RES && sizeof(R) == 4 && ((G == 4 && I == 3) || (FAST && G == 1 && I == 4))),
                "tensor-memory plans: complex64, 4-bin CTAs at I = 3 (lean or full loop) or lean cluster CTAs at I = 4");
  using C2 = typename Cpx<R>::T;
  constexpr int JM = JT > 0 ? JT : 8;
  constexpr int IC = Shape<I, JM>::IC, NCH = Shape<I, JM>::NCH, NB = Shape<I, JM>::NB;
  constexpr bool PREG = Shape<I, JM>::PREG;
  constexpr int RS = Shape<I, JM>::RS;
  constexpr int VMAX = loop_vmax<I, JM>();
  constexpr int VA = JM * (1 + I) + 1;
  const int J = JT > 0 ? JT : a.J;
  const int JS = loop_js(I, JM, J);
  const int C = G > 1 ? 1 : a.C;  // multi-bin groups never form clusters (plan_loop): the DSMEM paths compile out
  const int tid = threadIdx.x;
  const int g = tid % G;
  const int slot = tid / G, nslots = blockDim.x / G;
  // complex128 one-bin CTAs reduce over 16-lane segments (bin_reduce): bitwise the G = 2 plan
  constexpr int SEG = (G == 1 && I <= 4 && (sizeof(R) == 8 || I == 3)) ? 16 : 32 / G;
  constexpr bool PAIRS = loop_pairs(I, int(sizeof(R)));

  extern __shared__ __align__(16) unsigned char smem[];
  const int W = blockDim.x >> 5;
  const bool resident = RES || a.scratch == nullptr;
  const LoopSmem& L = a.L;
  // the host sized the launch with this carve-up; trap rather than run past it
  if (L.total > dynamic_smem_bytes()) __trap();

  int crank = 0;
  if (C > 1) crank = int(cg::this_cluster().block_rank());
  int parity = 0;
  const long long group = blockIdx.x / C;
  const int N = a.N, F = a.F;
  const int n0 = int((long long)crank * N / C);
  const int n1 = int((long long)(crank + 1) * N / C);
  const int NLr = n1 - n0;
  const int NL = a.NL;
  const int NLs = PAIRS ? (NL + 1) & ~1 : NL;  // frames the slab holds (frame pairs: even)

  unsigned char* slab = resident ? smem : (unsigned char*)a.scratch + (long long)blockIdx.x * a.slab_bytes;
  C2* ys = (C2*)(slab + L.y);
  R* vs = Shape<I, JM>::ILV ? (R*)(ys + I) : (R*)(slab + L.v);  // interleaved: v follows y in each record
  R* vfs = (R*)(slab + L.vf);
  C2* Pc = (C2*)(smem + L.Pc);
  double2* Pd = (double2*)(smem + L.Pd);
  double2* Pinv = (double2*)(smem + L.Pinv);
  R* lamc = (R*)(smem + L.lamc);
  double* lamd = (double*)(smem + L.lamd);
  double* vfl = (double*)(smem + L.vfl);
  double* ldet = (double*)(smem + L.ldet);
  R* wpart = (R*)(smem + L.wpart);
  double* cpart = (double*)(smem + L.cpart);
  double* tot = (double*)(smem + L.tot);
  double2* Msys = (double2*)(smem + L.M);
  double2* rhsv = (double2*)(smem + L.rhs);
  int* pivs = (int*)(smem + L.piv);

  const long long bin = group * G + g;
  const bool active = bin < a.total_bins;
  const long long u = active ? bin / F : 0;
  const int f = active ? int(bin % F) : 0;

  const C2* __restrict__ yg = (const C2*)a.y;
  const R* __restrict__ vg = (const R*)a.v_in;
  FFCA_FIXED_T0

  // ---------------- load: gather (I,N,F) -> slab records ----------------
  // Consecutive lanes take consecutive bins g of the group, then frames, so a
  // warp reads whole 32-byte sectors of y[i, n, f..f+G).  Resident slabs are
  // filled with cp.async (zero-fill for padding), keeping every load of the
  // thread in flight at once.
  __shared__ unsigned long long gather_bar;
  // TM: the y records of the CTA's bins live in tensor memory as thread-private arrays (thread t
  // owns frame pairs slot + k nslots, k < nrec, 4 I columns each).  I = 3: 128 columns x 128 lanes
  // per 4-bin CTA, four CTAs fill the SM's 512 columns.  I = 4 (cluster plans): 256 columns, two CTAs
  // per SM, each holding twice the frames shared memory alone would.  Shared memory holds the powers v.
  __shared__ unsigned tm_base_s;
  unsigned tmy = 0, tmcols = 0;
  const int nrec = (NLs / 2 + nslots - 1) / nslots;
  if constexpr (TM) {
    constexpr int TMW = 4 * I;
    tmcols = nrec * TMW <= 128 ? 128u : (nrec * TMW <= 256 ? 256u : 512u);
    if (nrec * TMW > 512 || blockDim.x != 128) __trap();
    if (tid < 32) tmem_alloc(&tm_base_s, tmcols);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    tmy = tm_base_s + ((unsigned((tid >> 5) & 3) * 32u) << 16);
#pragma unroll 2
    for (int k = 0; k < nrec; ++k) {
      const int m = slot + k * nslots;
      float r[TMW];
#pragma unroll
      for (int i = 0; i < I; ++i)
#pragma unroll
        for (int par = 0; par < 2; ++par) {
          const int n = 2 * m + par;
          C2 z = mk<C2, R>(R(0), R(0));
          if (active && n < NLr) z = __ldg(yg + ((u * I + i) * (long long)N + n0 + n) * F + f);
          r[4 * i + 2 * par] = z.x;
          r[4 * i + 2 * par + 1] = z.y;
        }
      tm_rec_st<TMW>(tmy + k * TMW, r);
    }
    tmem_wait_st();
  }
  if (a.packed && resident) {
    // one TMA-engine bulk copy stream of this CTA's contiguous slab image (y and v records)
    const unsigned bytes = unsigned(L.ybytes + L.vbytes);
    if (tid == 0) {
      mbar_init(&gather_bar, 1);
      mbar_expect_tx(&gather_bar, bytes);
      const unsigned char* src = (const unsigned char*)a.packed + (long long)blockIdx.x * a.slab_bytes;
      constexpr unsigned CH = 32768;
      for (unsigned o = 0; o < bytes; o += CH) bulk_g2s(smem + o, src + o, bytes - o < CH ? bytes - o : CH, &gather_bar);
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
  }
  if (!(a.packed && resident)) {
    const R* vfg = (const R*)a.vf;
    const bool vf2g = !FAST && a.vf_mode == 2;
    if (resident) {
      // Pointer-bumped frame loops: iteration k copies frame slot + k * nslots (nslots is even, so
      // the slab offset advances by a constant in both record layouts); frames >= NLr zero-fill.
      const int nit = slot < NLs ? (NLs - slot + nslots - 1) / nslots : 0;
      const int nok = (active && slot < NLr) ? (NLr - slot + nslots - 1) / nslots : 0;
      const long long gstep = (long long)nslots * F;
      const int ystep = nslots * G * RS, vstep = nslots * G * JS;
#pragma unroll 1
      for (int i = 0; i < (TM ? 0 : I); ++i) {
        const C2* col = yg + ((u * I + i) * (long long)N + n0) * F + f;
        const C2* src = col + (long long)slot * F;
        C2* dst = ys + slab_y<PAIRS>(slot, g, i, G, RS);
#pragma unroll 1
        for (int k = 0; k < nit; ++k, src += gstep, dst += ystep) cp_async<sizeof(C2)>(dst, k < nok ? src : col, k < nok);
      }
#pragma unroll 1
      for (int j = 0; j < J; ++j) {
        const long long c0 = ((u * J + j) * (long long)N + n0) * F + f;
        const R* src = vg + c0 + (long long)slot * F;
        R* dst = vs + slab_v<PAIRS>(slot, g, j, G, JS);
#pragma unroll 1
        for (int k = 0; k < nit; ++k, src += gstep, dst += vstep) cp_async<sizeof(R)>(dst, k < nok ? src : vg + c0, k < nok);
        if (vf2g) {
          const R* fsrc = vfg + c0 + (long long)slot * F;
          R* fdst = vfs + slab_v<PAIRS>(slot, g, j, G, JS);
#pragma unroll 1
          for (int k = 0; k < nit; ++k, fsrc += gstep, fdst += vstep)
            cp_async<sizeof(R)>(fdst, k < nok ? fsrc : vfg + c0, k < nok);
        }
      }
    } else {
      for (int i = 0; i < I; ++i)
        for (int n = slot; n < NLs; n += nslots) {
          const bool ok = active && n < NLr;
          ys[slab_y<PAIRS>(n, g, i, G, RS)] = ok ? yg[((u * I + i) * (long long)N + n0 + n) * F + f] : mk<C2, R>(R(0), R(0));
        }
      for (int j = 0; j < J; ++j)
        for (int n = slot; n < NLs; n += nslots) {
          const bool ok = active && n < NLr;
          const long long off = ((u * J + j) * (long long)N + n0 + n) * F + f;
          vs[slab_v<PAIRS>(n, g, j, G, JS)] = ok ? vg[off] : R(0);
          if (vf2g) vfs[slab_v<PAIRS>(n, g, j, G, JS)] = ok ? vfg[off] : R(0);
        }
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
  cp_async_wait_all();
  if (a.packed && resident) {
    mbar_wait(&gather_bar, 0);
    if (NLs > NLr) {  // frames past this CTA's range: zero records, as the element gather leaves them
      for (int t = tid; t < (NLs - NLr) * G * RS; t += blockDim.x) {
        const int n = NLr + t / (G * RS), e = t % (G * RS);
        ys[slab_y<PAIRS>(n, e / RS, e % RS, G, RS)] = mk<C2, R>(R(0), R(0));
      }
      if (!Shape<I, JM>::ILV)
        for (int t = tid; t < (NLs - NLr) * G * JS; t += blockDim.x) {
          const int n = NLr + t / (G * JS), e = t % (G * JS);
          vs[slab_v<PAIRS>(n, e / JS, e % JS, G, JS)] = R(0);
        }
    }
  }
  __syncthreads();
  FFCA_FIXED(0)

  // ---------------- v floor per bin (fca.py:82-89 when auto) ----------------
  if (a.vf_mode == 3) {
    R psum = R(0);
    if constexpr (TM) {  // own records (zero padding adds nothing); warp-collective loads
      constexpr int TMW = 4 * I;
      for (int k = 0; k < nrec; ++k) {
        float r[TMW];
        tm_rec_ld<TMW>(tmy + k * TMW, r);
        tm_rec_wait<TMW>(r);
#pragma unroll
        for (int w = 0; w < TMW; ++w) psum = fma(R(r[w]), R(r[w]), psum);
      }
    } else if (active)
      for (int n = slot; n < NLr; n += nslots)
#pragma unroll
        for (int i = 0; i < I; ++i) {
          const C2 z = ys[slab_y<PAIRS>(n, g, i, G, RS)];
          psum += z.x * z.x + z.y * z.y;
        }
    const R pv[1] = {psum};
    bin_reduce<R, 1, G, SEG>(pv, wpart, cpart, tot, C, VMAX, parity);
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

  const bool rec = !FAST && a.ll != nullptr;
  // [P^-H] precomputed during the lambda' update (needs a second warp; not in the P-only pass)
  const bool adj_pre = I <= 4 && blockDim.x >= 64 && (FAST || !a.p_only);
  const bool vf2 = !FAST && a.vf_mode == 2;
  const int KK = FAST ? 1 : a.K;
  const int nev = 1 + 2 * a.iters;
  const R wfl = Floors<R>::weight;
  const R invI = R(1) / R(I);
  const double invN = 1.0 / double(N);
  const int rec0 = slot * G + g;          // first record of this thread
  const int rstep = nslots * G;           // records between a thread's frames (= blockDim.x)
  const int npts = active ? (NLr > slot ? (NLr - slot + nslots - 1) / nslots : 0) : 0;

  PointWork<R, I, JM, G, TM> pw;
  pw.tmy = tmy; pw.nrec = nrec;
  pw.ys = ys; pw.vs = vs; pw.vfs = vfs; pw.Pc = Pc; pw.lamc = lamc;
  pw.gslab = !resident;
  pw.g = g; pw.J = J; pw.JS = JS; pw.rec0 = rec0; pw.rstep = rstep; pw.npts = npts;
  pw.wfl = wfl; pw.invI = invI;
  {  // frame pairs: this thread's full pairs m = slot, slot + nslots, ... < NLr / 2, and the half pair
    const int np = NLr >> 1;
    pw.nfull = active ? (np > slot ? (np - slot + nslots - 1) / nslots : 0) : 0;
    pw.part = active && (NLr & 1) && slot == np % nslots;
  }

  // accumulator unit of this lane in the I > 4 phase B: a complex entry (x, y < x) of the packed
  // lower triangle, or a pair of diagonal entries (2d, 2d + 1)
  // (two units per lane: lanes l and l + 16 both hold units l and l + 16, on alternate frames)
  int bua[2] = {0, 0}, bub[2] = {0, 0};
  bool bdiag[2] = {false, false}, bown[2] = {false, false};
  if constexpr (Shape<I, JM>::GROUPB) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int u = (tid & 15) + 16 * k;
      bown[k] = u < Shape<I, JM>::NU;
      if (u < Shape<I, JM>::NCX) {
        int x = 1;
        while ((x + 1) * x / 2 <= u) ++x;
        bua[k] = x;
        bub[k] = u - x * (x - 1) / 2;
      } else if (bown[k]) {
        const int d = u - Shape<I, JM>::NCX;
        bdiag[k] = true;
        bua[k] = 2 * d;
        bub[k] = 2 * d + 1 < I ? 2 * d + 1 : 2 * d;
      }
    }
  }

  // ======================= outer iterations =======================
  FFCA_PROBE_INIT
  for (int it = 0; it < a.iters; ++it) {
    // ---------------- phase A: fused E/M sweep ----------------
    double llA = 0.0;
    if (FAST || !a.p_only) {
      pw.load_PL();
      R acc[VA];
#pragma unroll
      for (int k = 0; k < VA; ++k) acc[k] = R(0);
      const R vfl_b = R(vfl[g]);
      if constexpr (PAIRS) {
        if (rec) {
          if (vf2) pw.template phaseA_pairs<true, true>(acc, vfl_b);
          else pw.template phaseA_pairs<true, false>(acc, vfl_b);
        } else {
          if (vf2) pw.template phaseA_pairs<false, true>(acc, vfl_b);
          else pw.template phaseA_pairs<false, false>(acc, vfl_b);
        }
      } else if constexpr (PREG) {
        if (rec) {
          if (vf2) pw.template phaseA<true, true>(acc, vfl_b);
          else pw.template phaseA<true, false>(acc, vfl_b);
        } else {
          if (vf2) pw.template phaseA<false, true>(acc, vfl_b);
          else pw.template phaseA<false, false>(acc, vfl_b);
        }
      } else {
        if (rec) {
          if (vf2) pw.template phaseA2<true, true>(acc, vfl_b);
          else pw.template phaseA2<true, false>(acc, vfl_b);
        } else {
          if (vf2) pw.template phaseA2<false, true>(acc, vfl_b);
          else pw.template phaseA2<false, false>(acc, vfl_b);
        }
      }
      FFCA_PROBE(0)
      bin_reduce<R, VA, G, SEG>(acc, wpart, cpart, tot, C, VMAX, parity);
      FFCA_PROBE(1)
      if (rec && tid < G) llA = tot[tid * VMAX + VA - 1];
      // ---------------- lambda' per (bin, source) (fastfca.py:341-345) -------
      for (int t = tid; t < G * J; t += blockDim.x) {
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
      // I <= 4: the columns [P^-H]_i = conj(row i of P^-1) of the current P (from its adjugate) are
      // formed here by lanes of warp 1 while lanes of warp 0 update lambda -- P does not change
      // before the solve, so the solve itself starts from them (off the per-iteration chain)
      if constexpr (I <= 4) {
        if (adj_pre) pinvh_columns<I, G>(Pd, Pinv, ldet, a.status, group, a.total_bins, crank, rec);
      }
      __syncthreads();
      FFCA_PROBE(2)
    }

    // ---------------- phase B: weighted covariances ----------------
    pw.load_PL();
    double llB = 0.0;
    if constexpr (Shape<I, JM>::GROUPB) {
      // The last warp inverts P meanwhile (8-lane Gauss-Jordan, partial pivoting: P does not
      // change before the solve), so P^-1 is off the per-iteration critical path; the other
      // W - 1 warps share the frames.
      C2 bac[2][I];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int i = 0; i < I; ++i) bac[k][i] = mk<C2, R>(R(0), R(0));
      R lacc = R(0);
      const int warp = tid >> 5;
      if (warp == W - 1) {
        const int r = tid & 31;
        if (r < 8) invert_P_group<I>(Pd, Pinv, rhsv, r, rec, ldet, a.status, group, active && crank == 0);
      } else {
        R* wbuf = wpart + warp * 32 * Shape<I, JM>::IWS;  // free until the reduction below
        // chunk c of the bin goes to warp c % (W - 1) (measured: giving the P warp's scheduler
        // partner a double share made it the straggler)
        const int c0 = warp, cstep = W - 1;
        if (rec) pw.template phaseB_entry<true>(bac, lacc, NLr, active, wbuf, bua, bub, bdiag, c0, cstep);
        else pw.template phaseB_entry<false>(bac, lacc, NLr, active, wbuf, bua, bub, bdiag, c0, cstep);
      }
      FFCA_PROBE(3)
      if (rec) lacc = warp_sum_seg(lacc, 1);
      __syncthreads();  // every warp is done with its weight buffer (it aliases the partials)
      {
        R* wp = wpart + (tid >> 5) * VMAX;
        if ((tid & 31) < 16)  // the folded sums (lanes l + 16 hold the same)
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            if (bdiag[k]) {
#pragma unroll
              for (int i = 0; i < I; ++i) {
                wp[i * I * I + bua[k] * bua[k]] = bac[k][i].x;
                if (bub[k] != bua[k]) wp[i * I * I + bub[k] * bub[k]] = bac[k][i].y;
              }
            } else if (bown[k]) {
              const int e = bua[k] * bua[k] + 1 + 2 * bub[k];
#pragma unroll
              for (int i = 0; i < I; ++i) {
                wp[i * I * I + e] = bac[k][i].x;
                wp[i * I * I + e + 1] = bac[k][i].y;
              }
            }
          }
        if ((tid & 31) == 0) wp[I * I * I] = lacc;
      }
      bin_reduce_tail<G>(I * I * I + 1, wpart, cpart, tot, C, VMAX, parity);
      if (rec && tid < G) llB = tot[tid * VMAX + I * I * I];
    } else {
    static_assert(NCH == 1, "I <= 4 accumulates every B_i in one pass");
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
      R acc[NB + 1];
#pragma unroll
      for (int k = 0; k < NB + 1; ++k) acc[k] = R(0);
      if constexpr (PAIRS) {
        if (rec) pw.template phaseB_pairs<true>(acc);
        else pw.template phaseB_pairs<false>(acc);
      } else {
        if (rec && ch == 0) pw.template phaseB<true>(acc, ch);
        else pw.template phaseB<false>(acc, ch);
      }
      FFCA_PROBE(3)
      bin_reduce<R, NB + 1, G, SEG>(acc, wpart, cpart, tot, C, VMAX, parity);
      if (rec && ch == 0 && tid < G) llB = tot[tid * VMAX + NB];
    }
    }
    FFCA_PROBE(4)

    // ---------------- solve: P^-1 and new columns (fastfca.py:359-370) --------
    if constexpr (I <= 4) {
      // Thread (bin gg, s = 1 + i) factors B_i = L D L^H in registers, forms
      // [P^-H]_i = conj(row i of P^-1) from the adjugate (cofactors / det, each thread
      // alone: no divergent LU thread, no publication step) and solves B_i x = [P^-H]_i.
      static_assert(G * (I + 1) <= 32, "the per-bin solver threads must be lanes of one warp");
      const int s = tid % (I + 1);
      const int gg = tid / (I + 1);
      const long long b = group * G + gg;
      const bool bact = gg < G && b < a.total_bins;
      double2* Ms = Msys + gg * (I + 1) * I * I;  // LU(P) + reciprocal pivots
      int* pv = pivs + gg * (I + 1) * I;
      // I <= 3: B_i^-1 through its adjugate (a shallow dependency chain); I = 4: L D L^H
      std::conditional_t<(I <= 3), HermAdj<I>, SmallLDL<I>> ldl;
#ifdef FFCA_EXP_SKIP_SOLVE  // timing experiment only: P is never updated (results are wrong)
      if (false) {
#else
      if (bact && s > 0) {
#endif
        const int i = s - 1;
        const double* T = tot + gg * VMAX + i * I * I;  // the reduced sums, published by bin_reduce
        double2 B[I][I];
        double tr = 0.0;
        int kk = 0;
#pragma unroll
        for (int x = 0; x < I; ++x) {
          B[x][x] = make_double2(T[kk++] * invN, 0.0);
          tr += B[x][x].x;
#pragma unroll
          for (int y2 = 0; y2 < x; ++y2) {
            B[x][y2] = make_double2(T[kk] * invN, T[kk + 1] * invN);
            kk += 2;
          }
        }
        ldl.factor(B);
        if (!ldl.ok) {  // one trace-loaded retry (fastfca.py:184-194)
#pragma unroll
          for (int x = 0; x < I; ++x) B[x][x].x += 1e-10 * tr;
          ldl.factor(B);
          if (crank == 0) atomicOr(&a.status[b], ldl.ok ? ST_B_LOADED : ST_SINGULAR_B);
        }
      }
      FFCA_PROBE(5)
#ifdef FFCA_EXP_SKIP_SOLVE
      for (int k = 0; k < 0; ++k) {
#else
#pragma unroll 1
      for (int k = 0; k < KK; ++k) {
#endif
        if constexpr (I <= 4) {
          // Measured: a divergent LU thread and the LDL threads of one warp ran serially
          // (11 % of the iteration at I = 3, 13 % at I = 4).  An exactly zero determinant flags
          // SingularP, as an exactly zero LU pivot does for the structurally singular P the
          // reference rejects (zero rows / columns).
          double2 z[I], det = make_double2(0.0, 0.0);
          if (k == 0 && adj_pre) {
            if (bact && s > 0)
#pragma unroll
              for (int x = 0; x < I; ++x) z[x] = Pinv[(gg * I + s - 1) * I + x];
          } else if constexpr (I == 4) {
            // I = 4 (3x3 minors): det along column 0 from the i = 0 thread's own cofactors,
            // shuffled to the bin's other solver threads (lanes of warp 0) -- measured 8.03 ->
            // 7.92 ms at config 2; at I <= 3 recomputing column 0 per thread is faster
            if (bact && s > 0) {
              const double2* Pb = Pd + gg * I * I;
              adjugate_column<I>(Pb, s - 1, z);  // cofactors C[x][i]
              if (s == 1)
#pragma unroll
                for (int x = 0; x < I; ++x) det = cadd(det, cmul(Pb[x * I], z[x]));
            }
            const int src = ((threadIdx.x & 31) / (I + 1)) * (I + 1) + 1;
            det.x = __shfl_sync(FULL, det.x, src);
            det.y = __shfl_sync(FULL, det.y, src);
          } else if (bact && s > 0) {
            const double2* Pb = Pd + gg * I * I;
            double2 c0[I];
            adjugate_column<I>(Pb, s - 1, z);  // cofactors C[x][i]
            adjugate_column<I>(Pb, 0, c0);     // cofactors C[x][0] for det
#pragma unroll
            for (int x = 0; x < I; ++x) det = cadd(det, cmul(Pb[x * I], c0[x]));
          }
          __syncwarp();  // every column is read before any thread writes its new one
          FFCA_PROBE(6)
          if (bact && s > 0) {
            const int i = s - 1;
            if (!(k == 0 && adj_pre)) {
              if (det.x == 0.0 && det.y == 0.0) {
                if (i == 0 && crank == 0) atomicOr(&a.status[b], ST_SINGULAR_P);
              }
              if (rec && k == 0 && i == 0) ldet[gg] = log(hypot(det.x, det.y));
              const double2 rd = crecip(det);
#pragma unroll
              for (int x = 0; x < I; ++x) {  // [P^-H]_{x,i} = conj(P^-1_{i,x}) = conj(C[x][i] / det)
                const double2 t = cmul(z[x], rd);
                z[x] = make_double2(t.x, -t.y);
              }
            }
            ldl.solve(z);
#pragma unroll
            for (int x = 0; x < I; ++x) {
              Pd[(gg * I + x) * I + i] = z[x];
              Pc[(gg * I + x) * I + i] = mk<C2, R>(R(z[x].x), R(z[x].y));
            }
          }
          __syncwarp();
        }
      }
      __syncthreads();
      FFCA_PROBE(7)
    } else {
      // I > 4: thread i < I factors B_i = L D L^H in registers (Hermitian positive definite,
      // fastfca.py:184-194 loading retry) and solves B_i x = [P^-H]_i with the P^-1 the last warp
      // formed during phase B.  For K > 1 the later P^-1 come from the 8-lane group mP here.
      static_assert(G == 1, "I > 4 runs one bin per CTA");
      constexpr int mP = loop_pgroup(I);
      using LDL = PackedLDL<I>;
      double2* Lsm = Msys + tid * LDL::NP;  // this thread's factor (the solver workspace is free)
      if (tid < I) {
        const double* T = tot + tid * I * I;
        double tr = 0.0;
#pragma unroll
        for (int x = 0; x < I; ++x) tr += T[x * x];
        tr *= invN;
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          double2 b[LDL::NP];
          int kk = 0;
#pragma unroll
          for (int x = 0; x < I; ++x) {
#pragma unroll
            for (int y2 = 0; y2 < x; ++y2) b[LDL::id(x, y2)] = make_double2(T[kk + 1 + 2 * y2] * invN, T[kk + 2 + 2 * y2] * invN);
            b[LDL::id(x, x)] = make_double2(T[kk] * invN + (pass ? 1e-10 * tr : 0.0), 0.0);
            kk += 1 + 2 * x;
          }
          const bool ok = LDL::factor(b);
#pragma unroll
          for (int e = 0; e < LDL::NP; ++e) Lsm[e] = b[e];
          // one trace-loaded retry (fastfca.py:184-194)
          if (pass == 1 && active && crank == 0) atomicOr(&a.status[group], ok ? ST_B_LOADED : ST_SINGULAR_B);
          if (ok) break;
        }
      }
      FFCA_PROBE(5)
#pragma unroll 1
      for (int k = 0; k < KK; ++k) {
        if (k > 0) {
          if ((tid >> 3) == mP) invert_P_group<I>(Pd, Pinv, rhsv, tid & 7, false, ldet, a.status, group, active && crank == 0);
          __syncthreads();
        }
        if (tid < I) {
          const int i = tid;
          double2 z[I];
#pragma unroll
          for (int x = 0; x < I; ++x) {  // [P^-H]_{x,i} = conj(P^-1_{i,x})
            const double2 q = Pinv[i * I + x];
            z[x] = make_double2(q.x, -q.y);
          }
          LDL::solve(Lsm, z);
#pragma unroll
          for (int x = 0; x < I; ++x) {
            Pd[x * I + i] = z[x];
            Pc[x * I + i] = mk<C2, R>(R(z[x].x), R(z[x].y));
          }
        }
        __syncthreads();
      }
      FFCA_PROBE(7)
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
    pw.load_PL();
    R acc[1] = {R(0)};
    if constexpr (PAIRS) pw.phaseL_pairs(acc);
    else pw.phaseL(acc);
    bin_reduce<R, 1, G, SEG>(acc, wpart, cpart, tot, C, VMAX, parity);
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

  // ---------------- write back ----------------
  FFCA_FIXED(1)
  R* vo = (R*)a.v_out;
  if (active)
    for (int j = 0; j < J; ++j) {
      R* col = vo + ((u * J + j) * (long long)N + n0) * F + f;
      for (int n = slot; n < NLr; n += nslots) col[(long long)n * F] = vs[slab_v<PAIRS>(n, g, j, G, JS)];
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
  FFCA_FIXED(2)
  if constexpr (TM) {
    tmem_fence_before();
    __syncthreads();
    if (tid < 32) tmem_dealloc(tm_base_s, tmcols);
  }
  // no CTA may exit while a peer can still read its shared memory
  if (C > 1) cg::this_cluster().sync();
}

}  // namespace ffca
