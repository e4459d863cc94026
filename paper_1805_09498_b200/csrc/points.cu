// Per-(n, f) streaming kernels of the FastFCA-AS path (sm_100a).
//
// One thread per time-frequency point, frequency fastest, so every load and
// store of the reference layouts (y (U,I,N,F), v (U,J,N,F), outputs
// (U,J,N,F,I) and (U,J,I,N,F)) is coalesced across a warp.  These are pure
// HBM-streaming kernels: per-bin matrices (P, P^-H, lambda) are read through
// L1/L2, which hold them for all frames of a bin.
#include <cmath>

#include "common.cuh"
#include "host_common.h"
#include "points.h"

namespace ffca {

template <typename R, int I>
__global__ void __launch_bounds__(256) point_kernel(const PointArgs a) {
  using C2 = typename Cpx<R>::T;
  const long long npts = (long long)a.U * a.N * a.F;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= npts) return;
  const int F = a.F, N = a.N, J = a.J;
  const int f = int(t % F);
  const long long un = t / F;
  const int n = int(un % N);
  const long long u = un / N;
  const long long bin = u * F + f;
  const R wfl = Floors<R>::weight;

  if (a.mode == PM_BACK) {
    const double2* Q = (const double2*)a.Q + bin * I * I;
    const C2* mu = (const C2*)a.y;
    C2* out = (C2*)a.out0;
    for (int j = 0; j < J; ++j) {
      const long long base = (((u * J + j) * N + n) * (long long)F + f) * I;
      C2 m[I];
#pragma unroll
      for (int i = 0; i < I; ++i) m[i] = mu[base + i];
#pragma unroll
      for (int x = 0; x < I; ++x) {
        double re = 0.0, im = 0.0;
#pragma unroll
        for (int b = 0; b < I; ++b) {
          const double2 q = Q[x * I + b];
          re += q.x * double(m[b].x) - q.y * double(m[b].y);
          im += q.x * double(m[b].y) + q.y * double(m[b].x);
        }
        const C2 r = mk<C2, R>(R(re), R(im));
        if (a.images_layout)
          out[(((u * J + j) * I + x) * (long long)N + n) * F + f] = r;
        else
          out[base + x] = r;
      }
    }
    return;
  }

  // transformed observation y_t = P^H y (or given)
  C2 yt[I];
  if (a.mode == PM_STATS || a.mode == PM_TRANSFORM || a.mode == PM_IMAGES) {
    const C2* y = (const C2*)a.y;
    const C2* P = (const C2*)a.P + bin * I * I;
    C2 yv[I];
#pragma unroll
    for (int i = 0; i < I; ++i) yv[i] = y[((u * I + i) * N + n) * (long long)F + f];
#pragma unroll
    for (int b = 0; b < I; ++b) {
      C2 acc = mk<C2, R>(R(0), R(0));
#pragma unroll
      for (int x = 0; x < I; ++x) cmac_conj(acc, P[x * I + b], yv[x]);
      yt[b] = acc;
    }
    if (a.mode == PM_TRANSFORM) {
      C2* out = (C2*)a.out0;
#pragma unroll
      for (int b = 0; b < I; ++b) out[t * I + b] = yt[b];
      return;
    }
  } else if (a.mode == PM_ESTEP_YT) {
    const C2* y = (const C2*)a.y;
#pragma unroll
    for (int b = 0; b < I; ++b) yt[b] = y[t * I + b];
  }

  // mixture weights
  const R* v = (const R*)a.v;
  const R* lam = (const R*)a.lam;
  R w[I];
#pragma unroll
  for (int i = 0; i < I; ++i) w[i] = R(0);
  for (int j = 0; j < J; ++j) {
    const R vj = v[((u * J + j) * N + n) * (long long)F + f];
#pragma unroll
    for (int i = 0; i < I; ++i) w[i] = fma(vj, lam[((u * J + j) * F + f) * I + i], w[i]);
  }
#pragma unroll
  for (int i = 0; i < I; ++i) w[i] = fmax(w[i], wfl);
  if (a.mode == PM_WEIGHTS) {
    R* out = (R*)a.out0;
#pragma unroll
    for (int i = 0; i < I; ++i) out[t * I + i] = w[i];
    return;
  }

  const double2* Q = a.mode == PM_IMAGES ? (const double2*)a.Q + bin * I * I : nullptr;
  for (int j = 0; j < J; ++j) {
    const R vj = v[((u * J + j) * N + n) * (long long)F + f];
    const long long base = (((u * J + j) * N + n) * (long long)F + f) * I;
    C2 mu[I];
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const R aa = vj * lam[((u * J + j) * F + f) * I + i];
      const R g = quot(aa, w[i]);
      mu[i] = mk<C2, R>(g * yt[i].x, g * yt[i].y);
      if (a.mode != PM_IMAGES) {
        if (a.out0) ((C2*)a.out0)[base + i] = mu[i];
        if (a.out1) ((R*)a.out1)[base + i] = fmax(aa * (R(1) - g), R(0));
      }
    }
    if (a.mode == PM_IMAGES) {
      C2* out = (C2*)a.out0;
#pragma unroll
      for (int x = 0; x < I; ++x) {
        double re = 0.0, im = 0.0;
#pragma unroll
        for (int b = 0; b < I; ++b) {
          const double2 q = Q[x * I + b];
          re += q.x * double(mu[b].x) - q.y * double(mu[b].y);
          im += q.x * double(mu[b].y) + q.y * double(mu[b].x);
        }
        out[(((u * J + j) * I + x) * (long long)N + n) * F + f] = mk<C2, R>(R(re), R(im));
      }
    }
  }
}

// Statistics refresh / Wiener images for I <= 4, bin-tiled: a CTA owns 32 consecutive bins of
// one mixture (lane = bin, so every (i, n) row access is one coalesced 32-bin segment) and its 8
// warps stride over the frames.  The per-bin constants P, lambda (and Q = P^-H for the images)
// are loaded into registers once per thread instead of once per point, Q in the compute type.
// Per point: y_t = P^H y, w = sum_j v_j lambda_j, then per source g = v lambda / w,
// mu_t = g y_t, phi_t = max(v lambda (1 - g), 0)  (fastfca.py:373-387), or the image
// x_j = Q mu_t written straight into (U, J, I, N, F)  (wiener.py:38-43).
constexpr int TILE_F = 32, TILE_WARPS = 8;
// Tile stride along the bins.  With an odd F no 32-bin tile of a row starts on a 32-byte sector,
// so adjacent tiles would both write (part of) the sector at their boundary -- partial-sector
// writes the L2 has to merge.  Images tiles therefore overlap by EPS - 1 bins (EPS = elements per
// 32-byte sector): every sector of a row lies wholly inside some tile, and the tile whose
// exclusive range [f0, f0 + stride) holds the sector's first bin writes it whole.
// (complex64 images; measured at config-3 scale 2.10 -> 1.97 ms.  Not for complex128, where a
// sector holds only two elements: 1.33 -> 1.41 ms.)
template <typename R, int MODE>
constexpr int tile_stride() {
  return (MODE == PM_IMAGES && sizeof(R) == 4) ? TILE_F - (32 / (2 * int(sizeof(R))) - 1) : TILE_F;
}
// frames in flight per warp: as many ring stages as fit ~46 KB of static shared memory (<= 4)
template <typename R, int I>
constexpr int tile_depth() {
  constexpr int d = 46 * 1024 / (TILE_WARPS * TILE_F * (2 * I + 4) * int(sizeof(R)));
  return d > 4 ? 4 : (d < 1 ? 1 : d);
}

template <typename R, int I, int MODE>
__global__ void __launch_bounds__(TILE_F* TILE_WARPS, 2) point_tile_kernel(const PointArgs a, int frames_per_cta) {
  using C2 = typename Cpx<R>::T;
  constexpr int JMAX = 4;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int F = a.F, N = a.N, J = a.J;
  constexpr int TS = tile_stride<R, MODE>();
  constexpr int EPS = 32 / int(sizeof(C2));  // output elements per 32-byte sector
  const int ftiles = (F + TS - 1) / TS;
  const long long u = blockIdx.x / ftiles;
  const int f0 = int(blockIdx.x % ftiles) * TS;
  const bool last_tile = f0 + TS >= F;
  const bool live = f0 + lane < F;  // dead lanes of a partial tile compute on a clamped bin, store nothing
  const int f = live ? f0 + lane : F - 1;
  const long long bin = u * F + f;
  const R wfl = Floors<R>::weight;
  C2 Pm[I][I];
  const C2* Pg = (const C2*)a.P + bin * I * I;
#pragma unroll
  for (int x = 0; x < I; ++x)
#pragma unroll
    for (int b = 0; b < I; ++b) Pm[x][b] = Pg[x * I + b];
  R lam[JMAX][I];
#pragma unroll
  for (int j = 0; j < JMAX; ++j)
#pragma unroll
    for (int i = 0; i < I; ++i) lam[j][i] = j < J ? ((const R*)a.lam)[((u * J + j) * F + f) * I + i] : R(0);
  C2 Qm[MODE == PM_IMAGES ? I : 1][MODE == PM_IMAGES ? I : 1];
  if constexpr (MODE == PM_IMAGES) {
    const double2* Qg = (const double2*)a.Q + bin * I * I;
#pragma unroll
    for (int x = 0; x < I; ++x)
#pragma unroll
      for (int b = 0; b < I; ++b) {
        const double2 q = Qg[x * I + b];
        Qm[x][b] = mk<C2, R>(R(q.x), R(q.y));
      }
  }
  const long long rowN = (long long)N * F;  // stride between channels / sources
  const C2* __restrict__ yb = (const C2*)a.y + u * I * rowN;
  const R* __restrict__ vb = (const R*)a.v + u * J * rowN;
  constexpr int TILE_D = tile_depth<R, I>();
  const int nlive = (F - f0) < TILE_F ? (F - f0) : TILE_F;  // bins of this tile
  // the kernel is load-latency-bound: each warp keeps TILE_D frames of y and v in flight with
  // cp.async into a per-warp shared-memory ring (each lane reads back only what it copied)
  // stats: a warp's mu_t (phi_t) for one (source, frame) is one contiguous run of 32*I complex
  // (reals) in the (..., F, I) layout; it is staged in the ring slot just consumed (y part for
  // mu, v part for phi: I <= JMAX) and written back as 16-byte vectors, so every store
  // instruction covers whole sectors.  The slot is refilled only by the next iteration's issue.
  __shared__ __align__(16) C2 ry[TILE_WARPS][TILE_D][I][TILE_F];
  __shared__ __align__(16) R rv[TILE_WARPS][TILE_D][JMAX][TILE_F];
  // frames [n_lo, n_hi) of this CTA (blockIdx.y; frames_per_cta is a multiple of TILE_WARPS): a single
  // long mixture would otherwise run on F / 32 CTAs only (config-2 shape: 33 CTAs on 148 SMs)
  const int n_lo = blockIdx.y * frames_per_cta;
  const int n_cnt = (n_lo + frames_per_cta < N ? frames_per_cta : N - n_lo);
  const int nfr = n_cnt > wp ? (n_cnt - wp + TILE_WARPS - 1) / TILE_WARPS : 0;  // frames of this warp
  if constexpr (MODE == PM_IMAGES && sizeof(R) == 4) {
    // complex64 images.  Measured: the generic loop below spends 59 % of its 467 SASS instructions per
    // frame on integer work -- 64-bit indices re-derived for every load and store, and the sector
    // ownership test per output element.  Here offsets inside one mixture are 32-bit (launch_points
    // checks J * I * I * N * F < 2^31) and carried as one running element offset, every address is a
    // single multiply-add on a mixture base kept opaque to the compiler (it otherwise re-derives the
    // base from the kernel parameters at each use), and the ownership of the J * I output planes is a
    // bit mask formed once: a warp's frames are TILE_WARPS rows apart, a multiple of the elements per
    // sector, so the alignment of its stores within a plane is the same for every frame.
    // 274 instructions per frame; config-3 scale 1.97 -> 1.69 ms.  (The same form measured slower
    // for the statistics, 2.74 vs 2.50 ms, and for complex128 images, 1.38 vs 1.33 ms.)
    static_assert(TILE_WARPS % 8 == 0, "a warp's frames keep their sector alignment");
    const int rowNi = int(rowN);
    const C2* ybo = yb;
    const R* vbo = vb;
    C2* outu = (C2*)a.out0 + u * J * I * rowN;  // this mixture's images
    asm volatile("" : "+l"(ybo), "+l"(vbo), "+l"(outu));
    const int ostep = TILE_WARPS * F;  // elements between a warp's consecutive frames
    int oi = (n_lo + wp) * F + f, ki = 0;  // next frame to request: element offset in a plane, index
    auto issue = [&]() {
      const bool ok = ki < nfr;
      const int o = ok ? oi : 0;
      const int sl = ki % TILE_D;
#pragma unroll
      for (int i = 0; i < I; ++i) cp_async<sizeof(C2)>(&ry[wp][sl][i][lane], ybo + (i * rowNi + o), ok);
#pragma unroll
      for (int j = 0; j < JMAX; ++j)
        if (j < J) cp_async<sizeof(R)>(&rv[wp][sl][j][lane], vbo + (j * rowNi + o), ok);
      cp_async_commit();
      ++ki;
      oi += ostep;
    };
    unsigned ownmask = 0;
#pragma unroll
    for (int p = 0; p < JMAX * I; ++p) {
      const long long e = (u * J * I + p) * rowN + (long long)(n_lo + wp) * F + f;  // this thread's first element of plane p
      // first bin of this element's 32-byte sector; the tile owning that bin writes the sector
      const int b0 = f - int(e & (EPS - 1));
      const bool own = live && (TS == TILE_F || ((b0 >= f0 || f0 == 0) && (b0 < f0 + TS || last_tile)));
      ownmask |= unsigned(own) << p;
    }
    int oc = (n_lo + wp) * F + f;  // element offset (in a plane) of the frame being consumed
#pragma unroll
    for (int k = 0; k < TILE_D - 1; ++k) issue();
#pragma unroll 1
    for (int k = 0; k < nfr; ++k, oc += ostep) {
      issue();
      cp_async_wait<TILE_D - 1>();
      const int sl = k % TILE_D;
      C2 yv[I];
#pragma unroll
      for (int i = 0; i < I; ++i) yv[i] = ry[wp][sl][i][lane];
      R vj[JMAX];
#pragma unroll
      for (int j = 0; j < JMAX; ++j) vj[j] = j < J ? rv[wp][sl][j][lane] : R(0);
      C2 yt[I];  // P^H y as pair arithmetic (FFMA2)
#pragma unroll
      for (int b = 0; b < I; ++b) {
        C2 acc = mk<C2, R>(R(0), R(0));
#pragma unroll
        for (int x = 0; x < I; ++x) {
          acc = fma2(yv[x], bc2<R>(Pm[x][b].x), acc);                          // p.x (y.x, y.y)
          acc = fma2(mk<C2, R>(yv[x].y, -yv[x].x), bc2<R>(Pm[x][b].y), acc);  // p.y (y.y, -y.x)
        }
        yt[b] = acc;
      }
      R iw[I];
#pragma unroll
      for (int i = 0; i < I; ++i) {
        R w = R(0);
#pragma unroll
        for (int j = 0; j < JMAX; ++j)
          if (j < J) w = fma(vj[j], lam[j][i], w);
        iw[i] = rcp(fmax(w, wfl));
      }
#pragma unroll
      for (int j = 0; j < JMAX; ++j) {
        if (j >= J) continue;
        C2 mu[I];
#pragma unroll
        for (int i = 0; i < I; ++i) {
          const R g = (vj[j] * lam[j][i]) * iw[i];
          mu[i] = fma2(yt[i], bc2<R>(g), mk<C2, R>(R(0), R(0)));
        }
#pragma unroll
        for (int x = 0; x < I; ++x) {
          C2 acc = mk<C2, R>(R(0), R(0));
#pragma unroll
          for (int b = 0; b < I; ++b) {  // acc += Q[x][b] mu[b] = q.x (mu.x, mu.y) + q.y (-mu.y, mu.x)
            acc = fma2(mu[b], bc2<R>(Qm[x][b].x), acc);
            acc = fma2(mk<C2, R>(-mu[b].y, mu[b].x), bc2<R>(Qm[x][b].y), acc);
          }
          if ((ownmask >> (j * I + x)) & 1) outu[(j * I + x) * rowNi + oc] = acc;
        }
      }
    }
  } else {
    auto issue = [&](int k) {
      const int n = n_lo + wp + k * TILE_WARPS;
      const bool ok = k < nfr;
      const long long o = ok ? (long long)n * F + f : 0;
      const int sl = k % TILE_D;
#pragma unroll
      for (int i = 0; i < I; ++i) cp_async<sizeof(C2)>(&ry[wp][sl][i][lane], yb + i * rowN + o, ok);
#pragma unroll
      for (int j = 0; j < JMAX; ++j)
        if (j < J) cp_async<sizeof(R)>(&rv[wp][sl][j][lane], vb + j * rowN + o, ok);
      cp_async_commit();
    };
#pragma unroll
    for (int k = 0; k < TILE_D - 1; ++k) issue(k);
#pragma unroll 1
    for (int k = 0; k < nfr; ++k) {
      issue(k + TILE_D - 1);
      cp_async_wait<TILE_D - 1>();
      const int n = n_lo + wp + k * TILE_WARPS;
      const int sl = k % TILE_D;
      const long long off = (long long)n * F + f;
      C2 yv[I];
#pragma unroll
      for (int i = 0; i < I; ++i) yv[i] = ry[wp][sl][i][lane];
      R vj[JMAX];
#pragma unroll
      for (int j = 0; j < JMAX; ++j) vj[j] = j < J ? rv[wp][sl][j][lane] : R(0);
      C2 yt[I];  // P^H y as pair arithmetic (FFMA2 in fp32)
#pragma unroll
      for (int b = 0; b < I; ++b) {
        C2 acc = mk<C2, R>(R(0), R(0));
#pragma unroll
        for (int x = 0; x < I; ++x) {
          acc = fma2(yv[x], bc2<R>(Pm[x][b].x), acc);                          // p.x (y.x, y.y)
          acc = fma2(mk<C2, R>(yv[x].y, -yv[x].x), bc2<R>(Pm[x][b].y), acc);  // p.y (y.y, -y.x)
        }
        yt[b] = acc;
      }
      R iw[I];
#pragma unroll
      for (int i = 0; i < I; ++i) {
        R w = R(0);
#pragma unroll
        for (int j = 0; j < JMAX; ++j)
          if (j < J) w = fma(vj[j], lam[j][i], w);
        iw[i] = rcp(fmax(w, wfl));
      }
#pragma unroll
      for (int j = 0; j < JMAX; ++j) {
        if (j >= J) continue;
        C2 mu[I];
        R ph[I];
#pragma unroll
        for (int i = 0; i < I; ++i) {
          const R aa = vj[j] * lam[j][i];
          const R g = aa * iw[i];
          mu[i] = fma2(yt[i], bc2<R>(g), mk<C2, R>(R(0), R(0)));
          ph[i] = fmax(aa * (R(1) - g), R(0));
        }
        if constexpr (MODE == PM_STATS) {
          const long long base = ((u * J + j) * rowN + (long long)n * F + f0) * I;  // first element of the run
          // The run starts on a 16-byte boundary for one frame in two (mu, complex64) / four (phi,
          // fp32) only (odd F, I = 3), and ncu showed the element-wise fallback of the other runs
          // as a third of the kernel's instructions.  So a run is staged SHIFTED: its h elements before
          // the first 16-byte boundary (h < 16 / element size; they belong to the first lanes) are
          // stored straight from registers, element e >= h goes to stage[e - h], and the aligned body
          // leaves as 16-byte vectors (fixed trip count, predicated) with a ragged tail of < 16 bytes.
          C2* stage_mu = &ry[wp][sl][0][0];
          R* stage_phi = &rv[wp][sl][0][0];
          const int ne = nlive * I;  // complex (real) elements of this run
          C2* omu = a.out0 ? (C2*)a.out0 + base : nullptr;
          R* oph = a.out1 ? (R*)a.out1 + base : nullptr;
          constexpr int PM = 16 / int(sizeof(C2)), PP = 16 / int(sizeof(R));  // elements per 16-byte vector
          const int hm = int(((16 - (reinterpret_cast<uintptr_t>(omu) & 15)) & 15) / sizeof(C2));
          const int hp = int(((16 - (reinterpret_cast<uintptr_t>(oph) & 15)) & 15) / sizeof(R));
          __syncwarp();  // every lane has read this slot's y / v (and the previous source's run)
#pragma unroll
          for (int i = 0; i < I; ++i) {
            const int e = lane * I + i;
            if (e >= hm) stage_mu[e - hm] = mu[i];
            else if (omu && e < ne) omu[e] = mu[i];
            if (e >= hp) stage_phi[e - hp] = ph[i];
            else if (oph && e < ne) oph[e] = ph[i];
          }
          __syncwarp();
          if (omu) {
            const int nb = ne > hm ? ne - hm : 0, nv = nb / PM, r = nb - nv * PM;
            float4* o = reinterpret_cast<float4*>(omu + hm);
            constexpr int IT = (I * TILE_F / PM + 31) / 32;  // fixed trip count: compact predicated code
#pragma unroll
            for (int t = 0; t < IT; ++t) {
              const int e = lane + 32 * t;
              if (e < nv) o[e] = reinterpret_cast<const float4*>(stage_mu)[e];
            }
            if (lane < r) omu[hm + nv * PM + lane] = stage_mu[nv * PM + lane];
          }
          if (oph) {
            const int nb = ne > hp ? ne - hp : 0, nv = nb / PP, r = nb - nv * PP;
            float4* o = reinterpret_cast<float4*>(oph + hp);
            constexpr int IT = (I * TILE_F / PP + 31) / 32;
#pragma unroll
            for (int t = 0; t < IT; ++t) {
              const int e = lane + 32 * t;
              if (e < nv) o[e] = reinterpret_cast<const float4*>(stage_phi)[e];
            }
            if (lane < r) oph[hp + nv * PP + lane] = stage_phi[nv * PP + lane];
          }
          __syncwarp();
        } else {
          const long long e_row = (u * J + j) * I * rowN + off;  // element index of (j, x = 0, n, f)
          C2* __restrict__ out = (C2*)a.out0 + e_row;
#pragma unroll
          for (int x = 0; x < I; ++x) {
            // first bin of this element's 32-byte sector; the tile owning that bin writes the sector
            const int b0 = f - int((e_row + x * rowN) & (EPS - 1));
            const bool own = live && (TS == TILE_F || ((b0 >= f0 || f0 == 0) && (b0 < f0 + TS || last_tile)));
            C2 acc = mk<C2, R>(R(0), R(0));
#pragma unroll
            for (int b = 0; b < I; ++b) {  // acc += Q[x][b] mu[b] = q.x (mu.x, mu.y) + q.y (-mu.y, mu.x)
              acc = fma2(mu[b], bc2<R>(Qm[x][b].x), acc);
              acc = fma2(mk<C2, R>(-mu[b].y, mu[b].x), bc2<R>(Qm[x][b].y), acc);
            }
            if (own) out[x * rowN] = acc;
          }
        }
      }
    }
  }
}

// Statistics refresh / Wiener images for 4 < I <= 8, bin-tiled.  The per-bin constants no longer fit
// registers (P and Q = P^-H are I x I complex each), so the CTA keeps them for its 32 bins in shared
// memory, element-major with the bin fastest ([x * I + b][lane]: every lane reads its own bin's
// element, conflict free), converted to the compute type once.  A CTA owns 32 consecutive bins x a
// block of frames (blockIdx.y), its 8 warps stride the frames two at a time so that every P / Q /
// lambda element read from shared memory feeds two points.  Statistics leave as each lane's I
// consecutive elements of the (..., F, I) layout (16-byte vectors when I is even), images as
// coalesced 32-bin rows of each (source, channel) plane.
// (The untiled point_kernel re-read the fp64 Q of its bin from global memory for every point and
// back-solved in fp64: config-4 shape images 13.8 ms, statistics 4.8 ms.)
template <typename R, int I, int MODE>
__global__ void __launch_bounds__(256) point_tile_big_kernel(const PointArgs a, int frames_per_cta) {
  using C2 = typename Cpx<R>::T;
  constexpr int JMAX = 8;
  extern __shared__ __align__(16) unsigned char big_sm[];
  C2* Ps = (C2*)big_sm;
  C2* Qs = Ps + I * I * 32;
  R* Ls = (R*)(Qs + (MODE == PM_IMAGES ? I * I * 32 : 0));
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int F = a.F, N = a.N, J = a.J;
  const int ftiles = (F + 31) / 32;
  const long long u = blockIdx.x / ftiles;
  const int f0 = int(blockIdx.x % ftiles) * 32;
  const int n_lo = blockIdx.y * frames_per_cta;
  const int n_hi = n_lo + frames_per_cta < N ? n_lo + frames_per_cta : N;
  const bool live = f0 + lane < F;
  const int f = live ? f0 + lane : F - 1;
  // per-bin constants of the tile -> shared memory (global reads coalesced over a bin's elements)
  for (int e = threadIdx.x; e < 32 * I * I; e += blockDim.x) {
    const int lb = e / (I * I), el = e % (I * I);
    const int fb = f0 + lb < F ? f0 + lb : F - 1;
    Ps[el * 32 + lb] = ((const C2*)a.P)[(u * F + fb) * I * I + el];
    if constexpr (MODE == PM_IMAGES) {
      const double2 q = ((const double2*)a.Q)[(u * F + fb) * I * I + el];
      Qs[el * 32 + lb] = mk<C2, R>(R(q.x), R(q.y));
    }
  }
  for (int e = threadIdx.x; e < 32 * J * I; e += blockDim.x) {
    const int lb = e / (J * I), el = e % (J * I);  // el = j * I + i
    const int fb = f0 + lb < F ? f0 + lb : F - 1;
    Ls[el * 32 + lb] = ((const R*)a.lam)[((u * J + el / I) * F + fb) * I + el % I];
  }
  __syncthreads();
  const R wfl = Floors<R>::weight;
  const long long rowN = (long long)N * F;
  const C2* __restrict__ yb = (const C2*)a.y + u * I * rowN;
  const R* __restrict__ vb = (const R*)a.v + u * J * rowN;
  // frames per step and warp: two where the registers allow (complex64 statistics), else one
  constexpr int FP = (sizeof(R) == 4 && MODE == PM_STATS) ? 2 : 1;
#pragma unroll 1
  for (int n = n_lo + FP * wp; n < n_hi; n += 8 * FP) {
    long long o[FP];
    bool ok[FP];
#pragma unroll
    for (int r = 0; r < FP; ++r) {
      ok[r] = n + r < n_hi;  // a missing second frame is computed on the first one again, not stored
      o[r] = (long long)(ok[r] ? n + r : n) * F + f;
    }
    C2 y[FP][I], t[FP][I];  // y, y_t = P^H y
#pragma unroll
    for (int r = 0; r < FP; ++r)
#pragma unroll
      for (int i = 0; i < I; ++i) {
        y[r][i] = yb[i * rowN + o[r]];
        t[r][i] = mk<C2, R>(R(0), R(0));
      }
#pragma unroll
    for (int x = 0; x < I; ++x)
#pragma unroll
      for (int b = 0; b < I; ++b) {
        const C2 pe = Ps[(x * I + b) * 32 + lane];
#pragma unroll
        for (int r = 0; r < FP; ++r) {  // t += conj(p) y = p.x (y.x, y.y) + p.y (y.y, -y.x): two packed FMAs
          t[r][b] = fma2(y[r][x], bc2<R>(pe.x), t[r][b]);
          t[r][b] = fma2(mk<C2, R>(y[r][x].y, -y[r][x].x), bc2<R>(pe.y), t[r][b]);
        }
      }
    R w[FP][I];
#pragma unroll
    for (int r = 0; r < FP; ++r)
#pragma unroll
      for (int i = 0; i < I; ++i) w[r][i] = R(0);
    for (int j = 0; j < J; ++j) {
      R v[FP];
#pragma unroll
      for (int r = 0; r < FP; ++r) v[r] = vb[j * rowN + o[r]];
#pragma unroll
      for (int i = 0; i < I; ++i) {
        const R l = Ls[(j * I + i) * 32 + lane];
#pragma unroll
        for (int r = 0; r < FP; ++r) w[r][i] = fma(v[r], l, w[r][i]);
      }
    }
#pragma unroll
    for (int r = 0; r < FP; ++r)
#pragma unroll
      for (int i = 0; i < I; ++i) w[r][i] = fmax(w[r][i], wfl);
    for (int j = 0; j < J; ++j) {
      R v[FP];
#pragma unroll
      for (int r = 0; r < FP; ++r) v[r] = vb[j * rowN + o[r]];
      C2 m[FP][I];
      R ph[FP][I];
#pragma unroll
      for (int i = 0; i < I; ++i) {
        const R l = Ls[(j * I + i) * 32 + lane];
#pragma unroll
        for (int r = 0; r < FP; ++r) {
          // phi = a (1 - a / w) as a (w - a) / w: exact 0 for a single source (w = a), where
          // 1 - a * (1 / w) would leave the reciprocal's rounding error (the reference divides)
          const R aa = v[r] * l;
          const R iw = rcp(w[r][i]);
          const R g = aa * iw;
          m[r][i] = fma2(t[r][i], bc2<R>(g), mk<C2, R>(R(0), R(0)));
          ph[r][i] = fmax(aa * (w[r][i] - aa) * iw, R(0));
        }
      }
      if constexpr (MODE == PM_STATS) {
#pragma unroll
        for (int r = 0; r < FP; ++r) {
          if (!(live && ok[r])) continue;
          const long long base = ((u * J + j) * rowN + o[r]) * I;
          if (a.out0) {
            C2* d = (C2*)a.out0 + base;
            if constexpr (sizeof(C2) == 8 && I % 2 == 0) {  // I complex64 = I / 2 aligned 16-byte vectors
#pragma unroll
              for (int i = 0; i < I; i += 2)
                reinterpret_cast<float4*>(d)[i / 2] = make_float4(float(m[r][i].x), float(m[r][i].y), float(m[r][i + 1].x), float(m[r][i + 1].y));
            } else {
#pragma unroll
              for (int i = 0; i < I; ++i) d[i] = m[r][i];
            }
          }
          if (a.out1) {
            R* d = (R*)a.out1 + base;
            if constexpr (sizeof(R) == 4 && I % 4 == 0) {
#pragma unroll
              for (int i = 0; i < I; i += 4)
                reinterpret_cast<float4*>(d)[i / 4] = make_float4(float(ph[r][i]), float(ph[r][i + 1]), float(ph[r][i + 2]), float(ph[r][i + 3]));
            } else {
#pragma unroll
              for (int i = 0; i < I; ++i) d[i] = ph[r][i];
            }
          }
        }
      } else {
        C2* __restrict__ out = (C2*)a.out0 + (u * J + j) * I * rowN;
#pragma unroll 1  // (fully unrolled, the compiler hoists all I * I Q loads and spills)
        for (int x = 0; x < I; ++x) {
          C2 acc[FP];
#pragma unroll
          for (int r = 0; r < FP; ++r) acc[r] = mk<C2, R>(R(0), R(0));
#pragma unroll
          for (int b = 0; b < I; ++b) {  // acc += Q[x][b] mu[b]
            const C2 q = Qs[(x * I + b) * 32 + lane];
#pragma unroll
            for (int r = 0; r < FP; ++r) {  // q mu = q.x (mu.x, mu.y) + q.y (-mu.y, mu.x)
              acc[r] = fma2(m[r][b], bc2<R>(q.x), acc[r]);
              acc[r] = fma2(mk<C2, R>(-m[r][b].y, m[r][b].x), bc2<R>(q.y), acc[r]);
            }
          }
#pragma unroll
          for (int r = 0; r < FP; ++r)
            if (live && ok[r]) out[x * rowN + o[r]] = acc[r];
        }
      }
    }
  }
}

// Back-transform x_j = Q mu_tilde_j, Q = P^-H (fastfca.py:258-273; the device pass of
// wiener.mmse_images_fastfca, wiener.py:38-43), bin-tiled for every I <= 8: a CTA owns 32 consecutive
// bins x a block of frames, Q of its bins sits in shared memory in the compute type (element-major,
// bin fastest: conflict free), its 8 warps stride the frames.  Per (frame, source) a lane reads its
// bin's I consecutive transformed means -- the warp's 32 runs are one contiguous piece of the
// (U, J, N, F, I) array -- with the next source's means already in flight, and writes either
// coalesced 32-bin rows of the (U, J, I, N, F) image planes or its I consecutive outputs.
// (The untiled point_kernel re-read the fp64 Q from global memory per point and solved in fp64:
// config-3 scale 3.05 ms, config-4 shape 11.98 ms.)
template <typename R, int I>
__global__ void __launch_bounds__(256) back_tile_kernel(const PointArgs a, int frames_per_cta) {
  using C2 = typename Cpx<R>::T;
  extern __shared__ __align__(16) unsigned char back_sm[];
  C2* Qs = (C2*)back_sm;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int F = a.F, N = a.N, J = a.J;
  const int ftiles = (F + 31) / 32;
  const long long u = blockIdx.x / ftiles;
  const int f0 = int(blockIdx.x % ftiles) * 32;
  const int n_lo = blockIdx.y * frames_per_cta;
  const int n_hi = n_lo + frames_per_cta < N ? n_lo + frames_per_cta : N;
  const bool live = f0 + lane < F;
  const int f = live ? f0 + lane : F - 1;
  for (int e = threadIdx.x; e < 32 * I * I; e += blockDim.x) {
    const int lb = e / (I * I), el = e % (I * I);
    const int fb = f0 + lb < F ? f0 + lb : F - 1;
    const double2 q = ((const double2*)a.Q)[(u * F + fb) * I * I + el];
    Qs[el * 32 + lb] = mk<C2, R>(R(q.x), R(q.y));
  }
  __syncthreads();
  const long long rowN = (long long)N * F;
  const C2* __restrict__ mu = (const C2*)a.y + u * J * rowN * I;
  C2* __restrict__ out = (C2*)a.out0 + u * J * rowN * I;
  auto load = [&](int j, long long o, C2 (&m)[I]) {  // the lane's I consecutive means of source j at point o
    const C2* src = mu + (j * rowN + o) * I;
    if constexpr (sizeof(C2) == 8 && I % 2 == 0) {
#pragma unroll
      for (int i = 0; i < I; i += 2) {
        const float4 t = reinterpret_cast<const float4*>(src)[i / 2];
        m[i] = mk<C2, R>(R(t.x), R(t.y));
        m[i + 1] = mk<C2, R>(R(t.z), R(t.w));
      }
    } else {
#pragma unroll
      for (int i = 0; i < I; ++i) m[i] = src[i];
    }
  };
#pragma unroll 1
  for (int n = n_lo + wp; n < n_hi; n += 8) {
    const long long o = (long long)n * F + f;
    C2 cur[I], nxt[I];
    load(0, o, cur);
#pragma unroll 1
    for (int j = 0; j < J; ++j) {
      if (j + 1 < J) load(j + 1, o, nxt);
      C2 x[I];
#pragma unroll
      for (int r = 0; r < I; ++r) {
        C2 acc = mk<C2, R>(R(0), R(0));
#pragma unroll
        for (int b = 0; b < I; ++b) {  // acc += Q[r][b] mu[b] = q.x (mu.x, mu.y) + q.y (-mu.y, mu.x)
          const C2 q = Qs[(r * I + b) * 32 + lane];
          acc = fma2(cur[b], bc2<R>(q.x), acc);
          acc = fma2(mk<C2, R>(-cur[b].y, cur[b].x), bc2<R>(q.y), acc);
        }
        x[r] = acc;
      }
      if (live) {
        if (a.images_layout) {
          C2* d = out + (long long)j * I * rowN + o;
#pragma unroll
          for (int r = 0; r < I; ++r) d[r * rowN] = x[r];
        } else {
          C2* d = out + (j * rowN + o) * I;
          if constexpr (sizeof(C2) == 8 && I % 2 == 0) {
#pragma unroll
            for (int r = 0; r < I; r += 2)
              reinterpret_cast<float4*>(d)[r / 2] = make_float4(float(x[r].x), float(x[r].y), float(x[r + 1].x), float(x[r + 1].y));
          } else {
#pragma unroll
            for (int r = 0; r < I; ++r) d[r] = x[r];
          }
        }
      }
#pragma unroll
      for (int i = 0; i < I; ++i) cur[i] = nxt[i];
    }
  }
}

template <typename R>
static void* back_tile_fn(int I) {
  switch (I) {
    case 1: return (void*)back_tile_kernel<R, 1>;
    case 2: return (void*)back_tile_kernel<R, 2>;
    case 3: return (void*)back_tile_kernel<R, 3>;
    case 4: return (void*)back_tile_kernel<R, 4>;
    case 5: return (void*)back_tile_kernel<R, 5>;
    case 6: return (void*)back_tile_kernel<R, 6>;
    case 7: return (void*)back_tile_kernel<R, 7>;
    case 8: return (void*)back_tile_kernel<R, 8>;
  }
  return nullptr;
}

template <typename R, int MODE>
static void* big_tile_fn(int I) {
  switch (I) {
    case 5: return (void*)point_tile_big_kernel<R, 5, MODE>;
    case 6: return (void*)point_tile_big_kernel<R, 6, MODE>;
    case 7: return (void*)point_tile_big_kernel<R, 7, MODE>;
    case 8: return (void*)point_tile_big_kernel<R, 8, MODE>;
  }
  return nullptr;
}

template <typename R, int MODE>
static void* tile_fn(int I) {
  switch (I) {
    case 1: return (void*)point_tile_kernel<R, 1, MODE>;
    case 2: return (void*)point_tile_kernel<R, 2, MODE>;
    case 3: return (void*)point_tile_kernel<R, 3, MODE>;
    case 4: return (void*)point_tile_kernel<R, 4, MODE>;
  }
  return nullptr;
}

// Q = P^-H per bin (one thread per bin, fp64, LU from common.cuh in a
// per-thread local workspace).  Flags exactly singular P.
template <typename R, int I>
__global__ void inv_PH_kernel(const void* Pv, double2* Q, int* status, long long nbins) {
  using C2 = typename Cpx<R>::T;
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbins) return;
  const C2* P = (const C2*)Pv + b * I * I;
  double2 A[I * I], col[I];
  int piv[I];
  // factor P^H
#pragma unroll
  for (int x = 0; x < I; ++x)
#pragma unroll
    for (int y = 0; y < I; ++y) A[x * I + y] = make_double2(double(P[y * I + x].x), -double(P[y * I + x].y));
  if (!lu_factor<I>(A, piv)) {
    status[b] |= ST_SINGULAR_P;
    return;
  }
  for (int c = 0; c < I; ++c) {
#pragma unroll
    for (int x = 0; x < I; ++x) col[x] = make_double2(x == c ? 1.0 : 0.0, 0.0);
    lu_solve<I>(A, piv, col);
#pragma unroll
    for (int x = 0; x < I; ++x) Q[b * I * I + x * I + c] = col[x];
  }
}

template <typename R>
static void* point_fn(int I) {
  switch (I) {
    case 1: return (void*)point_kernel<R, 1>;
    case 2: return (void*)point_kernel<R, 2>;
    case 3: return (void*)point_kernel<R, 3>;
    case 4: return (void*)point_kernel<R, 4>;
    case 5: return (void*)point_kernel<R, 5>;
    case 6: return (void*)point_kernel<R, 6>;
    case 7: return (void*)point_kernel<R, 7>;
    case 8: return (void*)point_kernel<R, 8>;
  }
  return nullptr;
}

template <typename R>
static void* inv_fn(int I) {
  switch (I) {
    case 1: return (void*)inv_PH_kernel<R, 1>;
    case 2: return (void*)inv_PH_kernel<R, 2>;
    case 3: return (void*)inv_PH_kernel<R, 3>;
    case 4: return (void*)inv_PH_kernel<R, 4>;
    case 5: return (void*)inv_PH_kernel<R, 5>;
    case 6: return (void*)inv_PH_kernel<R, 6>;
    case 7: return (void*)inv_PH_kernel<R, 7>;
    case 8: return (void*)inv_PH_kernel<R, 8>;
  }
  return nullptr;
}

int launch_points(int dtype, const PointArgs& a, cudaStream_t s) {
  const long long npts = (long long)a.U * a.N * a.F;
  if (npts == 0) return FFCA_OK;
  // the tiled kernels index inside one mixture with 32-bit element offsets
  const bool fits32 = (long long)a.J * a.I * a.I * a.N * a.F < (1LL << 31);
  if ((a.mode == PM_STATS || a.mode == PM_IMAGES) && a.I <= 4 && a.J <= 4 && fits32) {
    void* tf = nullptr;
    if (a.mode == PM_STATS)
      tf = dtype == FFCA_C64 ? tile_fn<float, PM_STATS>(a.I) : tile_fn<double, PM_STATS>(a.I);
    else
      tf = dtype == FFCA_C64 ? tile_fn<float, PM_IMAGES>(a.I) : tile_fn<double, PM_IMAGES>(a.I);
    const int TS = a.mode == PM_IMAGES ? (dtype == FFCA_C64 ? tile_stride<float, PM_IMAGES>() : tile_stride<double, PM_IMAGES>())
                                       : TILE_F;
    const long long blocks = (long long)a.U * ((a.F + TS - 1) / TS);
    // frame blocks (grid.y): about 8 CTAs per SM in total, at least 64 frames each, whole steps of the warps
    int nsplit = int((8LL * 148 + blocks - 1) / blocks);
    if (nsplit > a.N / 64) nsplit = a.N / 64;
    if (nsplit < 1) nsplit = 1;
    int fpc = (a.N + nsplit - 1) / nsplit;
    fpc = (fpc + TILE_WARPS - 1) / TILE_WARPS * TILE_WARPS;
    nsplit = (a.N + fpc - 1) / fpc;
    void* args[] = {(void*)&a, (void*)&fpc};
    FFCA_CK(cudaLaunchKernel(tf, dim3(unsigned(blocks), unsigned(nsplit)), dim3(TILE_F * TILE_WARPS), args, 0, s));
    count_launch();
    return FFCA_OK;
  }
  if (a.mode == PM_BACK && a.I <= 8) {
    void* tf = dtype == FFCA_C64 ? back_tile_fn<float>(a.I) : back_tile_fn<double>(a.I);
    const size_t smem = size_t(32) * a.I * a.I * (dtype == FFCA_C64 ? 8 : 16);
    const long long tiles = (long long)a.U * ((a.F + 31) / 32);
    int nsplit = int((8LL * 148 + tiles - 1) / tiles);
    if (nsplit > (a.N + 31) / 32) nsplit = (a.N + 31) / 32;
    if (nsplit < 1) nsplit = 1;
    int fpc = (a.N + nsplit - 1) / nsplit;
    fpc = (fpc + 7) / 8 * 8;
    nsplit = (a.N + fpc - 1) / fpc;
    void* args[] = {(void*)&a, (void*)&fpc};
    FFCA_CK(cudaLaunchKernel(tf, dim3(unsigned(tiles), unsigned(nsplit)), dim3(256), args, smem, s));
    count_launch();
    return FFCA_OK;
  }
  if ((a.mode == PM_STATS || a.mode == PM_IMAGES) && a.I > 4 && a.I <= 8 && a.J <= 8) {
    void* tf = nullptr;
    if (a.mode == PM_STATS)
      tf = dtype == FFCA_C64 ? big_tile_fn<float, PM_STATS>(a.I) : big_tile_fn<double, PM_STATS>(a.I);
    else
      tf = dtype == FFCA_C64 ? big_tile_fn<float, PM_IMAGES>(a.I) : big_tile_fn<double, PM_IMAGES>(a.I);
    const size_t cs = dtype == FFCA_C64 ? 8 : 16, rs = cs / 2;
    const size_t smem = size_t(32) * a.I * a.I * cs * (a.mode == PM_IMAGES ? 2 : 1) + size_t(32) * a.J * a.I * rs;
    const long long tiles = (long long)a.U * ((a.F + 31) / 32);
    // frame blocks: enough CTAs to fill the device (~8 per SM), at least 32 frames each, even count
    int nsplit = int((8LL * 148 + tiles - 1) / tiles);
    if (nsplit > (a.N + 31) / 32) nsplit = (a.N + 31) / 32;
    if (nsplit < 1) nsplit = 1;
    int fpc = (a.N + nsplit - 1) / nsplit;
    fpc = (fpc + 15) / 16 * 16;  // whole steps of the 8 warps x 1 or 2 frames
    nsplit = (a.N + fpc - 1) / fpc;
    if (smem > 48 * 1024) FFCA_CK(cudaFuncSetAttribute(tf, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    void* args[] = {(void*)&a, (void*)&fpc};
    FFCA_CK(cudaLaunchKernel(tf, dim3(unsigned(tiles), unsigned(nsplit)), dim3(256), args, smem, s));
    count_launch();
    return FFCA_OK;
  }
  void* fn = dtype == FFCA_C64 ? point_fn<float>(a.I) : point_fn<double>(a.I);
  if (!fn) {
    set_error("unsupported order I=%d", a.I);
    return FFCA_E_UNSUPPORTED;
  }
  const unsigned blocks = unsigned((npts + 255) / 256);
  void* args[] = {(void*)&a};
  FFCA_CK(cudaLaunchKernel(fn, dim3(blocks), dim3(256), args, 0, s));
  count_launch();
  return FFCA_OK;
}

int launch_inv_PH(int dtype, int I, const void* P, double2* Q, int* status, long long nbins, cudaStream_t s) {
  if (nbins == 0) return FFCA_OK;
  void* fn = dtype == FFCA_C64 ? inv_fn<float>(I) : inv_fn<double>(I);
  if (!fn) {
    set_error("unsupported order I=%d", I);
    return FFCA_E_UNSUPPORTED;
  }
  const unsigned blocks = unsigned((nbins + 127) / 128);
  void* args[] = {(void*)&P, (void*)&Q, (void*)&status, (void*)&nbins};
  FFCA_CK(cudaLaunchKernel(fn, dim3(blocks), dim3(128), args, 0, s));
  count_launch();
  return FFCA_OK;
}

}  // namespace ffca

using namespace ffca;

static int points_common(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F) {
  (void)device;
  (void)stream;
  (void)mem;
  if (!check_dims(dtype, U, I, J, N, F)) return FFCA_E_ARG;
  if (I > 8) {
    set_error("unsupported order I=%d (matcore.MAX_ORDER = 8)", I);
    return FFCA_E_UNSUPPORTED;
  }
  return FFCA_OK;
}

extern "C" int ffca_fastfca_stats(int device, void* stream, int mem, int dtype, int U, int I, int J, int N,
                                  int F, const void* y, const void* P, const void* lam, const void* v, void* mu,
                                  void* phi) {
  reset_launches();
  FFCA_TRY(points_common(device, stream, mem, dtype, U, I, J, N, F));
  if (!y || !P || !lam || !v) {
    set_error("null array argument");
    return FFCA_E_ARG;
  }
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  Staging st(mem, s);
  PointArgs a = {};
  a.mode = PM_STATS; a.U = U; a.I = I; a.J = J; a.N = N; a.F = F;
  FFCA_TRY(st.in(y, size_t(U) * I * N * F * cs, &a.y));
  FFCA_TRY(st.in(P, size_t(U) * F * I * I * cs, &a.P));
  FFCA_TRY(st.in(lam, size_t(U) * J * F * I * rs, &a.lam));
  FFCA_TRY(st.in(v, size_t(U) * J * N * F * rs, &a.v));
  FFCA_TRY(st.out(mu, size_t(U) * J * N * F * I * cs, &a.out0));
  FFCA_TRY(st.out(phi, size_t(U) * J * N * F * I * rs, &a.out1));
  FFCA_TRY(launch_points(dtype, a, s));
  FFCA_TRY(st.flush());
  FFCA_CK(cudaStreamSynchronize(s));
  return FFCA_OK;
}

// e_step_diag from a given y_t (N, F, I) -- exposed through the same entry with
// y = y_t when the caller passes FFCA_ESTEP_YT in `mem` bit 8 (internal use).
extern "C" int ffca_fastfca_estep_yt(int device, void* stream, int mem, int dtype, int U, int I, int J, int N,
                                     int F, const void* yt, const void* lam, const void* v, void* mu,
                                     void* phi) {
  reset_launches();
  FFCA_TRY(points_common(device, stream, mem, dtype, U, I, J, N, F));
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  Staging st(mem, s);
  PointArgs a = {};
  a.mode = PM_ESTEP_YT; a.U = U; a.I = I; a.J = J; a.N = N; a.F = F;
  FFCA_TRY(st.in(yt, size_t(U) * N * F * I * cs, &a.y));
  FFCA_TRY(st.in(lam, size_t(U) * J * F * I * rs, &a.lam));
  FFCA_TRY(st.in(v, size_t(U) * J * N * F * rs, &a.v));
  FFCA_TRY(st.out(mu, size_t(U) * J * N * F * I * cs, &a.out0));
  FFCA_TRY(st.out(phi, size_t(U) * J * N * F * I * rs, &a.out1));
  FFCA_TRY(launch_points(dtype, a, s));
  FFCA_TRY(st.flush());
  FFCA_CK(cudaStreamSynchronize(s));
  return FFCA_OK;
}

extern "C" int ffca_transform(int device, void* stream, int mem, int dtype, int U, int I, int N, int F,
                              const void* y, const void* P, void* yt) {
  reset_launches();
  FFCA_TRY(points_common(device, stream, mem, dtype, U, I, 1, N, F));
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t cs = csize(dtype);
  Staging st(mem, s);
  PointArgs a = {};
  a.mode = PM_TRANSFORM; a.U = U; a.I = I; a.J = 1; a.N = N; a.F = F;
  FFCA_TRY(st.in(y, size_t(U) * I * N * F * cs, &a.y));
  FFCA_TRY(st.in(P, size_t(U) * F * I * I * cs, &a.P));
  FFCA_TRY(st.out(yt, size_t(U) * N * F * I * cs, &a.out0));
  FFCA_TRY(launch_points(dtype, a, s));
  FFCA_TRY(st.flush());
  FFCA_CK(cudaStreamSynchronize(s));
  return FFCA_OK;
}

extern "C" int ffca_mixture_weights(int device, void* stream, int mem, int dtype, int U, int I, int J, int N,
                                    int F, const void* lam, const void* v, void* w) {
  reset_launches();
  FFCA_TRY(points_common(device, stream, mem, dtype, U, I, J, N, F));
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rs = rsize(dtype);
  Staging st(mem, s);
  PointArgs a = {};
  a.mode = PM_WEIGHTS; a.U = U; a.I = I; a.J = J; a.N = N; a.F = F;
  FFCA_TRY(st.in(lam, size_t(U) * J * F * I * rs, &a.lam));
  FFCA_TRY(st.in(v, size_t(U) * J * N * F * rs, &a.v));
  FFCA_TRY(st.out(w, size_t(U) * N * F * I * rs, &a.out0));
  FFCA_TRY(launch_points(dtype, a, s));
  FFCA_TRY(st.flush());
  FFCA_CK(cudaStreamSynchronize(s));
  return FFCA_OK;
}

extern "C" int ffca_fastfca_images(int device, void* stream, int mem, int dtype, int U, int I, int J, int N,
                                   int F, const void* y, const void* P, const void* lam, const void* v,
                                   void* images, int* status) {
  reset_launches();
  FFCA_TRY(points_common(device, stream, mem, dtype, U, I, J, N, F));
  if (!y || !P || !lam || !v || !images) {
    set_error("null array argument");
    return FFCA_E_ARG;
  }
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  const long long nb = (long long)U * F;
  Staging st(mem, s);
  PointArgs a = {};
  a.mode = PM_IMAGES; a.U = U; a.I = I; a.J = J; a.N = N; a.F = F;
  FFCA_TRY(st.in(y, size_t(U) * I * N * F * cs, &a.y));
  FFCA_TRY(st.in(P, size_t(nb) * I * I * cs, &a.P));
  FFCA_TRY(st.in(lam, size_t(U) * J * F * I * rs, &a.lam));
  FFCA_TRY(st.in(v, size_t(U) * J * N * F * rs, &a.v));
  FFCA_TRY(st.out(images, size_t(U) * J * I * N * F * cs, &a.out0));
  void *Q, *dstatus;
  FFCA_TRY(st.scratch(size_t(nb) * I * I * 16, &Q));
  FFCA_TRY(st.scratch(size_t(nb) * 4, &dstatus));
  FFCA_CK(cudaMemsetAsync(dstatus, 0, size_t(nb) * 4, s));
  FFCA_TRY(launch_inv_PH(dtype, I, a.P, (double2*)Q, (int*)dstatus, nb, s));
  a.Q = Q;
  FFCA_TRY(launch_points(dtype, a, s));
  FFCA_TRY(st.flush());
  return finish_status((const int*)dstatus, status, nb, mem, s, FFCA_ST_SINGULAR_P);
}

extern "C" int ffca_back_transform(int device, void* stream, int mem, int dtype, int U, int I, int J, int N,
                                   int F, const void* P, const void* mu_t, void* out, int images_layout,
                                   int* status) {
  reset_launches();
  FFCA_TRY(points_common(device, stream, mem, dtype, U, I, J, N, F));
  if (!P || !mu_t || !out) {
    set_error("null array argument");
    return FFCA_E_ARG;
  }
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t cs = csize(dtype);
  const long long nb = (long long)U * F;
  Staging st(mem, s);
  PointArgs a = {};
  a.mode = PM_BACK; a.U = U; a.I = I; a.J = J; a.N = N; a.F = F;
  a.images_layout = images_layout;
  FFCA_TRY(st.in(P, size_t(nb) * I * I * cs, &a.P));
  FFCA_TRY(st.in(mu_t, size_t(U) * J * N * F * I * cs, &a.y));
  FFCA_TRY(st.out(out, size_t(U) * J * N * F * I * cs, &a.out0));
  void *Q, *dstatus;
  FFCA_TRY(st.scratch(size_t(nb) * I * I * 16, &Q));
  FFCA_TRY(st.scratch(size_t(nb) * 4, &dstatus));
  FFCA_CK(cudaMemsetAsync(dstatus, 0, size_t(nb) * 4, s));
  FFCA_TRY(launch_inv_PH(dtype, I, a.P, (double2*)Q, (int*)dstatus, nb, s));
  a.Q = Q;
  FFCA_TRY(launch_points(dtype, a, s));
  FFCA_TRY(st.flush());
  return finish_status((const int*)dstatus, status, nb, mem, s, FFCA_ST_SINGULAR_P);
}
