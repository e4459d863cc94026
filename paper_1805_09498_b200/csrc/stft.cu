// STFT analysis / synthesis on the device (stft.analyze / stft.synthesize,
// stft.py:96-134) -- the caller of the estimation path.
//
//   analyze:    frame + sqrt-Hann window (one kernel) -> cuFFT batched R2C
//               -> pack (bins 1..L/2-1 as is; bin 0 = DC.re + i * Nyquist.re)
//   synthesize: unpack -> cuFFT batched C2R -> window + overlap-add as a gather
//               (each output sample sums the <= L/shift frames covering it, in
//               frame order: deterministic, no atomics)
// The reference's packing keeps F = L/2 complex bins (stft.py:7-13,110-111).
#include <cufft.h>

#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "host_common.h"

namespace ffca {

template <typename R>
__global__ void frame_window_kernel(const R* audio, R* frames, int I, long long S, int N, int L, int shift) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)I * N * L;
  if (t >= total) return;
  const int k = int(t % L);
  const long long in = t / L;
  const int n = int(in % N);
  const int i = int(in / N);
  const R w = R(sin(M_PI * double(k) / double(L)));
  frames[t] = audio[(long long)i * S + (long long)n * shift + k] * w;
}

template <typename R>
__global__ void pack_kernel(const typename Cpx<R>::T* spec, typename Cpx<R>::T* out, long long rows, int L) {
  using C2 = typename Cpx<R>::T;
  const int F = L / 2;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * F) return;
  const int f = int(t % F);
  const long long r = t / F;
  const C2* s = spec + r * (F + 1);
  out[t] = f == 0 ? mk<C2, R>(s[0].x, s[F].x) : s[f];
}

template <typename R>
__global__ void unpack_kernel(const typename Cpx<R>::T* in, typename Cpx<R>::T* spec, long long rows, int L) {
  using C2 = typename Cpx<R>::T;
  const int F = L / 2;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * (F + 1)) return;
  const int f = int(t % (F + 1));
  const long long r = t / (F + 1);
  const C2* s = in + r * F;
  C2 v;
  if (f == 0) v = mk<C2, R>(s[0].x, R(0));
  else if (f == F) v = mk<C2, R>(s[0].y, R(0));
  else v = s[f];
  spec[t] = v;
}

template <typename R>
__global__ void overlap_add_kernel(const R* frames, R* out, int I, int N, int L, int shift, long long S_out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)I * S_out) return;
  const long long s = t % S_out;
  const int i = int(t / S_out);
  long long nlo = (s - L + shift) / shift;  // ceil((s - L + 1) / shift) for s >= L
  if (s < L) nlo = 0;
  long long nhi = s / shift;
  if (nhi > N - 1) nhi = N - 1;
  double acc = 0.0;
  const double invL = 1.0 / double(L);
  for (long long n = nlo; n <= nhi; ++n) {
    const int k = int(s - n * shift);
    if (k < 0 || k >= L) continue;
    const double w = sin(M_PI * double(k) / double(L));
    acc += double(frames[((long long)i * N + n) * L + k]) * invL * w;
  }
  out[t] = R(acc);
}

// cuFFT plans cached per (type, L, batch, device).
static std::mutex g_plan_mu;
static std::map<std::tuple<int, int, long long, int>, cufftHandle> g_plans;

static int get_plan(cufftType type, int L, long long batch, int device, cufftHandle* out) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  auto key = std::make_tuple(int(type), L, batch, device);
  auto it = g_plans.find(key);
  if (it != g_plans.end()) {
    *out = it->second;
    return FFCA_OK;
  }
  cufftHandle h;
  int n[1] = {L};
  if (cufftPlanMany(&h, 1, n, nullptr, 1, 0, nullptr, 1, 0, type, int(batch)) != CUFFT_SUCCESS) {
    set_error("cufftPlanMany failed (L=%d batch=%lld)", L, batch);
    return FFCA_E_CUDA;
  }
  g_plans[key] = h;
  *out = h;
  return FFCA_OK;
}

}  // namespace ffca

using namespace ffca;

extern "C" int ffca_stft_analyze(int device, void* stream, int mem, int dtype, int I, long long S, int L, int shift,
                                 const void* audio, void* out) {
  reset_launches();
  if ((dtype != FFCA_C128 && dtype != FFCA_C64) || I < 1 || L < 2 || L % 2 || shift < 1 || S < L || !audio ||
      !out) {
    set_error("bad arguments to ffca_stft_analyze (I=%d S=%lld L=%d shift=%d)", I, S, L, shift);
    return FFCA_E_ARG;
  }
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const int N = int((S - L) / shift + 1), F = L / 2;
  const long long rows = (long long)I * N;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  Staging st(mem, s);
  const void* da;
  void *dout, *frames, *spec;
  FFCA_TRY(st.in(audio, size_t(I) * S * rs, &da));
  FFCA_TRY(st.out(out, size_t(rows) * F * cs, &dout));
  FFCA_TRY(st.scratch(size_t(rows) * L * rs, &frames));
  FFCA_TRY(st.scratch(size_t(rows) * (F + 1) * cs, &spec));
  const long long nfr = rows * L;
  cufftHandle plan;
  if (dtype == FFCA_C128) {
    frame_window_kernel<double><<<unsigned((nfr + 255) / 256), 256, 0, s>>>((const double*)da, (double*)frames, I, S,
                                                                             N, L, shift);
    FFCA_TRY(get_plan(CUFFT_D2Z, L, rows, device, &plan));
    cufftSetStream(plan, s);
    if (cufftExecD2Z(plan, (cufftDoubleReal*)frames, (cufftDoubleComplex*)spec) != CUFFT_SUCCESS) {
      set_error("cufftExecD2Z failed");
      return FFCA_E_CUDA;
    }
    pack_kernel<double><<<unsigned((rows * F + 255) / 256), 256, 0, s>>>((const double2*)spec, (double2*)dout, rows, L);
  } else {
    frame_window_kernel<float><<<unsigned((nfr + 255) / 256), 256, 0, s>>>((const float*)da, (float*)frames, I, S, N,
                                                                            L, shift);
    FFCA_TRY(get_plan(CUFFT_R2C, L, rows, device, &plan));
    cufftSetStream(plan, s);
    if (cufftExecR2C(plan, (cufftReal*)frames, (cufftComplex*)spec) != CUFFT_SUCCESS) {
      set_error("cufftExecR2C failed");
      return FFCA_E_CUDA;
    }
    pack_kernel<float><<<unsigned((rows * F + 255) / 256), 256, 0, s>>>((const float2*)spec, (float2*)dout, rows, L);
  }
  count_launch(3);
  FFCA_CK(cudaGetLastError());
  FFCA_TRY(st.flush());
  FFCA_CK(cudaStreamSynchronize(s));
  return FFCA_OK;
}

extern "C" int ffca_stft_synthesize(int device, void* stream, int mem, int dtype, int I, int N, int L, int shift,
                                    const void* in, void* audio) {
  reset_launches();
  if ((dtype != FFCA_C128 && dtype != FFCA_C64) || I < 1 || N < 1 || L < 2 || L % 2 || shift < 1 || !in ||
      !audio) {
    set_error("bad arguments to ffca_stft_synthesize");
    return FFCA_E_ARG;
  }
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const int F = L / 2;
  const long long rows = (long long)I * N;
  const long long S_out = (long long)(N - 1) * shift + L;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  Staging st(mem, s);
  const void* din;
  void *dout, *spec, *frames;
  FFCA_TRY(st.in(in, size_t(rows) * F * cs, &din));
  FFCA_TRY(st.out(audio, size_t(I) * S_out * rs, &dout));
  FFCA_TRY(st.scratch(size_t(rows) * (F + 1) * cs, &spec));
  FFCA_TRY(st.scratch(size_t(rows) * L * rs, &frames));
  cufftHandle plan;
  const long long nsp = rows * (F + 1), nout = (long long)I * S_out;
  if (dtype == FFCA_C128) {
    unpack_kernel<double><<<unsigned((nsp + 255) / 256), 256, 0, s>>>((const double2*)din, (double2*)spec, rows, L);
    FFCA_TRY(get_plan(CUFFT_Z2D, L, rows, device, &plan));
    cufftSetStream(plan, s);
    if (cufftExecZ2D(plan, (cufftDoubleComplex*)spec, (cufftDoubleReal*)frames) != CUFFT_SUCCESS) {
      set_error("cufftExecZ2D failed");
      return FFCA_E_CUDA;
    }
    overlap_add_kernel<double><<<unsigned((nout + 255) / 256), 256, 0, s>>>((const double*)frames, (double*)dout, I, N,
                                                                             L, shift, S_out);
  } else {
    unpack_kernel<float><<<unsigned((nsp + 255) / 256), 256, 0, s>>>((const float2*)din, (float2*)spec, rows, L);
    FFCA_TRY(get_plan(CUFFT_C2R, L, rows, device, &plan));
    cufftSetStream(plan, s);
    if (cufftExecC2R(plan, (cufftComplex*)spec, (cufftReal*)frames) != CUFFT_SUCCESS) {
      set_error("cufftExecC2R failed");
      return FFCA_E_CUDA;
    }
    overlap_add_kernel<float><<<unsigned((nout + 255) / 256), 256, 0, s>>>((const float*)frames, (float*)dout, I, N, L,
                                                                            shift, S_out);
  }
  count_launch(3);
  FFCA_CK(cudaGetLastError());
  FFCA_TRY(st.flush());
  FFCA_CK(cudaStreamSynchronize(s));
  return FFCA_OK;
}

// ---------------------------------------------------------------------------
// SDR energies (evalkit.compute_sdr, evalkit.py:68-88): per source j the fp64
// sums ||s||^2 and ||s - s_hat||^2 over channels and the first L samples.
// 64 CTAs per source, then a fixed-order combine (deterministic).
// ---------------------------------------------------------------------------
namespace ffca {

constexpr int SDR_CHUNKS = 64;  // CTAs per source; partials combined in a fixed order

// CTA (chunk c, source j) sums samples [c*L/64, (c+1)*L/64) of every channel.
template <typename R>
__global__ void __launch_bounds__(256) sdr_energy_kernel(const R* ref, const R* est, double* part, int I, long long Sr,
                                                         long long Se, long long L) {
  const int j = blockIdx.y, c = blockIdx.x;
  const long long lo = L * c / SDR_CHUNKS, hi = L * (c + 1) / SDR_CHUNKS;
  double er = 0.0, ee = 0.0;
  for (int i = 0; i < I; ++i) {
    const R* r = ref + ((long long)j * I + i) * Sr;
    const R* e = est + ((long long)j * I + i) * Se;
    for (long long t = lo + threadIdx.x; t < hi; t += blockDim.x) {
      const double a = double(r[t]), d = a - double(e[t]);
      er = fma(a, a, er);
      ee = fma(d, d, ee);
    }
  }
  __shared__ double sr[8], se[8];
  for (int o = 16; o >= 1; o >>= 1) {
    er += __shfl_xor_sync(FULL, er, o);
    ee += __shfl_xor_sync(FULL, ee, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sr[w] = er;
    se[w] = ee;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int k = 0; k < 8; ++k) {
      x += sr[k];
      y += se[k];
    }
    part[((long long)j * SDR_CHUNKS + c) * 2] = x;
    part[((long long)j * SDR_CHUNKS + c) * 2 + 1] = y;
  }
}

__global__ void sdr_combine_kernel(const double* part, double* out, int J) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  double x = 0.0, y = 0.0;
  for (int c = 0; c < SDR_CHUNKS; ++c) {
    x += part[((long long)j * SDR_CHUNKS + c) * 2];
    y += part[((long long)j * SDR_CHUNKS + c) * 2 + 1];
  }
  out[2 * j] = x;
  out[2 * j + 1] = y;
}

}  // namespace ffca

// ref (J, I, Sr), est (J, I, Se) real (dtype C128 -> float64, C64 -> float32);
// out (J, 2) float64 = (||ref||^2, ||ref - est||^2) over the first min(Sr, Se) samples.
extern "C" int ffca_sdr_energies(int device, void* stream, int mem, int dtype, int J, int I, long long Sr,
                                 long long Se, const void* ref, const void* est, double* out) {
  reset_launches();
  if ((dtype != FFCA_C128 && dtype != FFCA_C64) || J < 1 || I < 1 || Sr < 0 || Se < 0 || !ref || !est || !out) {
    set_error("bad arguments to ffca_sdr_energies");
    return FFCA_E_ARG;
  }
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rs = rsize(dtype);
  Staging st(mem, s);
  const void *dr, *de;
  void* dout;
  FFCA_TRY(st.in(ref, size_t(J) * I * Sr * rs, &dr));
  FFCA_TRY(st.in(est, size_t(J) * I * Se * rs, &de));
  FFCA_TRY(st.out(out, size_t(J) * 2 * 8, &dout));
  const long long L = Sr < Se ? Sr : Se;
  void* part;
  FFCA_TRY(st.scratch(size_t(J) * SDR_CHUNKS * 2 * 8, &part));
  const dim3 grid(SDR_CHUNKS, J);
  if (dtype == FFCA_C128)
    sdr_energy_kernel<double><<<grid, 256, 0, s>>>((const double*)dr, (const double*)de, (double*)part, I, Sr, Se, L);
  else
    sdr_energy_kernel<float><<<grid, 256, 0, s>>>((const float*)dr, (const float*)de, (double*)part, I, Sr, Se, L);
  sdr_combine_kernel<<<(J + 127) / 128, 128, 0, s>>>((const double*)part, (double*)dout, J);
  count_launch(2);
  FFCA_CK(cudaGetLastError());
  FFCA_TRY(st.flush());
  FFCA_CK(cudaStreamSynchronize(s));
  return FFCA_OK;
}
