// C-ABI core: error state, launch accounting, small shared device kernels.
#include "host_common.h"

#include <mutex>

namespace ffca {

static thread_local char g_err[1024] = {0};
static thread_local int g_launches = 0;
static thread_local int g_timing = 0;
static thread_local float g_kernel_ms = 0.f;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void count_launch(int n) { g_launches += n; }

void retain_pool(int dev) {
  static std::mutex mu;
  static bool done[64] = {false};
  if (dev < 0 || dev >= 64) return;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done[dev] = true;
}
void reset_launches() { g_launches = 0; }
bool timing_enabled() { return g_timing != 0; }
void set_kernel_ms(float ms) { g_kernel_ms = ms; }

// Per-mixture likelihood totals: out[u*nev + e] = constant + sum_f part[(u*F + f)*nev + e],
// summed in bin order (deterministic).
__global__ void ll_reduce_kernel(const double* part, double* out, int U, int F, int nev, double constant) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= U * nev) return;
  const int u = t / nev, e = t % nev;
  double s = 0.0;
  for (int f = 0; f < F; ++f) s += part[((long long)u * F + f) * nev + e];
  out[t] = constant + s;
}

int reduce_ll(const double* ll_bins, double* ll_mix_dev, int U, int F, int nev, double constant,
              cudaStream_t s) {
  const int n = U * nev;
  if (n == 0) return FFCA_OK;
  ll_reduce_kernel<<<(n + 127) / 128, 128, 0, s>>>(ll_bins, ll_mix_dev, U, F, nev, constant);
  count_launch();
  FFCA_CK(cudaGetLastError());
  return FFCA_OK;
}

// OR of all per-bin status words and the first bin carrying a fatal bit (order independent, so
// deterministic): out[0] = OR, out[1] = first fatal bin or INT_MAX.
__global__ void status_summary_kernel(const int* st, long long n, int fatal_mask, int* out) {
  __shared__ int s_or, s_first;
  if (threadIdx.x == 0) {
    s_or = 0;
    s_first = 0x7fffffff;
  }
  __syncthreads();
  int o = 0, fst = 0x7fffffff;
  for (long long k = threadIdx.x; k < n; k += blockDim.x) {
    const int v = st[k];
    o |= v;
    if ((v & fatal_mask) && k < fst) fst = int(k);
  }
  atomicOr(&s_or, o);
  atomicMin(&s_first, fst);
  __syncthreads();
  if (threadIdx.x == 0) {
    out[0] = s_or;
    out[1] = s_first;
  }
}

int finish_status(const int* status_dev, int* status_user, long long nbins, int mem, cudaStream_t s,
                  int fatal_mask) {
  if (nbins == 0) return FFCA_OK;
  int any = 0;
  long long first = -1;
  std::vector<int> h;
  if (status_user && mem != FFCA_MEM_DEVICE) {  // the caller wants every bin's word on the host
    h.resize(nbins);
    FFCA_CK(cudaMemcpyAsync(h.data(), status_dev, nbins * sizeof(int), cudaMemcpyDeviceToHost, s));
    FFCA_CK(cudaStreamSynchronize(s));
    for (long long k = 0; k < nbins; ++k) {
      any |= h[k];
      if (first < 0 && (h[k] & fatal_mask)) first = k;
    }
  } else {  // summarise on the device: 8 bytes back instead of the whole status array
    int* d2 = nullptr;
    FFCA_CK(cudaMallocAsync(&d2, 2 * sizeof(int), s));
    status_summary_kernel<<<1, 1024, 0, s>>>(status_dev, nbins, fatal_mask, d2);
    count_launch();
    int h2[2] = {0, 0};
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(h2, d2, sizeof(h2), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(d2, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      set_error("status summary: %s", cudaGetErrorString(e));
      return FFCA_E_CUDA;
    }
    any = h2[0];
    first = h2[1] == 0x7fffffff ? -1 : h2[1];
  }
  if (status_user) {
    if (mem == FFCA_MEM_DEVICE)
      FFCA_CK(cudaMemcpyAsync(status_user, status_dev, nbins * sizeof(int), cudaMemcpyDeviceToDevice, s));
    else
      std::memcpy(status_user, h.data(), nbins * sizeof(int));
  }
  any &= fatal_mask;
  if (any & FFCA_ST_SINGULAR_P) {
    set_error("basis transform P is singular (bin index %lld)", first);
    return FFCA_E_SINGULAR_P;
  }
  if (any & FFCA_ST_SINGULAR_B) {
    set_error("weighted covariance stayed singular after diagonal loading (bin index %lld)", first);
    return FFCA_E_SINGULAR_B;
  }
  if (any & FFCA_ST_NOT_PD) {
    set_error("matrix not positive definite / singular (bin index %lld)", first);
    return FFCA_E_NOT_PD;
  }
  return FFCA_OK;
}

}  // namespace ffca

extern "C" {

int ffca_version(void) { return 100; }

const char* ffca_last_error(void) { return ffca::g_err; }

int ffca_last_launch_count(void) { return ffca::g_launches; }

void ffca_set_kernel_timing(int on) { ffca::g_timing = on; }

float ffca_last_kernel_ms(void) { return ffca::g_kernel_ms; }

int ffca_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int ffca_host_alloc(void** ptr, long long bytes) {
  FFCA_CK(cudaMallocHost(ptr, size_t(bytes)));
  return FFCA_OK;
}

int ffca_host_free(void* ptr) {
  FFCA_CK(cudaFreeHost(ptr));
  return FFCA_OK;
}

}  // extern "C"
