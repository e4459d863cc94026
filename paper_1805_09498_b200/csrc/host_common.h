// Host-side helpers shared by the C-ABI entry points.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ffca.h"

namespace ffca {

void set_error(const char* fmt, ...);
void count_launch(int n = 1);
void reset_launches();
bool timing_enabled();
void set_kernel_ms(float ms);

#define FFCA_CK(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      ::ffca::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
      return FFCA_E_CUDA;                                                                \
    }                                                                                    \
  } while (0)

#define FFCA_TRY(expr)        \
  do {                        \
    int rc_ = (expr);         \
    if (rc_ != FFCA_OK) return rc_; \
  } while (0)

void retain_pool(int dev);

// Selects `device` for the lifetime of the object, restoring the previous one.
// Also makes the device's stream-ordered pool keep its memory between calls
// (release threshold = max) so repeated calls do not re-map their buffers.
struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ok = cudaSetDevice(dev) == cudaSuccess;
    if (ok) retain_pool(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// A device view of one argument array.  In FFCA_MEM_HOST mode the array is
// staged through a stream-ordered device allocation; in FFCA_MEM_DEVICE mode
// the caller's pointer is used directly.
struct Arg {
  void* host = nullptr;
  void* dev = nullptr;
  size_t bytes = 0;
  bool owned = false;
};

class Staging {
 public:
  Staging(int mem, cudaStream_t s) : mem_(mem), s_(s) {}
  ~Staging() {
    for (auto& a : args_)
      if (a.owned && a.dev) cudaFreeAsync(a.dev, s_);
    for (void* p : tmp_) cudaFreeAsync(p, s_);
  }
  // input: copied H2D in host mode
  int in(const void* p, size_t bytes, const void** out) {
    if (!p || bytes == 0) { *out = p; return FFCA_OK; }
    if (mem_ == FFCA_MEM_DEVICE) { *out = p; return FFCA_OK; }
    Arg a;
    a.host = const_cast<void*>(p);
    a.bytes = bytes;
    FFCA_CK(cudaMallocAsync(&a.dev, bytes, s_));
    a.owned = true;
    FFCA_CK(cudaMemcpyAsync(a.dev, p, bytes, cudaMemcpyHostToDevice, s_));
    args_.push_back(a);
    *out = a.dev;
    return FFCA_OK;
  }
  // output: device buffer, copied D2H by flush() in host mode
  int out(void* p, size_t bytes, void** outp) {
    if (!p || bytes == 0) { *outp = p; return FFCA_OK; }
    if (mem_ == FFCA_MEM_DEVICE) { *outp = p; return FFCA_OK; }
    Arg a;
    a.host = p;
    a.bytes = bytes;
    FFCA_CK(cudaMallocAsync(&a.dev, bytes, s_));
    a.owned = true;
    outs_.push_back(args_.size());
    args_.push_back(a);
    *outp = a.dev;
    return FFCA_OK;
  }
  // device scratch, freed at destruction
  int scratch(size_t bytes, void** p) {
    *p = nullptr;
    if (bytes == 0) return FFCA_OK;
    FFCA_CK(cudaMallocAsync(p, bytes, s_));
    tmp_.push_back(*p);
    return FFCA_OK;
  }
  int flush() {
    for (size_t k : outs_) {
      Arg& a = args_[k];
      FFCA_CK(cudaMemcpyAsync(a.host, a.dev, a.bytes, cudaMemcpyDeviceToHost, s_));
    }
    return FFCA_OK;
  }
  int mem() const { return mem_; }
  cudaStream_t stream() const { return s_; }

 private:
  int mem_;
  cudaStream_t s_;
  std::vector<Arg> args_;
  std::vector<size_t> outs_;
  std::vector<void*> tmp_;
};

inline bool check_dims(int dtype, int U, int I, int J, int N, int F) {
  if (dtype != FFCA_C128 && dtype != FFCA_C64) {
    set_error("dtype must be FFCA_C128 or FFCA_C64, got %d", dtype);
    return false;
  }
  if (U < 0 || J < 1 || N < 1 || F < 0 || I < 1) {
    set_error("bad sizes U=%d I=%d J=%d N=%d F=%d", U, I, J, N, F);
    return false;
  }
  return true;
}

inline size_t rsize(int dtype) { return dtype == FFCA_C64 ? 4 : 8; }
inline size_t csize(int dtype) { return 2 * rsize(dtype); }

// Sum per-bin likelihood parts into per-mixture totals (device, fixed order).
int reduce_ll(const double* ll_bins, double* ll_mix_dev, int U, int F, int nev, double constant,
              cudaStream_t s);
// OR-reduce status and copy out; returns the FFCA_E_* code of the worst flag.
int finish_status(const int* status_dev, int* status_host_or_dev, long long nbins, int mem, cudaStream_t s,
                  int fatal_mask);

}  // namespace ffca
