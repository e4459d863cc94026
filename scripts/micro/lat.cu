// Dependent-chain latency of a few instructions on this GPU (cycles per op, one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* out, double a, double b, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_ffma(float* out, float a, float b, int n, long long* cyc) {
  float x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fmaf(x, b, a); x = fmaf(x, b, a); x = fmaf(x, b, a); x = fmaf(x, b, a); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_drcp(double* out, double a, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + a; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_shfl(float* out, float a, int n, long long* cyc) {
  float x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __shfl_xor_sync(0xffffffff, x, 1) + a; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dthr(double* out, double a, double b, int n, long long* cyc) {  // 8 independent chains
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, b, a); x1 = fma(x1, b, a); x2 = fma(x2, b, a); x3 = fma(x3, b, a);
    x4 = fma(x4, b, a); x5 = fma(x5, b, a); x6 = fma(x6, b, a); x7 = fma(x7, b, a);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7; if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* d; float* f; long long* c; long long h;
  cudaMalloc(&d, 4096); cudaMalloc(&f, 4096); cudaMalloc(&c, 8);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    k_dfma<<<1, 32>>>(d, 0.5, 0.999, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("DFMA dependent: %.2f cycles/op\n", double(h) / (4.0 * n));
    k_ffma<<<1, 32>>>(f, 0.5f, 0.999f, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("FFMA dependent: %.2f cycles/op\n", double(h) / (4.0 * n));
    k_drcp<<<1, 32>>>(d, 1.5, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("MUFU.RCP64H + DADD dependent: %.2f cycles/iter\n", double(h) / n);
    k_shfl<<<1, 32>>>(f, 0.5f, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("SHFL + FADD dependent: %.2f cycles/iter\n", double(h) / n);
    k_dthr<<<1, 32>>>(d, 0.5, 0.999, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("DFMA 8 chains, 1 warp: %.2f cycles per warp-DFMA\n", double(h) / (8.0 * n));
    k_dthr<<<1, 128>>>(d, 0.5, 0.999, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("DFMA 8 chains, 4 warps (1 per SMSP): %.2f cycles per warp-DFMA\n", double(h) / (8.0 * n));
    k_dthr<<<1, 512>>>(d, 0.5, 0.999, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("DFMA 8 chains, 16 warps: %.2f cycles per 8 DFMA per warp -> %.2f warp-DFMA/clk/SM\n", double(h) / n, 16.0 * 8 * n / double(h));
  }
  return 0;
}
