// Throughput of legacy mma.sync m16n8k8 TF32 (fp32 accumulate) on this GPU: warps x independent chains.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_mma(float* out, int n, long long* cyc) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  float c[4][4] = {};
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int m = 0; m < 4; ++m)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[m][0]), "+f"(c[m][1]), "+f"(c[m][2]), "+f"(c[m][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  float s = 0;
  for (int m = 0; m < 4; ++m) for (int k = 0; k < 4; ++k) s += c[m][k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* o; long long* c; long long h;
  cudaMalloc(&o, 1 << 24); cudaMalloc(&c, 8);
  const int n = 2048;
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int warps : {1, 4, 8, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k_mma<<<nsm, 32 * warps>>>(o, n, c);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      if (rep) printf("%2d warps/SM: %.2f cycles per mma per warp (clock64), %.1f TFLOP/s tf32 (events)\n", warps,
                      double(h) / (4.0 * n), 2.0 * 16 * 8 * 8 * 4.0 * n * warps * nsm / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
