#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdio>


#include "../../paper_1805_09498_b200/csrc/common.cuh"
using namespace ffca;
__global__ void k(float* o){
  __shared__ unsigned base;
  if (threadIdx.x < 32) tmem_alloc(&base, 128);
  tmem_fence_before(); __syncthreads(); tmem_fence_after();
  unsigned t = base + (((threadIdx.x>>5)&3)*32u << 16);
  float r8[8], r4[4];
  for (int i=0;i<8;++i) r8[i]=threadIdx.x*100+i;
  for (int i=0;i<4;++i) r4[i]=threadIdx.x*100+8+i;
  tmem_st8(t+12, r8); tmem_st4(t+20, r4); tmem_wait_st();
  float a8[8], a4[4];
  tmem_ld8(t+12, a8); tmem_ld4(t+20, a4); tmem_wait_ld();
  float s=0; for(int i=0;i<8;++i) s+=a8[i]; for(int i=0;i<4;++i) s+=a4[i];
  o[threadIdx.x]=s;
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(base, 128);
}
int main(){ float* d; cudaMalloc(&d, 128*4); k<<<1,128>>>(d); float h[128]; cudaMemcpy(h,d,512,cudaMemcpyDeviceToHost);
 int bad=0; for(int t=0;t<128;++t){ float e=12*t*100+66; if(h[t]!=e) bad++; } printf("err=%s bad=%d h[5]=%f\n", cudaGetErrorString(cudaGetLastError()), bad, h[5]); return bad; }
