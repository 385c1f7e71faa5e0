// Throughput probe: MUFU ex2 f32 vs packed bf16x2 / f16x2 vs FMA-pipe polynomial exp2.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ float ex2f(float x){float y;asm volatile("ex2.approx.ftz.f32 %0, %1;":"=f"(y):"f"(x));return y;}
__device__ __forceinline__ uint32_t ex2bf2(uint32_t x){uint32_t y;asm volatile("ex2.approx.ftz.bf16x2 %0, %1;":"=r"(y):"r"(x));return y;}
__device__ __forceinline__ uint32_t ex2h2(uint32_t x){uint32_t y;asm volatile("ex2.approx.f16x2 %0, %1;":"=r"(y):"r"(x));return y;}
// degree-3 polynomial 2^x on the FMA pipe (x <= 0)
__device__ __forceinline__ float ex2poly(float x){
  x = fmaxf(x, -127.f);
  float fi = floorf(x); float f = x - fi;
  float p = fmaf(fmaf(fmaf(0.0555041086f, f, 0.2402264923f), f, 0.6931471806f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (int(fi) << 23));
}
template<int MODE> __global__ void k(float* out, int iters){
  float a[8]; uint32_t b[8];
  for(int i=0;i<8;i++){a[i]=-(threadIdx.x+i)*1e-3f; b[i]=0xbf00bf00u+i;}
  for(int it=0; it<iters; ++it){
#pragma unroll
    for(int i=0;i<8;i++){
      if(MODE==0) a[i]=ex2f(a[i])-1.5f;
      if(MODE==1) b[i]=ex2bf2(b[i])^0x80008000u;
      if(MODE==2) b[i]=ex2h2(b[i])^0x80008000u;
      if(MODE==3) a[i]=ex2poly(a[i])-1.5f;
    }
  }
  float s=0; for(int i=0;i<8;i++) s+=a[i]+__uint_as_float(b[i]);
  if(s==12345.f) out[0]=s;
}
int main(){
  float* o; cudaMalloc(&o,4); int iters=4096; int blocks=148*4, thr=512;
  const char* names[4]={"ex2.f32","ex2.bf16x2","ex2.f16x2","poly3.f32(FMA)"};
  for(int m=0;m<4;m++){
    cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for(int rep=0;rep<2;rep++){
      cudaEventRecord(e0);
      if(m==0)k<0><<<blocks,thr>>>(o,iters); if(m==1)k<1><<<blocks,thr>>>(o,iters);
      if(m==2)k<2><<<blocks,thr>>>(o,iters); if(m==3)k<3><<<blocks,thr>>>(o,iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double n = double(blocks)*thr*iters*8*((m==1||m==2)?2:1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-16s %.3f ms  %.2f Texp/s  (%.1f exp/clk/SM at %d MHz)\n", names[m], ms, n/ms/1e9, n/(ms*1e-3)/148/(clk*1e3), clk/1000);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
