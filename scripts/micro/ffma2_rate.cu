#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2(u64 a, u64 b, u64 c){ u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;}
__global__ void kffma(float* out, int iters, float s){
  float a[8]; for(int k=0;k<8;++k) a[k]=threadIdx.x*0.001f+k;
  for(int i=0;i<iters;++i){
#pragma unroll
    for(int k=0;k<8;++k) a[k]=fmaf(a[k], s, a[(k+1)&7]);
  }
  float t=0; for(int k=0;k<8;++k) t+=a[k]; out[blockIdx.x*blockDim.x+threadIdx.x]=t;
}
__global__ void kffma2(float* out, int iters, float s){
  u64 a[8]; float2 sv = make_float2(s,s); u64 ss=*(u64*)&sv;
  for(int k=0;k<8;++k){ float2 v=make_float2(threadIdx.x*0.001f+k, k*0.5f); a[k]=*(u64*)&v; }
  for(int i=0;i<iters;++i){
#pragma unroll
    for(int k=0;k<8;++k) a[k]=f2(a[k], ss, a[(k+1)&7]);
  }
  float t=0; for(int k=0;k<8;++k){ float2 v=*(float2*)&a[k]; t+=v.x+v.y;} out[blockIdx.x*blockDim.x+threadIdx.x]=t;
}
// mixed: FFMA + LDS + ISETP-like int ops
int main(){
  float* out; cudaMalloc(&out, 148*8*256*4*4);
  int iters=1<<16; cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for(int rep=0;rep<2;++rep){
  for(int w=4; w<=32; w*=2){
    int blocks=148*4, thr=w*32/4; // w warps per SM
    float ms;
    kffma<<<blocks,thr>>>(out,iters,0.999f); cudaEventRecord(e0); kffma<<<blocks,thr>>>(out,iters,0.999f); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
    double fl = 2.0*8*iters*(double)blocks*thr;
    printf("FFMA  warps/SM=%2d  %.1f TFLOP/s  (%.3f ms)\n", w, fl/ms/1e9, ms);
    kffma2<<<blocks,thr>>>(out,iters,0.999f); cudaEventRecord(e0); kffma2<<<blocks,thr>>>(out,iters,0.999f); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
    printf("FFMA2 warps/SM=%2d  %.1f TFLOP/s  (%.3f ms)\n", w, 2*fl/ms/1e9, ms);
  }}
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock %d kHz\n", clk);
  return 0;
}
