// Shared-memory wavefronts per warp-wide load for 32/64/128-bit loads when the 32 lanes read only
// D distinct addresses (D = 1, 2, 4).  Run under ncu and read
// l1tex__data_pipe_lsu_wavefronts_mem_shared_cmd_read.sum / smsp__inst_executed_op_shared_ld.sum.
#include <cstdio>
#include <cuda_runtime.h>
template <int BYTES, int D>
__global__ void k(float* out, int iters) {
  __shared__ __align__(16) float s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned a = (unsigned)__cvta_generic_to_shared(s) + (unsigned)((lane % D) * 16);
  float acc = 0;
  for (int it = 0; it < iters; ++it) {
    unsigned ad = a + ((it * 64) & 8191);
    if (BYTES == 4) { float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(ad)); acc += v; }
    if (BYTES == 8) { float v0, v1; asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v0), "=f"(v1) : "r"(ad)); acc += v0 + v1; }
    if (BYTES == 16) { float v0, v1, v2, v3; asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v0), "=f"(v1), "=f"(v2), "=f"(v3) : "r"(ad)); acc += v0 + v1 + v2 + v3; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  float* o; cudaMalloc(&o, 1 << 20);
  k<4, 1><<<1, 32>>>(o, 1000); k<4, 2><<<1, 32>>>(o, 1000);
  k<8, 1><<<1, 32>>>(o, 1000); k<8, 2><<<1, 32>>>(o, 1000); k<8, 4><<<1, 32>>>(o, 1000);
  k<16, 1><<<1, 32>>>(o, 1000); k<16, 2><<<1, 32>>>(o, 1000);
  cudaDeviceSynchronize();
  printf("ok\n");
  return 0;
}
