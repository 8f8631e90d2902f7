// Shared-memory wavefronts of warp-wide LDS.64 when the 32 lanes read D distinct 8-byte words that are
// ADJACENT (spacing 8 B) or spread (spacing 16 B / far apart).  Run under ncu:
// l1tex__data_pipe_lsu_wavefronts_mem_shared_cmd_read.sum / smsp__inst_executed_op_shared_ld.sum
#include <cstdio>
#include <cuda_runtime.h>
template <int D, int SPACING>
__global__ void k(float* out, int iters) {
  __shared__ __align__(16) float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i * 0.5f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned a = (unsigned)__cvta_generic_to_shared(s) + (unsigned)((lane % D) * SPACING);
  float acc = 0;
  for (int it = 0; it < iters; ++it) {
    unsigned ad = a + ((it * 64) & 4095);
    float v0, v1;
    asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v0), "=f"(v1) : "r"(ad));
    acc += v0 + v1;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  float* o; cudaMalloc(&o, 1 << 20);
  k<2, 8><<<1, 32>>>(o, 1000); k<3, 8><<<1, 32>>>(o, 1000); k<4, 8><<<1, 32>>>(o, 1000);
  k<8, 8><<<1, 32>>>(o, 1000); k<16, 8><<<1, 32>>>(o, 1000); k<32, 8><<<1, 32>>>(o, 1000);
  k<2, 1160><<<1, 32>>>(o, 1000); k<3, 1160><<<1, 32>>>(o, 1000); k<4, 1160><<<1, 32>>>(o, 1000);
  cudaDeviceSynchronize();
  printf("ok\n");
  return 0;
}
