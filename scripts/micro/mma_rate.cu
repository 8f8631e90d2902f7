// Legacy warp-level tensor-core rate on sm_100a (mma.sync -> HMMA): m16n8k4 and m16n8k8 tf32,
// fp32 accumulate, plus a fragment-layout check of m16n8k4 against a CPU product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma1684(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0, const float (&c)[4]) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%7,%8,%9,%10};"
               : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
               : "r"(a0), "r"(a1), "r"(b0), "f"(c[0]), "f"(c[1]), "f"(c[2]), "f"(c[3]));
}
__device__ __forceinline__ void mma1688(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                        uint32_t b1, const float (&c)[4]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%12,%13};"
               : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(c[0]), "f"(c[1]), "f"(c[2]), "f"(c[3]));
}

// rate: each warp issues `iters` x 8 independent MMAs whose C is a fixed register set (the filter's
// usage: fresh C every time, D consumed by one integer op)
template <int K>
__global__ void rate(float* out, int iters) {
  const int lane = threadIdx.x & 31;
  uint32_t a0 = __float_as_uint(1.0f + lane), a1 = __float_as_uint(2.0f), b0 = __float_as_uint(0.5f + lane), b1 = b0;
  float c[4] = {0.1f, 0.2f, 0.3f, 0.4f};
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float d[4];
      if (K == 4) mma1684(d, a0 + u, a1, b0, c);
      else mma1688(d, a0 + u, a1, a0, a1, b0, b1, c);
      acc += __float_as_uint(d[0]) >> 31;
      acc += __float_as_uint(d[3]) >> 31;
    }
    b0 += 1;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}

__global__ void layout(const float* A, const float* B, float* D) {  // A 16x4 row-major, B 4x8 (k, n), D 16x8
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  uint32_t a0 = __float_as_uint(A[g * 4 + t]), a1 = __float_as_uint(A[(g + 8) * 4 + t]);
  uint32_t b0 = __float_as_uint(B[t * 8 + g]);
  float c[4] = {0, 0, 0, 0}, d[4];
  mma1684(d, a0, a1, b0, c);
  D[g * 8 + 2 * t] = d[0];
  D[g * 8 + 2 * t + 1] = d[1];
  D[(g + 8) * 8 + 2 * t] = d[2];
  D[(g + 8) * 8 + 2 * t + 1] = d[3];
}

__global__ void layout8(const float* A, const float* B, float* D) {  // A 16x8 row-major, B 8x8 (k, n), D 16x8; C = 0
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  uint32_t a0 = __float_as_uint(A[g * 8 + t]), a1 = __float_as_uint(A[(g + 8) * 8 + t]);
  uint32_t a2 = __float_as_uint(A[g * 8 + t + 4]), a3 = __float_as_uint(A[(g + 8) * 8 + t + 4]);
  uint32_t b0 = __float_as_uint(B[t * 8 + g]), b1 = __float_as_uint(B[(t + 4) * 8 + g]);
  float d[4];
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%10,%10,%10};"
               : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(0.0f));
  D[g * 8 + 2 * t] = d[0];
  D[g * 8 + 2 * t + 1] = d[1];
  D[(g + 8) * 8 + 2 * t] = d[2];
  D[(g + 8) * 8 + 2 * t + 1] = d[3];
}

int main() {
  float *o, *A, *B, *D;
  cudaMalloc(&o, 148 * 1024 * 4 * 16);
  cudaMallocManaged(&A, 64 * 4);
  cudaMallocManaged(&B, 32 * 4);
  cudaMallocManaged(&D, 128 * 4);
  for (int i = 0; i < 64; ++i) A[i] = (float)((i * 7) % 5) - 2.0f;
  for (int i = 0; i < 32; ++i) B[i] = (float)((i * 3) % 7) - 3.0f;
  layout<<<1, 32>>>(A, B, D);
  cudaDeviceSynchronize();
  int bad = 0;
  for (int m = 0; m < 16; ++m)
    for (int n = 0; n < 8; ++n) {
      float s = 0;
      for (int k = 0; k < 4; ++k) s += A[m * 4 + k] * B[k * 8 + n];
      if (s != D[m * 8 + n]) ++bad;
    }
  printf("m16n8k4 layout check: %d mismatches\n", bad);
  {
    float *A8, *B8;
    cudaMallocManaged(&A8, 128 * 4);
    cudaMallocManaged(&B8, 64 * 4);
    for (int i = 0; i < 128; ++i) A8[i] = (float)((i * 7) % 5) - 2.0f;
    for (int i = 0; i < 64; ++i) B8[i] = (float)((i * 3) % 7) - 3.0f;
    layout8<<<1, 32>>>(A8, B8, D);
    cudaDeviceSynchronize();
    int bad8 = 0;
    for (int m = 0; m < 16; ++m)
      for (int n = 0; n < 8; ++n) {
        float s = 0;
        for (int k = 0; k < 8; ++k) s += A8[m * 8 + k] * B8[k * 8 + n];
        if (s != D[m * 8 + n]) ++bad8;
      }
    printf("m16n8k8 layout check: %d mismatches\n", bad8);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int K = 4; K <= 8; K += 4) {
    for (int wpb : {4, 8, 16}) {
      const int blocks = 148 * (32 / wpb) * 1;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (K == 4) rate<4><<<blocks, 32 * wpb>>>(o, iters);
        else rate<8><<<blocks, 32 * wpb>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double mmas = (double)blocks * wpb * iters * 8;
        const double flops = mmas * 16 * 8 * K * 2;
        if (rep) printf("m16n8k%d: %d warps/block %d blocks: %.3f ms, %.3e mma/s, %.1f TFLOP/s tf32, %.2f mma/clk/SM @1.965GHz\n",
                        K, wpb, blocks, ms, mmas / ms * 1e3, flops / ms * 1e-9, mmas / (ms * 1e-3) / 148 / 1.965e9);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
