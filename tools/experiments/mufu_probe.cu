// Throughput probe: ex2.approx.ftz.f32 vs ex2.approx.f16x2 (results per second per GPU).
#include <cstdio>
#include <cuda_fp16.h>
__global__ void k_f32(float* out, int iters) {
  float a = threadIdx.x * 1e-3f, b = a + 0.5f, c = a + 0.25f, d = a + 0.75f;
  for (int i = 0; i < iters; ++i) {
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(c));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(d));
    a -= 1.f; b -= 1.f; c -= 1.f; d -= 1.f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
__global__ void k_f16x2(float* out, int iters) {
  unsigned a = 0x3c003c00u + threadIdx.x, b = a ^ 1, c = a ^ 2, d = a ^ 3;
  for (int i = 0; i < iters; ++i) {
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a));
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(b));
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(c));
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(d));
    a ^= 0x80008000u; b ^= 0x80008000u; c ^= 0x80008000u; d ^= 0x80008000u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = float(a + b + c + d);
}
__global__ void k_bf16x2(float* out, int iters) {
  unsigned a = 0x3f803f80u + threadIdx.x, b = a ^ 1, c = a ^ 2, d = a ^ 3;
  for (int i = 0; i < iters; ++i) {
    asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a));
    asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(b));
    asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(c));
    asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(d));
    a ^= 0x80008000u; b ^= 0x80008000u; c ^= 0x80008000u; d ^= 0x80008000u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = float(a + b + c + d);
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
  const int iters = 20000, blocks = 148 * 8, th = 256;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(s); k_f32<<<blocks, th>>>(out, iters); cudaEventRecord(e); cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    printf("f32   ex2: %.3e results/s\n", 4.0 * iters * blocks * th / (ms * 1e-3));
    cudaEventRecord(s); k_f16x2<<<blocks, th>>>(out, iters); cudaEventRecord(e); cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    printf("f16x2 ex2: %.3e results/s (2 per instruction)\n", 8.0 * iters * blocks * th / (ms * 1e-3));
    cudaEventRecord(s); k_bf16x2<<<blocks, th>>>(out, iters); cudaEventRecord(e); cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    printf("bf16x2 ex2: %.3e results/s (2 per instruction)\n", 8.0 * iters * blocks * th / (ms * 1e-3));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
