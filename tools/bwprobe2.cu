// bwprobe2.cu — non-persistent tiled COPY ceilings (the K5 shape: one CTA per tile, the grid
// walks a 10 GB buffer once), CUDA events, best of 10:
//   tile_ldg<T,V>   : T threads × V 16-byte vectors per thread, LDG.nc → STG (.cs by default)
//   tile_tma<B>     : one thread bulk-loads a B-byte tile (cp.async.bulk) into smem, all
//                     threads read it and write with STG.cs
//   tile_dma<B>     : bulk load into smem then bulk store (no register pass: pure TMA copy)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o bwprobe2 tools/bwprobe2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint4 ldg(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg_cs(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void stg_def(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void stg_na(void* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void s2g(void* g, const void* s, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(su32(s)), "r"(n) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

template <int T, int V, int ST>
__global__ void __launch_bounds__(T) tile_ldg(const uint4* a, uint4* b) {
  const size_t base = (size_t)blockIdx.x * T * V + threadIdx.x;
  uint4 v[V];
#pragma unroll
  for (int k = 0; k < V; ++k) v[k] = ldg(a + base + (size_t)k * T);
#pragma unroll
  for (int k = 0; k < V; ++k) {
    if (ST == 0) stg_cs(b + base + (size_t)k * T, v[k]);
    else if (ST == 1) stg_def(b + base + (size_t)k * T, v[k]);
    else stg_na(b + base + (size_t)k * T, v[k]);
  }
}

template <int B>
__global__ void __launch_bounds__(256) tile_tma(const char* a, char* b) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = (uint64_t*)(sm + B);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_tx(bar, B);
    g2s(sm, a + (size_t)blockIdx.x * B, B, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < B / 16; i += 256)
    stg_cs(b + (size_t)blockIdx.x * B + i * 16, ((const uint4*)sm)[i]);
}

template <int B>
__global__ void __launch_bounds__(32) tile_dma(const char* a, char* b) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = (uint64_t*)(sm + B);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_tx(bar, B);
    g2s(sm, a + (size_t)blockIdx.x * B, B, bar);
    mbar_wait(bar, 0);
    s2g(b + (size_t)blockIdx.x * B, sm, B);
  }
}

int main() {
  const size_t bytes = 10ull << 30;
  char *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMemset(a, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto fn) {
    for (int i = 0; i < 3; ++i) fn();
    float best = 1e30f;
    for (int i = 0; i < 10; ++i) {
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("{\"probe\": \"%s\", \"GBps\": %.1f, \"err\": \"%s\"}\n", name, 2.0 * bytes / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
#define LDG(T, V, S, NAME)                                                                       \
  run(NAME, [&] { tile_ldg<T, V, S><<<(unsigned)(bytes / (16ull * T * V)), T>>>((const uint4*)a, (uint4*)b); })
  LDG(256, 4, 0, "ldg_256x4_cs_16k");
  LDG(256, 8, 0, "ldg_256x8_cs_32k");
  LDG(256, 16, 0, "ldg_256x16_cs_64k");
  LDG(512, 8, 0, "ldg_512x8_cs_64k");
  LDG(128, 8, 0, "ldg_128x8_cs_16k");
  LDG(256, 8, 1, "ldg_256x8_def_32k");
  LDG(256, 8, 2, "ldg_256x8_na_32k");
#define TMA(B, NAME)                                                                            \
  cudaFuncSetAttribute(tile_tma<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, B + 64);     \
  run(NAME, [&] { tile_tma<B><<<(unsigned)(bytes / B), 256, B + 64>>>(a, b); })
  TMA(16384, "tma_16k");
  TMA(32768, "tma_32k");
  TMA(65536, "tma_64k");
#define DMA(B, NAME)                                                                            \
  cudaFuncSetAttribute(tile_dma<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, B + 64);     \
  run(NAME, [&] { tile_dma<B><<<(unsigned)(bytes / B), 32, B + 64>>>(a, b); })
  DMA(16384, "dma_16k");
  DMA(32768, "dma_32k");
  DMA(65536, "dma_64k");
  return 0;
}
