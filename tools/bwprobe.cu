// bwprobe.cu — HBM ceilings of the data-movement primitives the ESPO sweeps are built from,
// measured on the B200 with CUDA events (10 GB buffers, best of 10):
//   read_ldg     : 128-bit LDG grid-stride, xor-reduced (read-only ceiling)
//   read_tma     : per-warp 3-stage cp.async.bulk ring, 4 KB chunks, lane reads (K2 shape)
//   write_stg    : 128-bit STG.cs zero fill
//   write_bulk   : cp.async.bulk shared→global of a zeroed 4 KB smem tile
//   copy_ldgstg  : LDG → STG.cs
//   copy_tma_stg : TMA ring load → STG.cs (K5 shape)
//   copy_tma_bulk: TMA ring load → smem staging → bulk store
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o bwprobe tools/bwprobe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void s2g(void* g, const void* s, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(su32(s)), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ uint4 ldg(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
#ifndef STG_HINT
#define STG_HINT ".cs"
#endif
__device__ __forceinline__ void stg(void* p, uint4 v) {
  asm volatile("st.global" STG_HINT ".v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

__global__ void read_ldg(const uint4* a, size_t n, uint32_t* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x * 4) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) { size_t j = i + (size_t)k * gridDim.x * blockDim.x; v[k] = j < n ? ldg(a + j) : make_uint4(0, 0, 0, 0); }
#pragma unroll
    for (int k = 0; k < 4; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  if (acc == 0x12345678) *out = acc;
}

__global__ void write_stg(uint4* a, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    stg(a + i, make_uint4(0, 0, 0, 0));
}

__global__ void copy_ldgstg(const uint4* a, uint4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x * 4) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) { size_t j = i + (size_t)k * gridDim.x * blockDim.x; if (j < n) v[k] = ldg(a + j); }
#pragma unroll
    for (int k = 0; k < 4; ++k) { size_t j = i + (size_t)k * gridDim.x * blockDim.x; if (j < n) stg(b + j, v[k]); }
  }
}

__global__ void copy_tile(const uint4* a, uint4* b, size_t n) {
  const size_t base = blockIdx.x * (size_t)blockDim.x * 4 + threadIdx.x;
  uint4 v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { size_t j = base + k * blockDim.x; if (j < n) v[k] = ldg(a + j); }
#pragma unroll
  for (int k = 0; k < 4; ++k) { size_t j = base + k * blockDim.x; if (j < n) stg(b + j, v[k]); }
}

// per-warp ring over contiguous 4 KB chunks (chunk c of warp w = w + c*nwarps)
template <int NW, int ST, int MODE, int CH = 4096>  // MODE 0 read, 1 copy via STG, 2 copy via bulk store
__global__ void __launch_bounds__(NW * 32, 1) ring(const char* a, char* b, size_t nchunks, uint32_t* out) {
  constexpr int VL = CH / 512;
  extern __shared__ __align__(128) uint8_t sm[];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  uint8_t* rg = sm + (size_t)w * ST * CH;
  uint8_t* ob = sm + (size_t)NW * ST * CH + (size_t)w * 2 * CH;
  uint64_t* bar = (uint64_t*)(sm + (size_t)NW * ST * CH + (MODE == 2 ? (size_t)NW * 2 * CH : 0)) + w * ST;
  if (l == 0) { for (int s = 0; s < ST; ++s) mbar_init(&bar[s], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncwarp();
  const size_t gw = blockIdx.x * (size_t)NW + w, nw = (size_t)gridDim.x * NW;
  size_t pc = gw;
  uint32_t q = 0, issued = 0;
  for (int s = 0; s < ST && pc < nchunks; ++s, pc += nw, ++issued) if (l == 0) { mbar_tx(&bar[s], CH); g2s(rg + s * CH, a + pc * CH, CH, &bar[s]); }
  uint32_t acc = 0;
  for (size_t c = gw; c < nchunks; c += nw, ++q) {
    const int s = q % ST;
    mbar_wait(&bar[s], (q / ST) & 1);
    uint4 v[VL];
#pragma unroll
    for (int u = 0; u < VL; ++u) v[u] = *(const uint4*)(rg + s * CH + (l + 32 * u) * 16);
    __syncwarp();
    if (pc < nchunks) { if (l == 0) { mbar_tx(&bar[s], CH); g2s(rg + s * CH, a + pc * CH, CH, &bar[s]); } pc += nw; }
    if (MODE == 0) {
#pragma unroll
      for (int u = 0; u < VL; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    } else if (MODE == 1) {
#pragma unroll
      for (int u = 0; u < VL; ++u) stg(b + c * CH + (l + 32 * u) * 16, v[u]);
    } else {
      uint8_t* o = ob + (q & 1) * CH;
      if (l == 0) bulk_wait_read<1>();
      __syncwarp();
#pragma unroll
      for (int u = 0; u < VL; ++u) *(uint4*)(o + (l + 32 * u) * 16) = v[u];
      fence_async();
      __syncwarp();
      if (l == 0) { s2g(b + c * CH, o, CH); bulk_commit(); }
    }
  }
  if (MODE == 2 && l == 0) bulk_wait_read<0>();
  if (acc == 0x12345678) *out = acc;
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) write_bulk(char* b, size_t nchunks) {
  constexpr int CH = 4096;
  __shared__ __align__(128) uint8_t z[CH];
  for (int i = threadIdx.x; i < CH / 16; i += blockDim.x) ((uint4*)z)[i] = make_uint4(0, 0, 0, 0);
  fence_async();
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l) return;
  const size_t gw = blockIdx.x * (size_t)NW + w, nw = (size_t)gridDim.x * NW;
  int k = 0;
  for (size_t c = gw; c < nchunks; c += nw) {
    s2g(b + c * CH, z, CH);
    bulk_commit();
    if (++k >= 8) bulk_wait_read<7>();
  }
  bulk_wait_read<0>();
}

template <int NW, int ST, int MODE, int CH>
void probe_ring(const char* name, char* a, char* b, size_t bytes, uint32_t* out, int sms, cudaEvent_t e0,
                cudaEvent_t e1) {
  const size_t smem = (size_t)NW * ST * CH + (MODE == 2 ? (size_t)NW * 2 * CH : 0) + 1024;
  if (smem > 227 * 1024) return;
  cudaFuncSetAttribute(ring<NW, ST, MODE, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const size_t nch = bytes / CH;
  auto fn = [&] { ring<NW, ST, MODE, CH><<<sms, NW * 32, smem>>>(a, b, nch, out); };
  for (int i = 0; i < 3; ++i) fn();
  float best = 1e30f;
  for (int i = 0; i < 10; ++i) {
    cudaEventRecord(e0); fn(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  const double traffic = (MODE == 0 ? 1.0 : 2.0) * bytes;
  printf("{\"probe\": \"%s_%dx%dx%dk\", \"GBps\": %.1f, \"err\": \"%s\"}\n", name, NW, ST, CH / 1024,
         traffic / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t bytes = 10ull << 30, n16 = bytes / 16, nch = bytes / 4096;
  char *a, *b;
  uint32_t* out;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMalloc(&out, 4);
  cudaMemset(a, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(ring<16, 3, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 3 * 4096 + 1024);
  cudaFuncSetAttribute(ring<8, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * 4096 + 1024);
  cudaFuncSetAttribute(ring<8, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * 4096 + 8 * 2 * 4096 + 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, double traffic, auto fn) {
    for (int i = 0; i < 3; ++i) fn();
    float best = 1e30f;
    for (int i = 0; i < 10; ++i) {
      cudaEventRecord(e0); fn(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("{\"probe\": \"%s\", \"GBps\": %.1f, \"err\": \"%s\"}\n", name, traffic / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  run("read_ldg", bytes, [&] { read_ldg<<<sms * 8, 256>>>((const uint4*)a, n16, out); });
  run("read_tma_16x3x4k", bytes, [&] { ring<16, 3, 0><<<sms, 512, 16 * 3 * 4096 + 1024>>>(a, b, nch, out); });
  run("write_stg", bytes, [&] { write_stg<<<sms * 8, 256>>>((uint4*)b, n16); });
  run("write_bulk", bytes, [&] { write_bulk<8><<<sms, 256>>>(b, nch); });
  run("copy_ldgstg", 2.0 * bytes, [&] { copy_ldgstg<<<sms * 8, 256>>>((const uint4*)a, (uint4*)b, n16); });
  run("copy_tma_stg_8x4x4k", 2.0 * bytes, [&] { ring<8, 4, 1><<<sms, 256, 8 * 4 * 4096 + 1024>>>(a, b, nch, out); });
  run("copy_tma_bulk_8x4x4k", 2.0 * bytes, [&] { ring<8, 4, 2><<<sms, 256, 8 * 4 * 4096 + 8 * 2 * 4096 + 1024>>>(a, b, nch, out); });
  run("copy_tile_np", 2.0 * bytes, [&] { copy_tile<<<(unsigned)((n16 + 1023) / 1024), 256>>>((const uint4*)a, (uint4*)b, n16); });
  if (0) {
  probe_ring<16, 3, 0, 4096>("read_tma", a, b, bytes, out, sms, e0, e1);
  probe_ring<16, 2, 0, 4096>("read_tma", a, b, bytes, out, sms, e0, e1);
  probe_ring<8, 3, 0, 8192>("read_tma", a, b, bytes, out, sms, e0, e1);
  probe_ring<12, 2, 0, 8192>("read_tma", a, b, bytes, out, sms, e0, e1);
  probe_ring<8, 2, 0, 12288>("read_tma", a, b, bytes, out, sms, e0, e1);
  probe_ring<4, 3, 0, 16384>("read_tma", a, b, bytes, out, sms, e0, e1);
  probe_ring<6, 2, 0, 16384>("read_tma", a, b, bytes, out, sms, e0, e1);
  probe_ring<24, 2, 0, 4096>("read_tma", a, b, bytes, out, sms, e0, e1);
  probe_ring<8, 6, 0, 4096>("read_tma", a, b, bytes, out, sms, e0, e1);
  }
  probe_ring<8, 4, 1, 4096>("copy_tma_stg", a, b, bytes, out, sms, e0, e1);
  probe_ring<8, 3, 1, 8192>("copy_tma_stg", a, b, bytes, out, sms, e0, e1);
  probe_ring<16, 3, 1, 4096>("copy_tma_stg", a, b, bytes, out, sms, e0, e1);
  probe_ring<4, 3, 1, 16384>("copy_tma_stg", a, b, bytes, out, sms, e0, e1);
  for (int cpb : {8, 16}) {
    char nm[64]; sprintf(nm, "read_ldg_%dcta", cpb);
    run(nm, bytes, [&] { read_ldg<<<sms * cpb, 256>>>((const uint4*)a, n16, out); });
    sprintf(nm, "copy_ldgstg_%dcta", cpb);
    run(nm, 2.0 * bytes, [&] { copy_ldgstg<<<sms * cpb, 256>>>((const uint4*)a, (uint4*)b, n16); });
  }
  return 0;
}
