// common.cuh — device helpers for the ESPO kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../../include/espo.h"

namespace espo {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kMaxK = ESPO_MAX_BUCKETS;
// Number of fp64 values in the per-rank reduction vector (all-reduced with NCCL).
//  0 ΣJ_i  1 N_active  2 T_active  3 n_zv_groups  4 n_groups  5 n_clipped
//  6 Σ|lp−old|  7 ΣH  8..11 tokens_k  12..15 clipped_k  16..19 Σv_k  20..23 Σε_k
constexpr int kRedLen = 26;

// ----------------------------------------------------------------------------- errors
__device__ __forceinline__ void set_error(int* err, int code) {
  atomicCAS(err, 0, code);  // first error wins; sticky until the next prepare
}

// ----------------------------------------------------------------------------- memory
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// coherent variant for in-place bwd (dlogits aliases logits)
__device__ __forceinline__ uint4 ld_stream_coherent(const void* p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream2(void* p, uint32_t x, uint32_t y) {
  asm volatile("st.global.cs.v2.u32 [%0], {%1,%2};" :: "l"(p), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void st_stream(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// ----------------------------------------------------------------------------- math
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^t on the FMA pipe (FA4-style software exp2): Cody-Waite split t = n + f, f ∈ [-½, ½]
// (magic-number rounding), degree-5 near-minimax polynomial for 2^f (max rel. err 2.3e-7 in
// fp32 evaluation, same class as MUFU ex2.approx), exponent added as integer n << 23.
// t ≤ −127 (incl. −inf) gives 0; NaN propagates. Used for a fraction of the elements so the
// forward sweep is not bound by the MUFU (XU) pipe.
__device__ __forceinline__ float ex2_poly(float t) {
  asm("max.NaN.f32 %0, %0, 0fC2FE0000;" : "+f"(t));  // max(t, -127)
  const float r = t + 12582912.0f;                    // 1.5·2^23: round(t) in the low bits
  const float f = t - (r - 12582912.0f);
  float p = fmaf(0x1.5c08e4p-10f, f, 0x1.3d0c52p-7f);
  p = fmaf(p, f, 0x1.c6b6e4p-5f);
  p = fmaf(p, f, 0x1.ebf918p-3f);
  p = fmaf(p, f, 0x1.62e428p-1f);
  p = fmaf(p, f, 0x1.000002p+0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(r) << 23));
}
// low half via PRMT (ALU pipe) rather than IMAD.SHL (FMA pipe, already the busier one)
__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(__byte_perm(w, 0u, 0x1044)); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// 16-byte vector of logits → EPV floats
template <typename T> struct Vec;
template <> struct Vec<float> {
  static constexpr int EPV = 4;
  static constexpr uint32_t kNegInfWord = 0xff800000u;  // −inf
  static constexpr uint32_t kBigNegWord = 0xf149f2cau;  // −1e30 (finite: 0·(−1e30·λ) = 0)
  // element e of the vector := −1e30 where (e == yoff || e >= keep); compile-time e only
  __device__ __forceinline__ static uint4 patch(uint4 v, int yoff, int keep) {
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (e == yoff || e >= keep) w[e] = kBigNegWord;
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  __device__ __forceinline__ static void unpack(const uint4& v, float* x) {
    x[0] = __uint_as_float(v.x); x[1] = __uint_as_float(v.y);
    x[2] = __uint_as_float(v.z); x[3] = __uint_as_float(v.w);
  }
  __device__ __forceinline__ static float load1(const void* row, int64_t j) {
    return __ldg(reinterpret_cast<const float*>(row) + j);
  }
};
template <> struct Vec<__nv_bfloat16> {
  static constexpr int EPV = 8;
  static constexpr uint32_t kNegInfWord = 0xff80ff80u;  // two bf16 −inf
  static constexpr uint32_t kBigNegWord = 0xf14af14au;  // two bf16 −1.0e30 (finite)
  __device__ __forceinline__ static uint4 patch(uint4 v, int yoff, int keep) {
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (e == yoff || e >= keep)
        w[e >> 1] = (e & 1) ? ((w[e >> 1] & 0x0000ffffu) | 0xf14a0000u)
                            : ((w[e >> 1] & 0xffff0000u) | 0x0000f14au);
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  __device__ __forceinline__ static void unpack(const uint4& v, float* x) {
    x[0] = bf16lo(v.x); x[1] = bf16hi(v.x); x[2] = bf16lo(v.y); x[3] = bf16hi(v.y);
    x[4] = bf16lo(v.z); x[5] = bf16hi(v.z); x[6] = bf16lo(v.w); x[7] = bf16hi(v.w);
  }
  __device__ __forceinline__ static float load1(const void* row, int64_t j) {
    const unsigned short s = __ldg(reinterpret_cast<const unsigned short*>(row) + j);
    return __uint_as_float(static_cast<uint32_t>(s) << 16);
  }
};

// output packing of EPV_in floats into 16-byte vectors of the grad dtype
template <typename Tout> struct Out;
template <> struct Out<float> {
  static constexpr int EPV = 4;
  __device__ __forceinline__ static uint4 pack(const float* d) {
    return make_uint4(__float_as_uint(d[0]), __float_as_uint(d[1]), __float_as_uint(d[2]),
                      __float_as_uint(d[3]));
  }
};
template <> struct Out<__nv_bfloat16> {
  static constexpr int EPV = 8;
  __device__ __forceinline__ static uint4 pack(const float* d) {
    return make_uint4(pack_bf16x2(d[0], d[1]), pack_bf16x2(d[2], d[3]),
                      pack_bf16x2(d[4], d[5]), pack_bf16x2(d[6], d[7]));
  }
};

// ----------------------------------------------------------------------------- TMA bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "ESPO_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra ESPO_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// global → shared bulk copy (TMA engine), completion counted on `bar` in bytes.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(smem_u32(p)));
  return r;
}

// Per-(kernel, device) one-time opt-in to large dynamic shared memory: the attribute is a
// property of the function on the *current* device, so a process driving several GPUs sets it
// once per device (bit d of a per-kernel mask; the race on first use is benign).
template <typename K>
inline cudaError_t ensure_smem_attr(K kernel, int bytes, unsigned long long& done_mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done_mask & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done_mask |= bit;
  return e;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace espo
