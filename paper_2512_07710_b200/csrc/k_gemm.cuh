// k_gemm.cuh — the library's tcgen05 GEMM core: the fused LM head's contractions (SURVEY §8(f)
// row 1; the Megatron log-prob recompute of PAPER.md:129-131). With logits z = h·Wᵀ:
//   forward   z tiles → per-row partials {R, S, W, u_y}  A = h (K-major), B = W (K-major)
//   recompute z tiles → dz = ∂(grad·loss)/∂z (bf16)     A = h (K-major), B = W (K-major)
//   dh = dz · W      M = rows,  N = d, K = vocabulary   A = dz  (K-major), B = W (MN-major)
//   dW += dzᵀ · h    M = vocab, N = d, K = rows         A = dzᵀ (MN-major), B = h (MN-major)
// Every operand stays in the layout the caller (or the recompute) produced — no transposed
// copies: tcgen05 reads MN-major bf16 tiles directly (instruction-descriptor bits 15/16).
//
// Persistent, warp-specialised kernels: warp 0 = TMA producer (a ring of {A, B} K-slices with
// 128-byte swizzle), warp 1 = TMEM allocator and the one thread issuing tcgen05.mma
// (kind::f16, fp32 accumulators in TMEM, completion by tcgen05.commit → mbarrier), the other
// warps = epilogue (tcgen05.ld 32 columns at a time: fp32 / bf16 store, fp32 read-add-write,
// or the LM-head reductions). Variants:
//   k_umma_gemm   one CTA per 128 × 256 tile, two TMEM accumulators (epilogue overlapped);
//   k_umma_gemm2  CTA pairs (cta_group::2, M = 256 split over the pair's SMs, B columns split
//                 likewise): 256 × 256 tiles (two accumulators) or 256 × 512 (one 512-column
//                 accumulator = all of TMEM, a quarter less L2 → SM traffic per FLOP, released
//                 in two column halves so the next tile's first K-steps overlap the epilogue),
//                 8 epilogue warps; grouped tile raster taken in order by a dynamic scheduler
//                 (atomic counter, work items handed to the pair's roles through a
//                 shared-memory queue), L2 cache-policy hints, device-side row counts
//                 (compacted operands), split-K over 2 (deterministic), soft lockstep between
//                 the clusters of a wave, fp32 accumulation into C by TMA reduce-add;
//   k_umma_gemm4  two pairs per cluster sharing A through TMA multicast (an option: only 33
//                 four-CTA clusters are resident on a B200, 132 of 148 SMs).
// Grids are sized from the resident cluster count (host side). Every barrier wait is bounded by
// the global timer: a protocol error traps instead of hanging the GPU.
//
// Shared-memory operand layouts (UMMA canonical forms, SWIZZLE_128B, 1024-B aligned):
//  K-major : rows of 64 K-elements (128 B), 8-row groups 1024 B apart (one TMA box
//            {64 K, rows}); +32 B per K = 16 step inside the swizzle atom.
//  MN-major: lines of 64 MN-elements (128 B), one line per K index, 8-line groups 1024 B
//            apart (SBO); 64-wide MN blocks 8 KB apart (LBO) = one TMA box {64 MN, 64 K}
//            each; +2048 B (16 lines) per K = 16 step.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "k_lmhead.cuh"
#include "k_lmhead2.cuh"

namespace espo {

constexpr int kGmBM = 128, kGmBN = 256, kGmBK = 64, kGmStages = 4;
constexpr int kGmABytes = kGmBM * kGmBK * 2;    // 16 KB
constexpr int kGmBBytes = kGmBN * kGmBK * 2;    // 32 KB
constexpr int kGmStageBytes = kGmABytes + kGmBBytes;
constexpr int kGmMNBox = 64 * kGmBK * 2;        // one MN-major TMA box {64 MN, 64 K}: 8 KB
constexpr int kGmThreads = 192;
constexpr int kG2Threads = 320;   // CTA-pair kernel: producer, MMA, 8 epilogue warps (two per
                                  // TMEM lane quarter, each draining half of the tile's columns)
constexpr size_t kGmSmem = size_t(kGmStages) * kGmStageBytes + 1024 + 256;

enum GemmOut { kOutF32 = 0, kOutBF16 = 1, kOutAddF32 = 2, kOutLmFwd = 3, kOutLmDz = 4 };

// Epilogue data of the LM-head kernels on this GEMM (C = logits tile z = h·Wᵀ, never stored):
// kOutLmFwd — per row and tile, the base-2 partial {R, S, W, u_y} of the tile's columns
// (K2's reduction, lm_row_chunk), written to partial[n-block][row]; k_fwd_combine merges the
// tiles exactly like vocabulary shards. kOutLmDz — K5's dz = λg(1[v=y] − p_v) of every element
// from the row's record, rounded to bf16 into dz[row][col] (lm_store_dz).
struct LmEpi {
  const int32_t* tokens;   // chunk-relative sampled tokens (fwd)
  const uint8_t* flag;     // chunk-relative valid flags (fwd)
  const BwdRec* rec;       // per-row backward records (dz)
  const uint8_t* mlive;    // per M-tile: 0 = no row to compute, the tile is skipped (nullable)
  float4* partial;         // [n-blocks][n_rows] (fwd)
  __nv_bfloat16* dz;       // [rows][ldz] (dz)
  int64_t ldz;
  float lamL;              // λ·log2(e)
  int V;                   // vocabulary columns (columns ≥ V are excluded / written as 0)
  int n_rows;              // partial row stride
  int* err;
};

struct GemmParams {
  int M, N, K;        // C[M, N] (+)= A[M, K] · B[K, N]
  int mblk, nblk, kblk;   // tile counts (tile = kGmBM × kGmBN, or 2·kGmBM × kGmBN for a pair)
  int group_m;        // tile order: groups of group_m M-blocks, M fastest inside a group
  int group_n;        // > 0: instead, groups of group_n N-blocks (N fastest, then M)
  int hint_a, hint_b, hint_c;   // L2 policy of A / B loads and C read-add-write: 0 normal,
                                // 1 evict_first (streamed), 2 evict_last (reused)
  void* C;
  int64_t ldc;        // elements
  // compacted operands (k_compact.cuh): the true M (dyn_which = 1) or K (= 2) is
  // clamp(*dyn_count − dyn_base, 0, M or K) rows, read on the device; row_map (nullable)
  // sends output row r to C row row_map[r]
  const int* dyn_count;
  int dyn_base, dyn_which;
  const int* row_map;
  // soft lockstep (CTA-pair kernel): the tiles of one wave (the i-th tile of every cluster)
  // read the same K-slices of their A and B panels; a cluster that is more than sync_slack
  // chunks of sync_chunk K-steps ahead of the slowest cluster of its wave waits (bounded by
  // ~sync_timeout_ns, then proceeds), so the panels' K-slices are reused from L2 instead of
  // being re-read from DRAM by clusters that drifted apart. sync (nullable) = one zeroed
  // counter per wave.
  unsigned* sync;
  int sync_chunk, sync_slack;
  unsigned sync_timeout_ns;
  LmEpi lm;               // kOutLmFwd / kOutLmDz only
  // split-K over 2 (kOutF32, CTA-pair kernels): work item t < 2·tiles covers tile t % tiles
  // for K-half t / tiles; K-half 0 writes C, K-half 1 writes split_out[row][col] (fp32,
  // pitch split_ld, compact row index); k_split_fixup adds it into C afterwards
  int ksplit;
  float* split_out;
  int64_t split_ld;
  int half_release;       // 512-column accumulators: overlap the next tile's first K-steps on
                          // half 0 with the epilogue's read of half 1 (1, default) or not (0)
  // dynamic tile scheduler (CTA-pair kernel; nullable = static round robin): a zeroed
  // counter; each pair's leader takes the next work item with an atomic add and hands it to
  // the pair's other roles through a small shared-memory queue, so the items in flight stay a
  // contiguous window of the raster (a static round robin spreads them as clusters drift)
  int* tile_ctr;
  // kOutAddF32 on CTA pairs: 1 = the epilogue stages each 32 × 32 fp32 block in shared memory
  // and adds it into C with a TMA reduce (cp.reduce.async.bulk.tensor .add) instead of an
  // SM-side read-add-write (the third tensor map of the launch describes C)
  int tma_red;
};

// wait until *ctr ≥ target or the timeout expired (acquire; a soft barrier: never deadlocks)
__device__ __forceinline__ void soft_wait(const unsigned* ctr, unsigned target, unsigned timeout_ns) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
  if (v >= target) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    __nanosleep(64);
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= target) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) return;
  }
}

// the launch's sizes with a device-side row count applied (uniform in every thread)
__device__ __forceinline__ GemmParams gemm_effective(const GemmParams& p, int bm) {
  GemmParams q = p;
  if (p.dyn_count) {
    const int n = max(0, *p.dyn_count - p.dyn_base);
    if (p.dyn_which == 1 || p.dyn_which == 3) {   // 3: rows up to the next 256 (zero records)
      q.M = min(p.M, p.dyn_which == 3 ? (n + 255) / 256 * 256 : n);
      q.mblk = (q.M + bm - 1) / bm;
    } else {
      q.K = min(p.K, n);
      q.kblk = (q.K + kGmBK - 1) / kGmBK;
    }
  }
  return q;
}

// tile index → (M block, N block): groups of group_m M-blocks; inside a group M varies
// fastest, so the tiles resident together cover ≈ group_m × (resident / group_m) blocks
// (group_m = 1: N fastest)
__device__ __forceinline__ void gemm_tile_coords(const GemmParams& p, int tile, int& mb, int& nb) {
  if (p.group_n > 0) {       // groups of group_n N-blocks; N fastest inside a group, then M
    const int per_group = p.group_n * p.mblk;
    const int g = tile / per_group, rem = tile - g * per_group;
    const int first = g * p.group_n;
    const int gn = min(p.nblk - first, p.group_n);
    nb = first + rem % gn;
    mb = rem / gn;
    return;
  }
  const int per_group = p.group_m * p.nblk;
  const int g = tile / per_group, rem = tile - g * per_group;
  const int first = g * p.group_m;
  const int gm = min(p.mblk - first, p.group_m);
  mb = first + rem % gm;
  nb = rem / gm;
}

// mbarrier wait bounded by the device's global timer: a protocol error traps (a CUDA error
// the host sees) instead of hanging the GPU.
__device__ __forceinline__ void gm_wait(uint64_t* bar, uint32_t parity) {
  uint64_t t0 = 0;
  for (uint32_t it = 0;; ++it) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    if (ok) return;
    if ((it & 255u) == 255u) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > 20000000000ull) __trap();     // 20 s
    }
  }
}

__device__ __forceinline__ uint64_t l2_policy(int hint) {
  uint64_t pol;
  if (hint == 1)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else if (hint == 2)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int c0, int c1,
                                                 uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair_hint(uint32_t dst, const CUtensorMap* map, int c0,
                                                      int c1, uint32_t cluster_bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(cluster_bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ float4 ld_f4_hint(const float4* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_f4_hint(float4* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}

// UMMA shared-memory descriptor for an MN-major SWIZZLE_128B operand (see header comment)
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr & 0x3FFFF) >> 4);        // start address
  d |= uint64_t(kGmMNBox >> 4) << 16;           // LBO: next 64-element MN block
  d |= uint64_t(1024 >> 4) << 32;               // SBO: next group of 8 K lines
  d |= uint64_t(1) << 46;                       // version (Blackwell)
  d |= uint64_t(2) << 61;                       // SWIZZLE_128B
  return d;
}

template <bool kAMN, bool kBMN>
__host__ __device__ constexpr uint32_t gemm_idesc() {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(kAMN) << 15) | (uint32_t(kBMN) << 16) |
         (uint32_t(kGmBN >> 3) << 17) | (uint32_t(kGmBM >> 4) << 24);
}

// Epilogue of one tile for TMEM lane `row` (= output row r): 8 × 32 columns from TMEM →
// C[r, n0 + …] as fp32, bf16 or fp32 read-add-write; rows ≥ M and columns ≥ N skipped.
template <int kOut>
__device__ __forceinline__ void gemm_store_tile(const GemmParams& p, uint32_t base, int r, int n0,
                                                uint64_t pol_c, int nchunk = kGmBN / 32) {
#pragma unroll 1
  for (int c = 0; c < nchunk; ++c) {
    float x[32];
    __syncwarp();
    tmem_ld32(base + uint32_t(c * 32), x);
    const int col0 = n0 + c * 32;
    if (r >= p.M || col0 >= p.N) continue;
    const int orow = p.row_map ? p.row_map[r] : r;
    const bool full_cols = col0 + 32 <= p.N;
    if constexpr (kOut == kOutBF16) {
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.C) + int64_t(orow) * p.ldc + col0;
      if (full_cols) {
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(x[2 * e], x[2 * e + 1]);
          w[e] = *reinterpret_cast<const uint32_t*>(&h2);
        }
        uint4* o4 = reinterpret_cast<uint4*>(o);
#pragma unroll
        for (int e = 0; e < 4; ++e) o4[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (col0 + e < p.N) o[e] = __float2bfloat16_rn(x[e]);
      }
    } else {
      float* o = static_cast<float*>(p.C) + int64_t(orow) * p.ldc + col0;
      if (full_cols) {
        float4* o4 = reinterpret_cast<float4*>(o);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float4 v = make_float4(x[4 * e], x[4 * e + 1], x[4 * e + 2], x[4 * e + 3]);
          if constexpr (kOut == kOutAddF32) {
            const float4 u = ld_f4_hint(o4 + e, pol_c);
            v.x += u.x;
            v.y += u.y;
            v.z += u.z;
            v.w += u.w;
            st_f4_hint(o4 + e, v, pol_c);
          } else {
            o4[e] = v;
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (col0 + e < p.N) o[e] = kOut == kOutAddF32 ? o[e] + x[e] : x[e];
      }
    }
  }
}

// LM-head epilogues over 256 TMEM columns (tile columns n0 .. n0 + 255) for output row r.
// Forward: (R, S, W, cS, cW, uy) carry across the calls for the tile's halves.
__device__ __forceinline__ void lm_fwd_cols(const GemmParams& p, uint32_t base, int r, int n0,
                                            float& R, float& S, float& W, float& cS, float& cW,
                                            float& uy, bool valid, int y, int nchunk) {
#pragma unroll 1
  for (int c = 0; c < nchunk; ++c) {
    float x[32];
    __syncwarp();
    tmem_ld32(base + uint32_t(c * 32), x);
    const int col0 = n0 + c * 32;
    if (!valid || col0 >= p.lm.V) continue;
    lm_row_chunk(x, col0, y, p.lm.V, p.lm.lamL, R, S, W, cS, cW, uy, p.lm.err);
  }
}
__device__ __forceinline__ void lm_dz_cols(const GemmParams& p, uint32_t base, int r, int n0,
                                           const BwdRec& rc, int nchunk) {
#pragma unroll 1
  for (int c = 0; c < nchunk; ++c) {
    float x[32];
    __syncwarp();
    tmem_ld32(base + uint32_t(c * 32), x);
    const int col0 = n0 + c * 32;
    if (r >= p.M || col0 >= p.lm.ldz) continue;
    lm_store_dz(x, rc, col0, p.lm.V, p.lm.lamL, p.lm.dz + int64_t(r) * p.lm.ldz + col0);
  }
}

template <bool kAMN, bool kBMN, int kOut>
__global__ void __launch_bounds__(kGmThreads, 1)
    k_umma_gemm(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                const GemmParams p0) {
  const GemmParams p = gemm_effective(p0, kGmBM);
  if (p.mblk * p.nblk == 0 || p.kblk == 0) return;   // nothing to add (uniform in the grid)
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);   // 1024-B aligned (SW128)
  uint8_t* sA = smem;
  uint8_t* sB = smem + kGmStages * kGmABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kGmStages * kGmStageBytes);
  uint64_t* empty = full + kGmStages;
  uint64_t* tfull = empty + kGmStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles = p.mblk * p.nblk;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kGmStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kGmBM);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pa = l2_policy(p.hint_a), pb = l2_policy(p.hint_b);
      uint32_t q = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        int mb, nb;
        gemm_tile_coords(p, tile, mb, nb);
        const int m0 = mb * kGmBM, n0 = nb * kGmBN;
        for (int kb = 0; kb < p.kblk; ++kb, ++q) {
          const int s = q % kGmStages;
          const int k0 = kb * kGmBK;
          gm_wait(&empty[s], ((q / kGmStages) & 1u) ^ 1u);
          mbar_arrive_tx(&full[s], kGmStageBytes);
          uint8_t* a = sA + s * kGmABytes;
          uint8_t* b = sB + s * kGmBBytes;
          if constexpr (kAMN) {
#pragma unroll
            for (int j = 0; j < kGmBM / 64; ++j) tma_load_2d_hint(a + j * kGmMNBox, &tmap_a, m0 + 64 * j, k0, &full[s], pa);
          } else {
            tma_load_2d_hint(a, &tmap_a, k0, m0, &full[s], pa);
          }
          if constexpr (kBMN) {
#pragma unroll
            for (int j = 0; j < kGmBN / 64; ++j) tma_load_2d_hint(b + j * kGmMNBox, &tmap_b, n0 + 64 * j, k0, &full[s], pb);
          } else {
            tma_load_2d_hint(b, &tmap_b, k0, n0, &full[s], pb);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = gemm_idesc<kAMN, kBMN>();
      uint32_t q = 0;
      int i = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
        const int acc = i & 1;
        gm_wait(&tempty[acc], ((i >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t dt = tmem + uint32_t(acc * kGmBN);
        for (int kb = 0; kb < p.kblk; ++kb, ++q) {
          const int s = q % kGmStages;
          gm_wait(&full[s], (q / kGmStages) & 1u);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * kGmABytes), b0 = smem_u32(sB + s * kGmBBytes);
#pragma unroll
          for (int k = 0; k < kGmBK / 16; ++k) {
            const uint64_t ad = kAMN ? umma_desc_sw128_mn(a0 + k * 2048) : umma_desc_sw128(a0 + k * 32);
            const uint64_t bd = kBMN ? umma_desc_sw128_mn(b0 + k * 2048) : umma_desc_sw128(b0 + k * 32);
            tc_mma(dt, ad, bd, idesc, (kb | k) != 0);
          }
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint64_t pol_c = l2_policy(p.hint_c);
    int i = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
      const int acc = i & 1;
      int mb, nb;
      gemm_tile_coords(p, tile, mb, nb);
      const int m0 = mb * kGmBM, n0 = nb * kGmBN;
      const int r = m0 + row;
      gm_wait(&tfull[acc], (i >> 1) & 1u);
      tc_fence_after();
      const uint32_t base = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(acc * kGmBN);
      gemm_store_tile<kOut>(p, base, r, n0, pol_c);
      __syncwarp();
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------------------
// CTA-pair variant (tcgen05.mma.cta_group::2): one 256 × 256 tile per cluster of two SMs.
// CTA `rank` loads its 128 rows of A and its 128 columns of B (half the B traffic of two
// independent 128 × 256 tiles: per K-step 32 KB per CTA for 4.2 MFLOP instead of 48 KB); the
// leader issues M = 256 MMAs over both CTAs' shared memory and commits to both CTAs' barriers
// (multicast); each CTA's epilogue drains its own TMEM rows (the k_lmhead2.cuh protocol).
// kNP = N columns per pair tile: 256 (two 256-column TMEM accumulators, so the next tile's
// MMAs overlap this tile's epilogue) or 512 (one 512-column accumulator = all of TMEM; per
// K-step 48 KB per CTA for 8.4 MFLOP instead of 32 KB for 4.2: a quarter less L2 → SM traffic,
// the epilogue not overlapped — the choice for long-K GEMMs).
template <int kNP>
struct G2 {
  static constexpr int kABytes = 128 * kGmBK * 2;              // this CTA's 128 rows of A
  static constexpr int kBBytes = (kNP / 2) * kGmBK * 2;         // this CTA's kNP/2 columns of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = kNP == 256 ? 6 : 4;
  static constexpr int kAcc = kNP == 256 ? 2 : 1;               // TMEM accumulator buffers
  static constexpr size_t kSmem = size_t(kStages) * kStageBytes + 1024 + 256;
  // + the TMA-reduce epilogue's staging: one 32 × 32 fp32 box (4 KB) per epilogue warp,
  // 1024-B aligned after the barrier region
  static constexpr size_t kSmemRed = size_t(kStages) * kStageBytes + 1024 + 1024 + 8 * 4096;
};

// TMA-reduce epilogue (kOutAddF32, CTA pairs): this warp's 32 rows × nchunk·32 columns of the
// accumulator, 32 columns at a time: TMEM → registers → the warp's staging box (row = lane,
// 128-byte swizzle: 16-byte chunk j at j ^ (lane & 7)) → one elected lane adds the box into C at
// (row0, n0 + 32·c) with cp.reduce.async.bulk.tensor (rows / columns past C are dropped by the
// TMA unit). The box is rewritten only after the previous reduce has read it.
__device__ __forceinline__ void gemm_red_tile(const CUtensorMap* tmap_c, uint32_t base, int row0,
                                              int n0, int nchunk, uint32_t stage, int lane) {
#pragma unroll 1
  for (int c = 0; c < nchunk; ++c) {
    float x[32];
    __syncwarp();
    tmem_ld32(base + uint32_t(c * 32), x);
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t a = stage + uint32_t(lane) * 128u + (uint32_t(j ^ (lane & 7)) << 4);
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x[4 * j]),
                   "f"(x[4 * j + 1]), "f"(x[4 * j + 2]), "f"(x[4 * j + 3])
                   : "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile(
          "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];"
          ::"l"(reinterpret_cast<uint64_t>(tmap_c)), "r"(stage), "r"(n0 + c * 32), "r"(row0)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
}

template <bool kAMN, bool kBMN>
__host__ __device__ constexpr uint32_t gemm2_idesc() {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(kAMN) << 15) | (uint32_t(kBMN) << 16) |
         (uint32_t(kGmBN >> 3) << 17) | (uint32_t(256 >> 4) << 24);
}

constexpr int kTQ = 4;   // dynamic scheduler: work-item queue depth per CTA pair

// bounded wait with cluster-scope acquire: for the work-item queue, whose value the leader
// stores into this CTA's shared memory from the other SM before its remote arrive (rarely
// polled: the leader publishes items up to kTQ ahead)
__device__ __forceinline__ void gm_wait_acq_cluster(uint32_t bar, uint32_t parity) {
  uint64_t t0 = 0;
  for (uint32_t it = 0;; ++it) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    if (ok) return;
    if ((it & 255u) == 255u) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > 20000000000ull) __trap();     // 20 s
    }
  }
}

// bounded wait on a barrier of this CTA that the peer CTA also arrives on (TMA bytes, MMA
// commits, remote epilogue arrivals). The default (CTA-scope) acquire suffices: what the
// barrier guards is shared memory written through the async proxy and TMEM, ordered by
// complete_tx and the tcgen05 fences. A .acquire.cluster wait compiled to an L1 invalidation
// (CCTL.IVALL) per poll: 63 % of the forward GEMM's stall samples, 307 M executions per call.
__device__ __forceinline__ void gm_wait_cluster(uint32_t bar, uint32_t parity) {
  uint64_t t0 = 0;
  for (uint32_t it = 0;; ++it) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    if (ok) return;
    if ((it & 255u) == 255u) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > 20000000000ull) __trap();     // 20 s
    }
  }
}

// Multicast A: the same A K-slice (rows of one pair's M-tile) lands in the CTAs of `mask`
// (one CTA per pair); each destination pair's leader barrier collects the bytes (the barrier
// operand is the issuing pair leader's, peer bit 0 — the 2-SM multicast form).
__device__ __forceinline__ void tma_load_2d_pair_mc(uint32_t dst, const CUtensorMap* map, int c0,
                                                    int c1, uint32_t leader_bar, uint16_t mask,
                                                    uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster.L2::cache_hint [%0], [%1, {%4, %5}], [%2], %3, %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "h"(mask), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}
// tcgen05.commit of the pair's MMAs to the barrier at this offset in every CTA of `mask`
__device__ __forceinline__ void tc_commit_mask(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar), "h"(mask)
      : "memory");
}

// kPairs = CTA pairs per cluster: 1, or 2 — the two pairs compute the tiles (m, 2j) and
// (m, 2j + 1), share the A K-slices through TMA multicast (half the A traffic from L2, and the
// pairs move in lockstep: a stage is refilled only when both consumed it).
template <bool kAMN, bool kBMN, int kOut, int kNP, int kPairs>
__device__ __forceinline__ void gemm2_body(const CUtensorMap& tmap_a, const CUtensorMap& tmap_b,
                                           const CUtensorMap& tmap_c, const GemmParams& p0) {
  using C = G2<kNP>;
  constexpr int kG2Stages = C::kStages, kG2ABytes = C::kABytes, kG2BBytes = C::kBBytes;
  constexpr int kG2StageBytes = C::kStageBytes;
  const GemmParams p = gemm_effective(p0, 2 * kGmBM);
  if (p.mblk * p.nblk == 0 || p.kblk == 0) return;   // nothing to add (uniform in the grid)
  // super-tiles of kPairs N-blocks (pair `pair` takes N-block nbp·kPairs + pair)
  GemmParams ps = p;
  ps.nblk = (p.nblk + kPairs - 1) / kPairs;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kG2Stages * kG2ABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kG2Stages * kG2StageBytes);
  uint64_t* empty = full + kG2Stages;
  uint64_t* tfull = empty + kG2Stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* tq_full = tempty + 2;                   // dynamic scheduler: item queue slots
  uint64_t* tq_empty = tq_full + kTQ;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq_empty + kTQ);
  int* tq_ring = reinterpret_cast<int*>(tmem_slot + 1);

  const uint32_t crank = cluster_rank();
  const uint32_t rank = crank & 1u, pair = crank >> 1, leader = crank & ~1u;
  const uint16_t pair_mask = uint16_t(3u << (2 * pair));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cluster = blockIdx.x / (2 * kPairs), nclusters = gridDim.x / (2 * kPairs);
  const int tiles = ps.mblk * ps.nblk;
  const int ks_n = (kOut == kOutF32 && p.ksplit == 2) ? 2 : 1;
  const int items = tiles * ks_n;
  auto krange = [&](int t, int& kb0, int& kb1) {   // K-blocks of work item t
    const int ks = t / tiles;
    kb0 = ks_n == 1 ? 0 : (ks * p.kblk) / 2;
    kb1 = ks_n == 1 ? p.kblk : ((ks + 1) * p.kblk) / 2;
  };
  // dynamic scheduler: item k of this pair sits in queue slot k % kTQ of both CTAs; the
  // leader's producer writes it (−1 = no more work), every other role of the pair takes it and
  // releases the slot on the leader's tq_empty (1 + 1 + 2·8 arrivals: peer producer, MMA
  // issuer, the epilogue warps of both CTAs)
  const bool dyn = kPairs == 1 && p.tile_ctr != nullptr;
  const uint32_t peer = crank | 1u;
  auto tq_take = [&](int k) -> int {                // one thread
    const int s = k % kTQ;
    gm_wait_acq_cluster(smem_u32(&tq_full[s]), uint32_t(k / kTQ) & 1u);
    const int it = *reinterpret_cast<volatile int*>(&tq_ring[s]);
    if (rank == 0) mbar_arrive(&tq_empty[s]);
    else arrive_remote(mapa_rank(smem_u32(&tq_empty[s]), leader));
    return it;
  };
  auto tq_put = [&](int k, int it) {                // the leader's producer
    const int s = k % kTQ;
    gm_wait_cluster(smem_u32(&tq_empty[s]), (uint32_t(k / kTQ) & 1u) ^ 1u);
    tq_ring[s] = it;
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(mapa_rank(smem_u32(&tq_ring[s]), peer)),
                 "r"(it) : "memory");
    mbar_arrive(&tq_full[s]);
    arrive_remote(mapa_rank(smem_u32(&tq_full[s]), peer));
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kG2Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kPairs);                 // every pair's commit frees the stage
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * (kG2Threads - 64));   // every epilogue thread of both CTAs
    }
    for (int s = 0; s < kTQ; ++s) {
      mbar_init(&tq_full[s], 1);
      mbar_init(&tq_empty[s], 2 + 2 * ((kG2Threads - 64) / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pa = l2_policy(p.hint_a), pb = l2_policy(p.hint_b);
      const bool pace = p.sync != nullptr && rank == 0;
      uint32_t q = 0;
      int k_tq = 0, item_s = cluster;
      // a skipped tile (no row to compute) still reports every chunk, so its wave never waits
      auto skip_report = [&](int it) {
        int kb0s, kb1s;
        krange(it, kb0s, kb1s);
        if (pace && kb1s > kb0s)
          atomicAdd(p.sync + it / nclusters, unsigned((kb1s - kb0s - 1) / p.sync_chunk));
      };
      auto dead = [&](int it) {
        if (!p.lm.mlive) return false;
        int mbd, nbd;
        gemm_tile_coords(ps, it % tiles, mbd, nbd);
        return !p.lm.mlive[mbd];
      };
      for (;;) {
        int item;
        if (dyn) {
          if (rank == 0) {
            item = atomicAdd(p.tile_ctr, 1);
            while (item < items && dead(item)) {
              skip_report(item);
              item = atomicAdd(p.tile_ctr, 1);
            }
            if (item >= items) item = -1;
            tq_put(k_tq, item);
          } else {
            item = tq_take(k_tq);
          }
          ++k_tq;
          if (item < 0) break;
        } else {
          item = item_s;
          if (item >= items) break;
          item_s += nclusters;
        }
        const int wave = item / nclusters;
        int mb, nb, kb0, kb1;
        gemm_tile_coords(ps, item % tiles, mb, nb);
        nb = nb * kPairs + int(pair);
        krange(item, kb0, kb1);
        if (dead(item)) {                                 // static schedule: skipped tile
          skip_report(item);
          continue;
        }
        const int m0 = mb * 2 * kGmBM + int(rank) * kGmBM;
        const int n0 = nb * kNP + int(rank) * 128;
        const unsigned members = unsigned(min(nclusters, items - wave * nclusters));
        for (int kb = kb0; kb < kb1; ++kb, ++q) {
          const int s = q % kG2Stages;
          const int k0 = kb * kGmBK;
          // chunks count from the item's first K-step (a split-K half starts mid-K)
          if (pace && (kb - kb0) % p.sync_chunk == 0) {
            const int c = (kb - kb0) / p.sync_chunk;   // entering chunk c: chunk c − 1 is issued
            if (c > 0) atomicAdd(p.sync + wave, 1u);
            if (c > p.sync_slack)
              soft_wait(p.sync + wave, unsigned(c - p.sync_slack) * members, p.sync_timeout_ns);
          }
          gm_wait_cluster(smem_u32(&empty[s]), ((q / kG2Stages) & 1u) ^ 1u);
          const uint32_t leader_full = mapa_rank(smem_u32(&full[s]), leader);
          if (rank == 0) arrive_expect_tx_u32(smem_u32(&full[s]), 2 * kG2StageBytes);
          const uint32_t a = smem_u32(sA + s * kG2ABytes), b = smem_u32(sB + s * kG2BBytes);
          if constexpr (kPairs == 2) {
            // pair 0's CTAs load the A K-slice of their 128 rows for both pairs
            if (pair == 0) {
              const uint16_t mc = uint16_t((1u << rank) | (1u << (rank + 2)));
              if constexpr (kAMN) {
                tma_load_2d_pair_mc(a, &tmap_a, m0, k0, leader_full, mc, pa);
                tma_load_2d_pair_mc(a + kGmMNBox, &tmap_a, m0 + 64, k0, leader_full, mc, pa);
              } else {
                tma_load_2d_pair_mc(a, &tmap_a, k0, m0, leader_full, mc, pa);
              }
            }
          } else if constexpr (kAMN) {
            tma_load_2d_pair_hint(a, &tmap_a, m0, k0, leader_full, pa);
            tma_load_2d_pair_hint(a + kGmMNBox, &tmap_a, m0 + 64, k0, leader_full, pa);
          } else {
            tma_load_2d_pair_hint(a, &tmap_a, k0, m0, leader_full, pa);
          }
#pragma unroll
          for (int hh = 0; hh < kNP / 256; ++hh) {   // MMA half hh: this CTA's 128 columns
            const uint32_t bh = b + hh * (128 * kGmBK * 2);
            const int nh = n0 + hh * 256;
            if constexpr (kBMN) {
              tma_load_2d_pair_hint(bh, &tmap_b, nh, k0, leader_full, pb);
              tma_load_2d_pair_hint(bh + kGmMNBox, &tmap_b, nh + 64, k0, leader_full, pb);
            } else {
              tma_load_2d_pair_hint(bh, &tmap_b, k0, nh, leader_full, pb);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (leader)
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = gemm2_idesc<kAMN, kBMN>();
      uint32_t q = 0;
      int i = 0;
      int k_tq = 0, item_s = cluster;
      for (;;) {
        int item;
        if (dyn) {
          item = tq_take(k_tq++);
          if (item < 0) break;
        } else {
          item = item_s;
          if (item >= items) break;
          item_s += nclusters;
        }
        if (p.lm.mlive) {
          int mb, nb;
          gemm_tile_coords(ps, item % tiles, mb, nb);
          if (!p.lm.mlive[mb]) continue;
        }
        int kb0, kb1;
        krange(item, kb0, kb1);
        const int acc = C::kAcc == 2 ? (i & 1) : 0;
        const int use = C::kAcc == 2 ? (i >> 1) : i;     // earlier uses of this buffer
        ++i;
        gm_wait_cluster(smem_u32(&tempty[acc]), (use & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t dt = tmem + uint32_t(acc * kGmBN);
        int kbs = kb0;
        if constexpr (kNP == 512) {
          // One 512-column accumulator, released in halves (tempty[0] = columns 0-255 read,
          // tempty[1] = 256-511): the first P K-steps go to half 0 only, while the epilogue
          // still reads the previous tile's half 1; their half-1 MMAs follow from the same
          // (still held) stages once half 1 is free. Hides half of the epilogue.
          const int P = p.half_release ? min(kG2Stages, kb1 - kb0) : 0;
          for (int j = 0; j < P; ++j) {
            const uint32_t qj = q + uint32_t(j);
            const int s = qj % kG2Stages;
            gm_wait_cluster(smem_u32(&full[s]), (qj / kG2Stages) & 1u);
            tc_fence_after();
            const uint32_t a0 = smem_u32(sA + s * kG2ABytes), b0 = smem_u32(sB + s * kG2BBytes);
#pragma unroll
            for (int k = 0; k < kGmBK / 16; ++k) {
              const uint64_t ad = kAMN ? umma_desc_sw128_mn(a0 + k * 2048) : umma_desc_sw128(a0 + k * 32);
              const uint64_t bd = kBMN ? umma_desc_sw128_mn(b0 + k * 2048) : umma_desc_sw128(b0 + k * 32);
              tc_mma_pair(dt, ad, bd, idesc, (j != 0) || (k != 0));
            }
          }
          gm_wait_cluster(smem_u32(&tempty[1]), (use & 1u) ^ 1u);
          tc_fence_after();
          for (int j = 0; j < P; ++j, ++q) {
            const int s = q % kG2Stages;
            const uint32_t a0 = smem_u32(sA + s * kG2ABytes);
            const uint32_t bh = smem_u32(sB + s * kG2BBytes) + 128 * kGmBK * 2;
#pragma unroll
            for (int k = 0; k < kGmBK / 16; ++k) {
              const uint64_t ad = kAMN ? umma_desc_sw128_mn(a0 + k * 2048) : umma_desc_sw128(a0 + k * 32);
              const uint64_t bd = kBMN ? umma_desc_sw128_mn(bh + k * 2048) : umma_desc_sw128(bh + k * 32);
              tc_mma_pair(dt + 256u, ad, bd, idesc, (j != 0) || (k != 0));
            }
            tc_commit_mask(smem_u32(&empty[s]), kPairs == 2 ? uint16_t(0xF) : pair_mask);
          }
          kbs = kb0 + P;
        }
        for (int kb = kbs; kb < kb1; ++kb, ++q) {
          const int s = q % kG2Stages;
          gm_wait_cluster(smem_u32(&full[s]), (q / kG2Stages) & 1u);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * kG2ABytes), b0 = smem_u32(sB + s * kG2BBytes);
#pragma unroll
          for (int k = 0; k < kGmBK / 16; ++k) {
            const uint64_t ad = kAMN ? umma_desc_sw128_mn(a0 + k * 2048) : umma_desc_sw128(a0 + k * 32);
#pragma unroll
            for (int hh = 0; hh < kNP / 256; ++hh) {
              const uint32_t bh = b0 + hh * (128 * kGmBK * 2);
              const uint64_t bd = kBMN ? umma_desc_sw128_mn(bh + k * 2048) : umma_desc_sw128(bh + k * 32);
              tc_mma_pair(dt + uint32_t(hh * 256), ad, bd, idesc, (kb != kb0) || (k != 0));
            }
          }
          // slot s consumed by this pair: arrive on the empty barrier of every CTA of the
          // cluster (with shared A, a stage is free only once both pairs consumed it)
          tc_commit_mask(smem_u32(&empty[s]), kPairs == 2 ? uint16_t(0xF) : pair_mask);
        }
        tc_commit_mask(smem_u32(&tfull[acc]), pair_mask);   // accumulator ready in the pair
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int chalf = (warp - 2) >> 2;                 // which half of the tile's columns
    constexpr int kCols = kNP / 2, kChunks = kCols / 32;
    const uint64_t pol_c = l2_policy(p.hint_c);
    const uint32_t leader_tempty0 = mapa_rank(smem_u32(&tempty[0]), leader);
    const uint32_t leader_tempty1 = mapa_rank(smem_u32(&tempty[1]), leader);
    const uint32_t stage_w = smem_u32(smem + kG2Stages * kG2StageBytes + 1024) +
                             uint32_t(warp - 2) * 4096u;   // TMA-reduce staging box of this warp
    int i = 0;
    GemmParams p1 = p;                                  // K-half 1 of a split: the scratch
    p1.C = p.split_out;
    p1.ldc = p.split_ld;
    p1.row_map = nullptr;
    int k_tq = 0, item_s = cluster;
    for (;;) {
      int item;
      if (dyn) {
        int it = 0;
        if (lane == 0) it = tq_take(k_tq);
        item = __shfl_sync(0xffffffffu, it, 0);
        ++k_tq;
        if (item < 0) break;
      } else {
        item = item_s;
        if (item >= items) break;
        item_s += nclusters;
      }
      int mb, nb;
      gemm_tile_coords(ps, item % tiles, mb, nb);
      nb = nb * kPairs + int(pair);
      if (p.lm.mlive && !p.lm.mlive[mb]) continue;
      const bool second = item >= tiles;
      const int acc = C::kAcc == 2 ? (i & 1) : 0;
      const int use = C::kAcc == 2 ? (i >> 1) : i;
      ++i;
      gm_wait_cluster(smem_u32(&tfull[acc]), use & 1u);
      tc_fence_after();
      const int r = mb * 2 * kGmBM + int(rank) * kGmBM + row;
      if constexpr (kNP == 512) {
        // both warp groups drain accumulator half 0 (128 columns each), release it, then half 1
        const uint32_t lb = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(chalf * 128);
        const int cb = nb * kNP + chalf * 128;
        if constexpr (kOut == kOutLmFwd) {
          const bool valid = r < p.M && p.lm.flag[r];
          const int y = valid ? p.lm.tokens[r] : -1;
          float R = -INFINITY, S = 0.f, W = 0.f, cS = 0.f, cW = 0.f, uy = __int_as_float(0x7fc00000);
#pragma unroll 1
          for (int hh = 0; hh < 2; ++hh) {
            lm_fwd_cols(p, lb + uint32_t(hh * 256), r, cb + hh * 256, R, S, W, cS, cW, uy, valid, y, 4);
            __syncwarp();
            tc_fence_before();
            arrive_remote(hh ? leader_tempty1 : leader_tempty0);
          }
          if (valid && nb < p.nblk)   // one partial per (tile, column group): partial[2·nb + chalf][row]
            p.lm.partial[int64_t(2 * nb + chalf) * p.lm.n_rows + r] = make_float4(R, S - cS, W - cW, uy);
        } else if constexpr (kOut == kOutLmDz) {
          BwdRec rc;
          rc.ng = 0.f;
          rc.y = -1;
          if (r < p.M) rc = p.lm.rec[r];
#pragma unroll 1
          for (int hh = 0; hh < 2; ++hh) {
            lm_dz_cols(p, lb + uint32_t(hh * 256), r, cb + hh * 256, rc, 4);
            __syncwarp();
            tc_fence_before();
            arrive_remote(hh ? leader_tempty1 : leader_tempty0);
          }
        } else {
#pragma unroll 1
          for (int hh = 0; hh < 2; ++hh) {
            if (kOut == kOutAddF32 && p.tma_red)
              gemm_red_tile(&tmap_c, lb + uint32_t(hh * 256), r - lane, cb + hh * 256, 4, stage_w, lane);
            else
              gemm_store_tile<kOut>(second ? p1 : p, lb + uint32_t(hh * 256), r, cb + hh * 256, pol_c, 4);
            __syncwarp();
            tc_fence_before();
            arrive_remote(hh ? leader_tempty1 : leader_tempty0);
          }
        }
        continue;
      }
      const uint32_t base = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(acc * kGmBN) +
                            uint32_t(chalf * kCols);
      const int c0 = nb * kNP + chalf * kCols;         // first tile column this thread drains
      if constexpr (kOut == kOutLmFwd) {
        const bool valid = r < p.M && p.lm.flag[r];
        const int y = valid ? p.lm.tokens[r] : -1;
        float R = -INFINITY, S = 0.f, W = 0.f, cS = 0.f, cW = 0.f, uy = __int_as_float(0x7fc00000);
        lm_fwd_cols(p, base, r, c0, R, S, W, cS, cW, uy, valid, y, kChunks);
        if (valid && nb < p.nblk)   // one partial per (tile, column half): partial[2·nb + half][row]
          p.lm.partial[int64_t(2 * nb + chalf) * p.lm.n_rows + r] = make_float4(R, S - cS, W - cW, uy);
      } else if constexpr (kOut == kOutLmDz) {
        BwdRec rc;
        rc.ng = 0.f;
        rc.y = -1;
        if (r < p.M) rc = p.lm.rec[r];
        lm_dz_cols(p, base, r, c0, rc, kChunks);
      } else if (kOut == kOutAddF32 && p.tma_red) {
        gemm_red_tile(&tmap_c, base, r - lane, c0, kChunks, stage_w, lane);
      } else {
        gemm_store_tile<kOut>(second ? p1 : p, base, r, c0, pol_c, kChunks);
      }
      __syncwarp();
      tc_fence_before();
      arrive_remote(acc ? leader_tempty1 : leader_tempty0);
    }
  }
  if (kOut == kOutAddF32 && p.tma_red && warp >= 2 && lane == 0)
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // every reduce performed
  tc_fence_before();
  cluster_sync_all();     // all CTAs done with TMEM and with remote barriers
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512)
                 : "memory");
  }
}

template <bool kAMN, bool kBMN, int kOut, int kNP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kG2Threads, 1)
    k_umma_gemm2(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                 const __grid_constant__ CUtensorMap tmap_c, const GemmParams p0) {
  gemm2_body<kAMN, kBMN, kOut, kNP, 1>(tmap_a, tmap_b, tmap_c, p0);
}

template <bool kAMN, bool kBMN, int kOut, int kNP>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(kG2Threads, 1)
    k_umma_gemm4(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                 const __grid_constant__ CUtensorMap tmap_c, const GemmParams p0) {
  gemm2_body<kAMN, kBMN, kOut, kNP, 2>(tmap_a, tmap_b, tmap_c, p0);
}

// C[row_map ? row_map[r] : r][0, N) += split[r][0, N) for r < the (device) row count.
__global__ void __launch_bounds__(256) k_split_fixup(float* C, int64_t ldc, const float* split,
                                                     int64_t lds, int M, int N, const int* dyn_count,
                                                     int dyn_base, const int* row_map) {
  int m = M;
  if (dyn_count) m = min(M, max(0, *dyn_count - dyn_base));
  const int nv = N / 4;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < int64_t(m) * nv;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(i / nv), v = int(i % nv);
    const int orow = row_map ? row_map[r] : r;
    float4* o = reinterpret_cast<float4*>(C + int64_t(orow) * ldc) + v;
    const float4 a = reinterpret_cast<const float4*>(split + int64_t(r) * lds)[v];
    float4 b = *o;
    b.x += a.x;
    b.y += a.y;
    b.z += a.z;
    b.w += a.w;
    *o = b;
  }
}

}  // namespace espo
