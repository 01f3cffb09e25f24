// k_lmhead2.cuh — the fused LM head on CTA PAIRS (tcgen05.mma.cta_group::2): the same
// computation as k_lmhead.cuh (forward statistics, or the backward's bf16 dz tile) with an
// M = 256 × N = 256 MMA shared by the two SMs of a cluster.
//
// Why: with one CTA per 128×256 tile every K-step moves 16 KB of A and 32 KB of B from L2 for
// 4.2 MFLOP (1/87 B/FLOP) — at ~1.4 PFLOP/s that is ~16 TB/s of L2→SM traffic, above what the
// L2 slices deliver, so large d ran L2/DRAM-bound (ncu at d = 8192: 43 % L2 hit, 531 GB of
// DRAM reads per launch). A CTA pair computes a 256×256 tile per K-step from 32 KB per CTA
// (its 128 rows of A and half of the 256 B rows): 1/128 B/FLOP, 1.5× less L2 traffic.
//
// Pair layout: cluster (2, 1, 1); blockIdx.x = 2·part + rank, blockIdx.y = row-block pair.
// CTA `rank` owns rows m0 = (2·blockIdx.y + rank)·128 (its TMEM lanes hold them) and loads
// W rows [tile·256 + rank·128, +128) of every vocabulary tile. The leader (rank 0):
//   - its full[s] barriers collect the TMA bytes of BOTH CTAs (the peer's loads signal the
//     leader's barrier: cp.async.bulk.tensor .cta_group::2);
//   - its MMA thread issues tcgen05.mma.cta_group::2 (A rows split by CTA, B columns split
//     by CTA, same smem offsets in both) and commits with .multicast::cluster to both CTAs'
//     empty[s] (smem slot free) and tfull[acc] (accumulator ready) barriers;
//   - its tempty[acc] barriers count the 256 epilogue threads of both CTAs (the peer's arrive
//     remotely through mapa / shared::cluster).
// Each CTA's epilogue (warps 2–5) reads its own TMEM exactly as in k_lmhead.cuh.
// All barrier waits are bounded: a protocol error traps (a CUDA error) instead of hanging.
#pragma once
#include <cuda.h>

#include "k_lmhead.cuh"

namespace espo {

constexpr int kL2Stages = 6;
constexpr int kL2ABytes = kLmBM * kLmBK * 2;          // 16 KB: this CTA's 128 rows of A
constexpr int kL2BBytes = (kLmBN / 2) * kLmBK * 2;    // 16 KB: this CTA's half of B
constexpr int kL2StageBytes = kL2ABytes + kL2BBytes;
constexpr size_t kL2Smem = size_t(kL2Stages) * kL2StageBytes + 1024 + 256;
// instruction descriptor: bf16 × bf16 → f32, K-major A and B, M = 256 (pair), N = 256
constexpr uint32_t kL2Idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(kLmBN >> 3) << 17) |
                              (uint32_t(256 >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `local` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void bounded_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  for (uint32_t it = 0; it < (1u << 22); ++it) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    if (ok) return;
  }
  __trap();   // a barrier that never completes is a protocol bug: fail, do not hang
}
__device__ __forceinline__ void arrive_expect_tx_u32(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
// TMA 2D load into this CTA's smem, completing bytes on a barrier of either pair CTA
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                                 uint32_t cluster_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(cluster_bar)
      : "memory");
}
__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar), "h"(static_cast<uint16_t>(3))
      : "memory");
}

template <bool kDz>
__device__ __forceinline__ void lmhead2_body(const CUtensorMap& tmap_h, const CUtensorMap& tmap_w,
                                             const LmParams& p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sA = smem;                                  // [stages][16 KB]
  uint8_t* sB = smem + kL2Stages * kL2ABytes;          // [stages][16 KB]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kL2Stages * kL2StageBytes);
  uint64_t* empty = full + kL2Stages;
  uint64_t* tfull = empty + kL2Stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_any = reinterpret_cast<int*>(tmem_slot + 1);

  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int part = blockIdx.x >> 1;
  const int m0 = (blockIdx.y * 2 + int(rank)) * kLmBM;
  const int t_begin = int((int64_t(p.ntiles) * part) / p.parts);
  const int t_end = int((int64_t(p.ntiles) * (part + 1)) / p.parts);
  const int nk = (p.d + kLmBK - 1) / kLmBK;

  // rows beyond the compacted count (lm_rows) count as absent; a pair whose rows are all
  // absent still runs the barrier handshake below and leaves together
  const int n_rows = lm_rows(p);
  // does this CTA have a row to work on? the pair proceeds unless both are empty
  if (threadIdx.x == 0) *s_any = 0;
  __syncthreads();
  if (threadIdx.x < kLmBM) {
    const int r = m0 + threadIdx.x;
    if (r < n_rows) {
      if constexpr (kDz) {
        if (p.rec[r].ng != 0.f) *s_any = 1;
      } else {
        if (p.ws.flag[p.row_begin + r]) *s_any = 1;
      }
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kL2Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kLmBM);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync_all();
  int peer_any = 0;
  {
    const uint32_t ra = mapa_rank(smem_u32(s_any), rank ^ 1u);
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(peer_any) : "r"(ra) : "memory");
  }
  const bool run = (*s_any != 0 || peer_any != 0) && t_begin < t_end;
  if (!run) {
    if constexpr (kDz) {   // no gradient in this pair: zero this CTA's rows of the part
      if (t_begin < t_end) {
        const int c0 = t_begin * kLmBN / 8, c1 = t_end * kLmBN / 8;
        const int nr = max(0, min(kLmBM, n_rows - m0));
        for (int rr = 0; rr < nr; ++rr) {
          uint4* o = reinterpret_cast<uint4*>(p.dz + int64_t(m0 + rr) * p.ldz);
          for (int c = c0 + int(threadIdx.x); c < c1; c += kLmThreads) o[c] = make_uint4(0, 0, 0, 0);
        }
      }
    }
    cluster_sync_all();    // the peer's ld of s_any completed before this CTA exits
    return;
  }

  if (warp == 1) {   // TMEM: two 256-column fp32 accumulators in each CTA of the pair
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
      uint32_t q = 0;
      for (int tile = t_begin; tile < t_end; ++tile) {
        for (int kb = 0; kb < nk; ++kb, ++q) {
          const int s = q % kL2Stages;
          bounded_wait(smem_u32(&empty[s]), ((q / kL2Stages) & 1u) ^ 1u);
          const uint32_t leader_full = mapa_rank(smem_u32(&full[s]), 0);
          if (rank == 0) arrive_expect_tx_u32(smem_u32(&full[s]), 2 * kL2StageBytes);
          tma_load_2d_pair(smem_u32(sA + s * kL2ABytes), &tmap_h, kb * kLmBK, m0, leader_full);
          tma_load_2d_pair(smem_u32(sB + s * kL2BBytes), &tmap_w, kb * kLmBK,
                           tile * kLmBN + int(rank) * (kLmBN / 2), leader_full);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (leader)
    if (rank == 0 && lane == 0) {
      uint32_t q = 0;
      int i = 0;
      for (int tile = t_begin; tile < t_end; ++tile, ++i) {
        const int acc = i & 1;
        bounded_wait(smem_u32(&tempty[acc]), ((i >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t dt = tmem + uint32_t(acc * kLmBN);
        for (int kb = 0; kb < nk; ++kb, ++q) {
          const int s = q % kL2Stages;
          bounded_wait(smem_u32(&full[s]), (q / kL2Stages) & 1u);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * kL2ABytes), b0 = smem_u32(sB + s * kL2BBytes);
#pragma unroll
          for (int k = 0; k < kLmBK / 16; ++k)
            tc_mma_pair(dt, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), kL2Idesc,
                        (kb | k) != 0);
          tc_commit_pair(smem_u32(&empty[s]));     // slot s free in both CTAs
        }
        tc_commit_pair(smem_u32(&tfull[acc]));     // accumulator ready in both CTAs
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int r = m0 + row;
    const uint32_t leader_tempty0 = mapa_rank(smem_u32(&tempty[0]), 0);
    const uint32_t leader_tempty1 = mapa_rank(smem_u32(&tempty[1]), 0);
    if constexpr (kDz) {
      BwdRec rc;
      rc.ng = 0.f;
      rc.y = -1;
      if (r < n_rows) rc = p.rec[r];
      int i = 0;
      for (int tile = t_begin; tile < t_end; ++tile, ++i) {
        const int acc = i & 1;
        bounded_wait(smem_u32(&tfull[acc]), (i >> 1) & 1u);
        tc_fence_after();
        const uint32_t base = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(acc * kLmBN);
#pragma unroll 1
        for (int c = 0; c < kLmBN / 32; ++c) {
          float x[32];
          __syncwarp();
          tmem_ld32(base + uint32_t(c * 32), x);
          const int col0 = tile * kLmBN + c * 32;
          if (r < n_rows) lm_store_dz(x, rc, col0, p.V, p.lam_log2e, p.dz + int64_t(r) * p.ldz + col0);
        }
        __syncwarp();
        tc_fence_before();
        arrive_remote(acc ? leader_tempty1 : leader_tempty0);
      }
    } else {
      const bool valid = r < n_rows && p.ws.flag[p.row_begin + r];
      const int y = valid ? p.tokens[r] : -1;
      const float lamL = p.lam_log2e;
      float R = -INFINITY, S = 0.f, W = 0.f, cS = 0.f, cW = 0.f, uy = __int_as_float(0x7fc00000);
      int i = 0;
      for (int tile = t_begin; tile < t_end; ++tile, ++i) {
        const int acc = i & 1;
        bounded_wait(smem_u32(&tfull[acc]), (i >> 1) & 1u);
        tc_fence_after();
        const uint32_t base = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(acc * kLmBN);
#pragma unroll 1
        for (int c = 0; c < kLmBN / 32; ++c) {
          float x[32];
          __syncwarp();
          tmem_ld32(base + uint32_t(c * 32), x);
          const int col0 = tile * kLmBN + c * 32;
          if (!valid) continue;
          lm_row_chunk(x, col0, y, p.V, lamL, R, S, W, cS, cW, uy, p.ws.err);
        }
        __syncwarp();
        tc_fence_before();
        arrive_remote(acc ? leader_tempty1 : leader_tempty0);
      }
      if (valid)
        reinterpret_cast<float4*>(p.partial)[int64_t(part) * p.n_rows + r] =
            make_float4(R, S - cS, W - cW, uy);
    }
  }
  tc_fence_before();
  cluster_sync_all();     // both CTAs done with TMEM and with remote barriers
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512)
                 : "memory");
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kLmThreads, 1)
    k_lmhead2_fwd(const __grid_constant__ CUtensorMap tmap_h, const __grid_constant__ CUtensorMap tmap_w,
                  const LmParams p) {
  lmhead2_body<false>(tmap_h, tmap_w, p);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kLmThreads, 1)
    k_lmhead2_dz(const __grid_constant__ CUtensorMap tmap_h, const __grid_constant__ CUtensorMap tmap_w,
                 const LmParams p) {
  lmhead2_body<true>(tmap_h, tmap_w, p);
}

}  // namespace espo
