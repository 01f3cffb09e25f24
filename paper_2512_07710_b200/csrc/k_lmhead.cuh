// k_lmhead.cuh — fused LM head + ESPO forward statistics on the 5th-gen tensor cores
// (SURVEY §8(f) row 1): logits z = h·Wᵀ are produced tile by tile in TMEM by tcgen05.mma and
// reduced on the fly into the row statistics (lse, lp, H, q) — the [T, V] logits never exist
// in HBM.
//
// CTA = one 128-row block of hidden states × one contiguous part of the vocabulary (P parts;
// grid = (P, row blocks), P chosen so the A tiles of the resident CTAs fit in L2).
// Warp roles (192 threads): warp 0 — TMA producer (cp.async.bulk.tensor 2D, 128-byte swizzle,
// 4-stage smem ring of {A: 128×64 bf16, B: 256×64 bf16}); warp 1 — TMEM allocator and MMA
// issuer (one thread, tcgen05.mma.cta_group::1.kind::f16, M=128, N=256, K=16, fp32
// accumulators in two 256-column TMEM buffers); warps 2–5 — epilogue: thread i owns row i
// (TMEM lane i), reads its 256 logits per tile with tcgen05.ld.32x32b.x32 and runs the same
// base-2 online (max, S, W) reduction as K2. Each CTA writes a 16-byte partial
// {R, S, W, u_y} per row; k_fwd_combine merges the P parts (the vocabulary-parallel merge).
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "k_rowlist.cuh"
#include "k_rowstats.cuh"
#include "workspace.cuh"

namespace espo {

constexpr int kLmBM = 128;          // rows per CTA (UMMA M)
constexpr int kLmBN = 256;          // vocabulary columns per tile (UMMA N)
constexpr int kLmBK = 64;           // K per stage (128 bytes of bf16: one swizzle atom)
constexpr int kLmStages = 4;
constexpr int kLmABytes = kLmBM * kLmBK * 2;   // 16 KB
constexpr int kLmBBytes = kLmBN * kLmBK * 2;   // 32 KB
constexpr int kLmStageBytes = kLmABytes + kLmBBytes;
constexpr int kLmThreads = 192;
constexpr size_t kLmSmem = size_t(kLmStages) * kLmStageBytes + 1024 /*align*/ + 256 /*barriers*/;

struct LmParams {
  int n_rows;            // rows of this chunk
  int64_t row_begin;
  int d;                 // hidden size (K)
  int V;                 // vocabulary rows of W
  int ntiles;            // ceil(V / 256)
  int parts;             // vocabulary parts (gridDim.y)
  float lam_log2e;
  const int32_t* tokens; // chunk-relative
  float* partial;        // [parts][n_rows] float4 (forward)
  const BwdRec* rec;     // per-row backward records, chunk-relative (k_lmhead_dz)
  __nv_bfloat16* dz;     // [n_rows][ldz] bf16 gradient tile output (k_lmhead_dz)
  int64_t ldz;           // ≥ ntiles·256 elements
  Workspace ws;
  // k_lmhead_dz on compacted rows: rows ≥ round_up(clamp(*dyn_count − dyn_base, 0, n_rows),
  // 256) are skipped (neither computed nor written)
  const int* dyn_count;
  int dyn_base;
};

__device__ __forceinline__ int lm_rows(const LmParams& p) {
  if (!p.dyn_count) return p.n_rows;
  const int n = max(0, *p.dyn_count - p.dyn_base);
  return min(p.n_rows, (n + 255) / 256 * 256);
}

// --------------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle (rows of 128 B, 8-row groups
// 1024 B apart), sm100 version field = 1.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr & 0x3FFFF) >> 4);        // start address
  d |= uint64_t(1) << 16;                       // LBO (unused for swizzled K-major) = 1
  d |= uint64_t(1024 >> 4) << 32;               // SBO = 1024 B
  d |= uint64_t(1) << 46;                       // version (Blackwell)
  d |= uint64_t(2) << 61;                       // SWIZZLE_128B
  return d;
}
// instruction descriptor: bf16 × bf16 → f32, K-major A and B, M = 128, N = 256
constexpr uint32_t kLmIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(kLmBN >> 3) << 17) |
                              (uint32_t(kLmBM >> 4) << 24);

// Epilogue of the backward recompute (kDz): the gradient of the 32 logits x[] of row `rc`
// starting at column col0, rounded to bf16 and stored (64 contiguous bytes of the row):
// dz_v = λ·g·(1[v = y] − p_v) — the same per-element formula as K5 (k_dlogits.cuh dz_vec).
__device__ __forceinline__ void lm_store_dz(const float* x, const BwdRec& rc, int col0, int V,
                                            float lamL, __nv_bfloat16* out) {
  uint32_t w[16];
  if (rc.ng != 0.f) {
    const bool special = (rc.y >= col0 && rc.y < col0 + 32) || (col0 + 32 > V);
    const float2 L2 = make_float2(lamL, lamL), N2 = make_float2(rc.nlseL, rc.nlseL),
                 G2 = make_float2(rc.ng, rc.ng);
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      const float2 t = __ffma2_rn(make_float2(x[e], x[e + 1]), L2, N2);
      const float2 o = __fmul2_rn(G2, make_float2(ex2(t.x), ex2(t.y)));
      float a = o.x, b = o.y;
      if (special) {
        if (col0 + e == rc.y) a = rc.gq;
        if (col0 + e + 1 == rc.y) b = rc.gq;
        if (col0 + e >= V) a = 0.f;
        if (col0 + e + 1 >= V) b = 0.f;
      }
      const __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
      w[e >> 1] = *reinterpret_cast<const uint32_t*>(&h2);
    }
  } else {
#pragma unroll
    for (int e = 0; e < 16; ++e) w[e] = 0u;
  }
  uint4* o = reinterpret_cast<uint4*>(out);
#pragma unroll
  for (int e = 0; e < 4; ++e) o[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
}

// One 32-column chunk of a row's logits x (fp32, from TMEM) into the row's base-2 online
// reduction (R, S, W) with Kahan compensation (cS, cW); captures u_y from the target's chunk.
__device__ __forceinline__ void lm_row_chunk(float* x, int col0, int y, int V, float lamL,
                                             float& R, float& S, float& W, float& cS, float& cW,
                                             float& uy, int* err) {
  const bool special = (y >= col0 && y < col0 + 32) || (col0 + 32 > V);
  if (special) {
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const int col = col0 + e;
      if (col == y) uy = x[e] * lamL;
      if (col == y || col >= V) x[e] = -INFINITY;
    }
  }
  if (R == -INFINITY) {                      // first chunk: reference = its max
    float m = x[0];
#pragma unroll
    for (int e = 1; e < 32; ++e) m = fmaxf(m, x[e]);
    R = m * lamL;
    if (R == -INFINITY) return;
  }
  // fast chunk: no clamp, no max (logits are finite; masked columns are −inf and go
  // through the checked path below via NaN = 0·(−inf))
  float bS, bW;
  {
    // two even/odd chains as packed FFMA2/FADD2 (bitwise the scalar arithmetic, as in K2)
    const float2 L2 = make_float2(lamL, lamL), N2 = make_float2(-R, -R);
    float2 s = make_float2(0.f, 0.f), w = make_float2(0.f, 0.f);
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      const float2 t = __ffma2_rn(make_float2(x[e], x[e + 1]), L2, N2);
      const float2 ex = make_float2(ex2(t.x), ex2(t.y));
      s = __fadd2_rn(s, ex);
      w = __ffma2_rn(ex, t, w);
    }
    bS = s.x + s.y;
    bW = w.x + w.y;
  }
  if (!(bS < 0x1p100f) || !(fabsf(bW) < 0x1p110f)) {  // overflow / −inf / NaN: checked
    S -= cS;
    W -= cW;
    cS = cW = 0.f;
    float m = -INFINITY;
    bool bad = false;
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      bad |= isnan(x[e]) || x[e] == INFINITY;
      m = fmaxf(m, x[e] * lamL);
    }
    if (bad) set_error(err, ESPO_ERR_NONFINITE_INPUT);
    if (m > R + 60.f) {
      rebase(R, m, S, W);
      R = m;
    }
    bS = 0.f;
    bW = 0.f;
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const float t = max_nan(fmaf(x[e], lamL, -R), -127.f);
      const float ex = ex2(t);
      bS += ex;
      bW = fmaf(ex, t, bW);
    }
  }
  kahan_add(S, cS, bS);
  kahan_add(W, cW, bW);
}

// kDz = false: forward statistics (k_lmhead_fwd); kDz = true: backward recompute writing the
// bf16 gradient tile dz = ∂(grad·loss)/∂z (k_lmhead_dz). Same TMA/MMA pipeline, same tile
// order and K order, so the recomputed logits are bitwise the forward's.
template <bool kDz>
__device__ __forceinline__ void lmhead_body(const CUtensorMap& tmap_h, const CUtensorMap& tmap_w,
                                            const LmParams& p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);   // 1024-B aligned (SW128)
  uint8_t* sA = smem;                                             // [stages][16 KB]
  uint8_t* sB = smem + kLmStages * kLmABytes;                     // [stages][32 KB]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kLmStages * kLmStageBytes);
  uint64_t* empty = full + kLmStages;
  uint64_t* tfull = empty + kLmStages;   // [2] accumulator ready
  uint64_t* tempty = tfull + 2;          // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_any = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // vocabulary part fastest-varying: the CTAs resident together share a few row blocks (their
  // A tiles stay in L2) and read the same W tiles in step
  const int m0 = blockIdx.y * kLmBM;
  const int part = blockIdx.x;
  const int t_begin = int((int64_t(p.ntiles) * part) / p.parts);
  const int t_end = int((int64_t(p.ntiles) * (part + 1)) / p.parts);
  const int nk = (p.d + kLmBK - 1) / kLmBK;

  const int n_rows = lm_rows(p);
  if (m0 >= n_rows) return;                   // beyond the compacted rows: nothing to do
  // skip blocks without a valid row (eliminated groups, masked tails)
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
  __syncthreads();
  if (t_begin >= t_end) return;
  if (*s_any == 0) {
    if constexpr (kDz) {   // no gradient in this block: zero its rows of this part's columns
      const int c0 = t_begin * kLmBN / 8, c1 = t_end * kLmBN / 8;   // uint4 columns
      const int nr = min(kLmBM, n_rows - m0);
      for (int rr = 0; rr < nr; ++rr) {
        uint4* o = reinterpret_cast<uint4*>(p.dz + int64_t(m0 + rr) * p.ldz);
        for (int c = c0 + int(threadIdx.x); c < c1; c += kLmThreads) o[c] = make_uint4(0, 0, 0, 0);
      }
    }
    return;
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < kLmStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kLmBM);
    }
    fence_mbar_init();
  }
  if (warp == 1) {   // TMEM: two 256-column fp32 accumulators (all 512 columns)
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
      uint32_t q = 0;
      for (int tile = t_begin; tile < t_end; ++tile) {
        for (int kb = 0; kb < nk; ++kb, ++q) {
          const int s = q % kLmStages;
          mbar_wait(&empty[s], ((q / kLmStages) & 1u) ^ 1u);
          mbar_arrive_tx(&full[s], kLmStageBytes);
          tma_load_2d(sA + s * kLmABytes, &tmap_h, kb * kLmBK, m0, &full[s]);
          tma_load_2d(sB + s * kLmBBytes, &tmap_w, kb * kLmBK, tile * kLmBN, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t q = 0;
      int i = 0;
      for (int tile = t_begin; tile < t_end; ++tile, ++i) {
        const int acc = i & 1;
        mbar_wait(&tempty[acc], ((i >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t dt = tmem + uint32_t(acc * kLmBN);
        for (int kb = 0; kb < nk; ++kb, ++q) {
          const int s = q % kLmStages;
          mbar_wait(&full[s], (q / kLmStages) & 1u);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * kLmABytes), b0 = smem_u32(sB + s * kLmBBytes);
#pragma unroll
          for (int k = 0; k < kLmBK / 16; ++k)   // K = 16 per MMA: +32 bytes inside the atom
            tc_mma(dt, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), kLmIdesc,
                   (kb | k) != 0);
          tc_commit(&empty[s]);                  // smem stage free once these MMAs finish
        }
        tc_commit(&tfull[acc]);                  // accumulator ready for the epilogue
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue
    const int quarter = warp & 3;                // TMEM lanes this warp may access
    const int row = quarter * 32 + lane;
    const int r = m0 + row;
    if constexpr (kDz) {
      BwdRec rc;
      rc.ng = 0.f;
      rc.y = -1;
      if (r < n_rows) rc = p.rec[r];
      int i = 0;
      for (int tile = t_begin; tile < t_end; ++tile, ++i) {
        const int acc = i & 1;
        mbar_wait(&tfull[acc], (i >> 1) & 1u);
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
        mbar_arrive(&tempty[acc]);
      }
    } else {
    const bool valid = r < n_rows && p.ws.flag[p.row_begin + r];
    const int y = valid ? p.tokens[r] : -1;
    const float lamL = p.lam_log2e;
    float R = -INFINITY, S = 0.f, W = 0.f, cS = 0.f, cW = 0.f, uy = __int_as_float(0x7fc00000);
    int i = 0;
    for (int tile = t_begin; tile < t_end; ++tile, ++i) {
      const int acc = i & 1;
      mbar_wait(&tfull[acc], (i >> 1) & 1u);
      tc_fence_after();
      const uint32_t base = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(acc * kLmBN);
#pragma unroll 1
      for (int c = 0; c < kLmBN / 32; ++c) {
        float x[32];
        __syncwarp();                              // tcgen05.ld is .sync.aligned
        tmem_ld32(base + uint32_t(c * 32), x);
        const int col0 = tile * kLmBN + c * 32;
        if (!valid) continue;
        lm_row_chunk(x, col0, y, p.V, lamL, R, S, W, cS, cW, uy, p.ws.err);
      }
      __syncwarp();
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
    if (valid)
      reinterpret_cast<float4*>(p.partial)[int64_t(part) * p.n_rows + r] =
          make_float4(R, S - cS, W - cW, uy);
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

__global__ void __launch_bounds__(kLmThreads, 1)
    k_lmhead_fwd(const __grid_constant__ CUtensorMap tmap_h, const __grid_constant__ CUtensorMap tmap_w,
                 const LmParams p) {
  lmhead_body<false>(tmap_h, tmap_w, p);
}

__global__ void __launch_bounds__(kLmThreads, 1)
    k_lmhead_dz(const __grid_constant__ CUtensorMap tmap_h, const __grid_constant__ CUtensorMap tmap_w,
                const LmParams p) {
  lmhead_body<true>(tmap_h, tmap_w, p);
}

// Row flags / token copies for the fused path (no logits to read the target from).
__global__ void __launch_bounds__(256) k_lmh_rows(const int32_t* tokens, const float* old_logp,
                                                  const uint8_t* mask, int64_t row_begin,
                                                  int64_t n_rows, int V, Workspace ws) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = row_begin + r;
    const int y = tokens[r];
    ws.old[t] = old_logp[r];
    ws.y[t] = y;
    bool valid = (mask ? mask[r] != 0 : true) && ws.cand[ws.row_seq[t]];
    if (valid && (y < 0 || y >= V)) {
      set_error(ws.err, ESPO_ERR_TOKEN_OUT_OF_RANGE);
      valid = false;
    }
    ws.flag[t] = valid ? 1 : 0;
  }
}

}  // namespace espo
