// k_fwdgrad.cuh — factored-gradient forward sweep (DESIGN.md §9 "Factored gradient").
//
// The gradient of the loss w.r.t. a logits row factors into a row-local tensor and a scalar
// that is known only after the rollout-level reduction (K3):
//   d loss/d z_{t,v} = λ·g_t·(1[v = y_t] − p_v) = scale_t · G_t[v],
//   G_t = onehot(y_t) − softmax(λ z_t),  scale_t = λ·g_t = −λ·grad·c_t/D
// (stop-gradient: only the Eq. 1 numerator log π_θ(y_t) carries gradient, PAPER.md:111-113;
// c_t from Eqs. 1-3). G_t needs only the row itself, so it can be written
// in the same sweep that computes the row statistics. One CTA owns one row at a time:
//   pass 1 streams the row from HBM into the base-2 sums relative to u_y (K2's formulas),
//   a fixed-order fp64 block reduction gives lse, lp, H, q (K2's finish_stats),
//   pass 2 reads the row again — an L2 hit: one row per SM is live, 148 × 2V ≈ 45 MB — and
//   writes G_t (target entry q_t, no 1 − p cancellation).
// HBM traffic per valid row: 2V read + one G row written, against 2V + 2V + G for K2 + K5.
// Measured: two live rows per SM (two CTAs, or prefetching the next row) already
// thrash the L2 (2.8× the DRAM reads), so the depth has to come from inside the row: the
// default k_fwd_grad_ring streams both passes through a CTA-wide TMA ring (one producer
// warp); k_fwd_grad (plain loads, 1024 threads) is the simple variant.
// The consumer applies scale_t (espo_loss_row_scale) in its own GEMM epilogue or operand.
#pragma once
#include "common.cuh"
#include "workspace.cuh"
#include "k_rowlist.cuh"
#include "k_rowstats.cuh"
#include "k_dlogits.cuh"

namespace espo {


__device__ __forceinline__ uint4 ld_policy(const void* p, uint64_t pol, bool coherent) {
  uint4 r;
  if (coherent)
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Block-wide fixed-order sum of two per-thread values in fp64 (every thread gets the result).
template <int NT>
__device__ __forceinline__ void block_sum2(double& a, double& b, double* sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();                       // sm reuse across calls
  if (lane == 0) {
    sm[w] = a;
    sm[NT / 32 + w] = b;
  }
  __syncthreads();
  a = 0.0;
  b = 0.0;
#pragma unroll 4
  for (int k = 0; k < NT / 32; ++k) {
    a += sm[k];
    b += sm[NT / 32 + k];
  }
}
template <int NT>
__device__ __forceinline__ float block_max(float v, float* sm) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sm[w] = v;
  __syncthreads();
  float m = -INFINITY;
#pragma unroll 4
  for (int k = 0; k < NT / 32; ++k) m = fmaxf(m, sm[k]);
  return m;
}

// Consumer-only variants (named barrier 1 over NTC threads; the producer warp does not join).
__device__ __forceinline__ void bar_consumers(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
template <int NTC>
__device__ __forceinline__ void block_sum2_named(double& a, double& b, double* sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bar_consumers(NTC);
  if (lane == 0) {
    sm[w] = a;
    sm[NTC / 32 + w] = b;
  }
  bar_consumers(NTC);
  a = 0.0;
  b = 0.0;
#pragma unroll 4
  for (int k = 0; k < NTC / 32; ++k) {
    a += sm[k];
    b += sm[NTC / 32 + k];
  }
}
template <int NTC>
__device__ __forceinline__ float block_max_named(float v, float* sm) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bar_consumers(NTC);
  if (lane == 0) sm[w] = v;
  bar_consumers(NTC);
  float m = -INFINITY;
#pragma unroll 4
  for (int k = 0; k < NTC / 32; ++k) m = fmaxf(m, sm[k]);
  return m;
}

// Statistics of one row from the reduced (R, S, W) and u_y — K2's finish_stats, returning
// −lse·log2(e) and q for pass 2 as well as writing the workspace.
__device__ __forceinline__ void fg_stats(float R, float S, float W, float uy, const Workspace& ws,
                                         int64_t t, bool writer, float& nlseL, float& q) {
  const float ty = uy - R;
  const float ey = ex2(ty);
  const float Stot = ey + S;
  float lnS, lp;
  if (ey >= S) {
    const float l1 = log1pf(S / ey);
    lnS = fmaf(ty, kLn2, l1);
    lp = -l1;
  } else {
    lnS = logf(Stot);
    lp = fmaf(ty, kLn2, -lnS);
  }
  const float Wt = fmaf(ey, ty, W);
  float H = lnS - kLn2 * (Wt / Stot);
  H = H > 0.f ? H : 0.f;
  const float lse = fmaf(R, kLn2, lnS);
  q = S / Stot;
  nlseL = -lse * kLog2e;
  if (writer) {
    ws.lse[t] = lse;
    ws.lp[t] = lp;
    ws.H[t] = H;
    ws.q[t] = q;
  }
}

// Rows: k < count[0] are listed valid rows (FwdRec), count[0] ≤ k < count[0] + count[1] the
// zero-fill rows (zlist), claimed from count[2] one row ahead of the one being processed.
template <typename Tin, typename Tout, int NT, int U>
__global__ void __launch_bounds__(NT, 1024 / NT) k_fwd_grad(const FwdParams p, const FwdRec* list,
                                                    const int32_t* zlist, const int* count,
                                                    void* grad, int64_t ldg, int aliased) {
  constexpr int EPV = Vec<Tin>::EPV;
  __shared__ double s_red[2 * (NT / 32)];
  __shared__ int s_next[2];
  const int n = count[0], nz = count[1];
  int* claim = const_cast<int*>(count) + 2;
  const int V = p.V;
  const int nvec = (V + EPV - 1) / EPV;
  const int jrag = (V % EPV) ? nvec - 1 : -1;
  const float lamL = p.lam_log2e;
  const int64_t pitch = p.ld * int64_t(sizeof(Tin));
  const int64_t gpitch = ldg * int64_t(sizeof(Tout));
  const uint64_t pol1 = policy_evict_normal(), pol2 = policy_evict_first();
  const bool coh = aliased != 0;
  const int tid = threadIdx.x;
  if (tid == 0) s_next[0] = atomicAdd(claim, 1);
  __syncthreads();
  int k = s_next[0];
  for (int it = 1; k < n + nz; ++it) {
    // claim the next row now; it is read by all threads after this row's next barrier
    if (tid == 0) s_next[it & 1] = atomicAdd(claim, 1);
    if (k >= n) {                          // no gradient: zero-fill without reading
      char* orow = static_cast<char*>(grad) + int64_t(zlist[k - n]) * gpitch;
      constexpr int EPO = Out<Tout>::EPV;
      const int nfull = V / EPO;
      const uint4 z = make_uint4(0, 0, 0, 0);
      for (int j = tid; j < nfull; j += NT) st_stream(orow + int64_t(j) * 16, z);
      for (int c = nfull * EPO + tid; c < V; c += NT) {
        if (sizeof(Tout) == 4) reinterpret_cast<float*>(orow)[c] = 0.f;
        else reinterpret_cast<uint16_t*>(orow)[c] = 0;
      }
      __syncthreads();
      k = s_next[it & 1];
      continue;
    }
    const FwdRec rec = list[k];
    const char* row = static_cast<const char*>(p.logits) + int64_t(rec.r) * pitch;
    char* orow = static_cast<char*>(grad) + int64_t(rec.r) * gpitch;
    const int vy = rec.y / EPV, yoff = rec.y % EPV;
    const float uy = rec.uy;

    // ---- pass 1: S, W relative to R = u_y (HBM read)
    // fp32 sums per batch (two chains of ≤ 4·EPV/2 terms), accumulated in fp64 across batches:
    // rows with a low-probability target (lp ≈ −14) lose ~44× in H = ln S − ln2·W/S, so a
    // plain fp32 running sum over a thread's ~250 terms is not enough for 1e-5 on H
    float R = uy;
    double S = 0.0, W = 0.0;
    {
      const float2 L2 = make_float2(lamL, lamL), N2 = make_float2(-R, -R);
      for (int j0 = tid; j0 < nvec; j0 += NT * U) {
        float2 s2 = make_float2(0.f, 0.f), w2 = make_float2(0.f, 0.f);
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + NT * u;
          if (j < nvec) v[u] = ld_policy(row + int64_t(j) * 16, pol1, coh);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + NT * u;
          if (j < nvec) {
            float x[EPV];
            Vec<Tin>::unpack(v[u], x);
            if (j == vy || j == jrag) {    // target / ragged end: −inf, clamped (SAFE)
              fix_special<EPV>(x, j, vy, yoff, V);
              float s = 0.f, w = 0.f;
              acc_vec<EPV, true>(x, lamL, -R, s, w);
              s2.x += s;
              w2.x += w;
            } else {
#pragma unroll
              for (int e = 0; e < EPV; e += 2) {
                const float2 tt = __ffma2_rn(make_float2(x[e], x[e + 1]), L2, N2);
                const float2 ex = make_float2(ex2(tt.x), ex2(tt.y));
                s2 = __fadd2_rn(s2, ex);
                w2 = __ffma2_rn(ex, tt, w2);
              }
            }
          }
        }
        S += double(s2.x) + double(s2.y);
        W += double(w2.x) + double(w2.y);
      }
    }
    block_sum2<NT>(S, W, s_red);
    if (!(S < 0x1p100) || !(fabs(W) < 0x1p110)) {
      // rare: overflow against u_y (lp < −69), −inf logits (0·−inf) or NaN/+inf input —
      // redo the row with the row maximum as the reference and clamped exponents
      float m = -INFINITY;
      bool bad = false;
      for (int j = tid; j < nvec; j += NT) {
        float x[EPV];
        Vec<Tin>::unpack(ld_policy(row + int64_t(j) * 16, pol1, coh), x);
#pragma unroll
        for (int e = 0; e < EPV; ++e) {
          if (j * EPV + e >= V) continue;
          bad |= isnan(x[e]) || x[e] == INFINITY;
          m = fmaxf(m, x[e] * lamL);
        }
      }
      if (bad) set_error(p.ws.err, ESPO_ERR_NONFINITE_INPUT);
      R = block_max<NT>(m, reinterpret_cast<float*>(s_red));
      if (R == -INFINITY || !(R < INFINITY)) R = uy;   // all −inf but the target / bad row
      float s = 0.f, w = 0.f;
      for (int j = tid; j < nvec; j += NT) {
        float x[EPV];
        Vec<Tin>::unpack(ld_policy(row + int64_t(j) * 16, pol1, coh), x);
        fix_special<EPV>(x, j, vy, yoff, V);
        acc_vec<EPV, true>(x, lamL, -R, s, w);
      }
      S = s;
      W = w;
      block_sum2<NT>(S, W, s_red);
    }
    float nlseL, q;
    fg_stats(R, float(S), float(W), uy, p.ws, p.row_begin + rec.r, tid == 0, nlseL, q);

    const int k_after = s_next[it & 1];       // published by block_sum2's barriers

    // ---- pass 2: G = onehot(y) − p (L2 re-read, streaming stores)
    BwdRec g;
    g.ng = -1.f;
    g.nlseL = nlseL;
    g.gq = q;
    for (int j0 = tid; j0 < nvec; j0 += NT * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + NT * u;
        if (j < nvec) v[u] = ld_policy(row + int64_t(j) * 16, pol2, coh);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + NT * u;
        if (j < nvec) {
          float d[EPV];
          dz_vec<Tin>(v[u], j, vy, yoff, lamL, g, d);
          store_out<Tin, Tout>(orow, j, d, V);
        }
      }
    }
    k = k_after;
  }
}


// TMEM stash helpers: one warp stores / loads N consecutive 32-bit columns of its 32 lanes.
template <int N>
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  if constexpr (N == 8)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
                 "r"(r[6]), "r"(r[7]) : "memory");
  else
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};"
                 ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
}
template <int N>
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[N];
  if constexpr (N == 8)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7]) : "r"(taddr));
  else
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = __uint_as_float(r[i]);
}

// TMA-ring variant: one producer warp streams every row through a CTA-wide shared-memory
// ring twice — pass 1 from HBM, pass 2 again (an L2 hit) — so up to STAGES × CH bytes are in
// flight per SM independent of the consumers' registers, and the next row's pass-1 chunks
// load while the consumers still write the current row's G (HBM reads overlap writes).
// NC consumer warps; chunk c of a row holds vectors [c·VPC, (c+1)·VPC), VPC = CH/16, and
// consumer thread i takes vectors i, i + 32·NC, … of it. The producer claims rows (count[2]),
// publishes each slot's row in slot_row[] before its arrive (mbarrier release/acquire); a
// zero-fill row is one slot without data, the end one slot with k = INT_MAX.
template <typename Tin, typename Tout, int NC, int STAGES, int CH, int TM = 0>
__global__ void __launch_bounds__((NC + 1) * 32, 1) k_fwd_grad_ring(const FwdParams p,
                                                                   const FwdRec* list,
                                                                   const int32_t* zlist,
                                                                   const int* count, void* grad,
                                                                   int64_t ldg, int aliased) {
  constexpr int EPV = Vec<Tin>::EPV;
  constexpr int VPC = CH / 16;
  constexpr int NTC = NC * 32;                 // consumer threads
  static_assert(VPC % NTC == 0, "chunk must hold whole vectors per consumer thread");
  constexpr int VPT = VPC / NTC;               // vectors per consumer thread per chunk
  // TM: pass 1 keeps its 2^(u − u_y) of the first CT chunks of a row in TMEM (each warp owns
  // COLS columns of its lane quarter) and pass 2 turns them into p = 2^(u − u_y)·p_y with one
  // FMUL instead of a second MUFU exponential
  constexpr int WPQ = (NC + 3) / 4;            // consumer warps per TMEM lane quarter
  constexpr int COLS = (512 / WPQ) / (VPT * EPV) * (VPT * EPV);
  constexpr int CT = TM ? COLS / (VPT * EPV) : 0;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(STAGES) * CH);
  uint64_t* empty = full + STAGES;
  int* slot_row = reinterpret_cast<int*>(empty + STAGES);
  double* s_red = reinterpret_cast<double*>(slot_row + STAGES + (STAGES & 1));  // 8-B aligned
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_red + 2 * NC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int k = 0; k < STAGES; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], NC);
    }
    fence_mbar_init();
  }
  if (TM && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (TM) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (TM) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int n = count[0], nz = count[1];
  const int V = p.V;
  const int nvec = (V + EPV - 1) / EPV;
  const uint32_t rowbytes = uint32_t(nvec) * 16u;
  const int nch = static_cast<int>((rowbytes + CH - 1) / CH);
  const int64_t pitch = p.ld * int64_t(sizeof(Tin));

  if (warp == NC) {                            // ---------------- producer
    if (lane != 0) return;
    int* claim = const_cast<int*>(count) + 2;
    const char* base = static_cast<const char*>(p.logits);
    const uint64_t pol1 = policy_evict_normal(), pol2 = policy_evict_first();
    uint32_t q = 0;
    auto next_slot = [&]() {
      const int slot = q % STAGES;
      if (q >= STAGES) mbar_wait(&empty[slot], ((q / STAGES) - 1) & 1u);
      ++q;
      return slot;
    };
    for (;;) {
      const int k = atomicAdd(claim, 1);
      if (k >= n) {                            // zero-fill row or the end: a slot without data
        const int slot = next_slot();
        slot_row[slot] = k < n + nz ? k : INT_MAX;
        mbar_arrive(&full[slot]);
        if (k >= n + nz) return;
        continue;
      }
      const char* row = base + int64_t(list[k].r) * pitch;
      for (int pass = 0; pass < 2; ++pass) {
        for (int c = 0; c < nch; ++c) {
          const int slot = next_slot();
          const uint32_t off = uint32_t(c) * CH;
          const uint32_t bytes = min(uint32_t(CH), rowbytes - off);
          slot_row[slot] = k;
          mbar_arrive_tx(&full[slot], bytes);
          bulk_g2s(ring + size_t(slot) * CH, row + off, bytes, &full[slot], pass ? pol2 : pol1);
        }
      }
    }
  }

  // ------------------------------------------------------------------ consumers
  const int tid = threadIdx.x;                 // 0 … NTC − 1
  const int jrag = (V % EPV) ? nvec - 1 : -1;
  const float lamL = p.lam_log2e;
  const int64_t gpitch = ldg * int64_t(sizeof(Tout));
  const bool coh = aliased != 0;
  uint32_t q = 0;
  auto take = [&](int& slot) {                 // waits for the next slot, returns its row
    slot = q % STAGES;
    mbar_wait(&full[slot], (q / STAGES) & 1u);
    ++q;
    return slot_row[slot];
  };
  auto release = [&](int slot) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  };
  // this warp's TMEM columns: lanes 32·(warp % 4) …, columns (warp / 4)·COLS …
  const uint32_t tcol = TM ? *tmem_slot + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * COLS) : 0u;
  const bool stash_ok = TM && nch > CT;        // the first CT chunks of every row are full
  for (;;) {
    int slot;
    const int k = take(slot);
    if (k >= n) {
      release(slot);
      if (k == INT_MAX) break;
      char* orow = static_cast<char*>(grad) + int64_t(zlist[k - n]) * gpitch;
      constexpr int EPO = Out<Tout>::EPV;
      const int nfull = V / EPO;
      const uint4 z = make_uint4(0, 0, 0, 0);
      for (int j = tid; j < nfull; j += NTC) st_stream(orow + int64_t(j) * 16, z);
      for (int c = nfull * EPO + tid; c < V; c += NTC) {
        if (sizeof(Tout) == 4) reinterpret_cast<float*>(orow)[c] = 0.f;
        else reinterpret_cast<uint16_t*>(orow)[c] = 0;
      }
      continue;
    }
    const FwdRec rec = list[k];
    const char* grow = static_cast<const char*>(p.logits) + int64_t(rec.r) * pitch;
    char* orow = static_cast<char*>(grad) + int64_t(rec.r) * gpitch;
    const int vy = rec.y / EPV, yoff = rec.y % EPV;
    const float uy = rec.uy;

    // ---- pass 1 (fp32 sums per chunk, fp64 across chunks: see k_fwd_grad)
    float R = uy;
    double S = 0.0, W = 0.0;
    {
      const float2 L2 = make_float2(lamL, lamL), N2 = make_float2(-R, -R);
      for (int c = 0; c < nch; ++c) {
        if (c > 0) take(slot);
        float2 s2 = make_float2(0.f, 0.f), w2 = make_float2(0.f, 0.f);
        uint4 v[VPT];
#pragma unroll
        for (int u = 0; u < VPT; ++u)
          v[u] = lds128(ring + size_t(slot) * CH + size_t(u * NTC + tid) * 16);
        release(slot);
        if (TM && stash_ok && c < CT) {          // full chunk: every lane has VPT vectors
#pragma unroll
          for (int u = 0; u < VPT; ++u) {
            const int j = c * VPC + u * NTC + tid;
            float x[EPV];
            Vec<Tin>::unpack(v[u], x);
            const bool spec = j == vy || j == jrag;
            if (spec) fix_special<EPV>(x, j, vy, yoff, V);
            uint32_t ev[EPV];
#pragma unroll
            for (int e = 0; e < EPV; e += 2) {
              float2 tt = __ffma2_rn(make_float2(x[e], x[e + 1]), L2, N2);
              if (spec) {
                tt.x = max_nan(tt.x, -127.f);
                tt.y = max_nan(tt.y, -127.f);
              }
              const float2 ex = make_float2(ex2(tt.x), ex2(tt.y));
              s2 = __fadd2_rn(s2, ex);
              w2 = __ffma2_rn(ex, tt, w2);
              ev[e] = __float_as_uint(ex.x);
              ev[e + 1] = __float_as_uint(ex.y);
            }
            tmem_st8<EPV>(tcol + uint32_t((c * VPT + u) * EPV), ev);
          }
          S += double(s2.x) + double(s2.y);
          W += double(w2.x) + double(w2.y);
          continue;
        }
#pragma unroll
        for (int u = 0; u < VPT; ++u) {
          const int j = c * VPC + u * NTC + tid;
          if (j >= nvec) continue;
          float x[EPV];
          Vec<Tin>::unpack(v[u], x);
          if (j == vy || j == jrag) {
            fix_special<EPV>(x, j, vy, yoff, V);
            float s = 0.f, w = 0.f;
            acc_vec<EPV, true>(x, lamL, -R, s, w);
            s2.x += s;
            w2.x += w;
          } else {
#pragma unroll
            for (int e = 0; e < EPV; e += 2) {
              const float2 tt = __ffma2_rn(make_float2(x[e], x[e + 1]), L2, N2);
              const float2 ex = make_float2(ex2(tt.x), ex2(tt.y));
              s2 = __fadd2_rn(s2, ex);
              w2 = __ffma2_rn(ex, tt, w2);
            }
          }
        }
        S += double(s2.x) + double(s2.y);
        W += double(w2.x) + double(w2.y);
      }
    }
    if (TM && stash_ok) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    block_sum2_named<NTC>(S, W, s_red);
    if (!(S < 0x1p100) || !(fabs(W) < 0x1p110)) {
      // rare (see k_fwd_grad): redo from global memory with the row maximum as reference
      float m = -INFINITY;
      bool bad = false;
      for (int j = tid; j < nvec; j += NTC) {
        float x[EPV];
        Vec<Tin>::unpack(coh ? ld_stream_coherent(grow + int64_t(j) * 16) : ld_stream(grow + int64_t(j) * 16), x);
#pragma unroll
        for (int e = 0; e < EPV; ++e) {
          if (j * EPV + e >= V) continue;
          bad |= isnan(x[e]) || x[e] == INFINITY;
          m = fmaxf(m, x[e] * lamL);
        }
      }
      if (bad) set_error(p.ws.err, ESPO_ERR_NONFINITE_INPUT);
      R = block_max_named<NTC>(m, reinterpret_cast<float*>(s_red));
      if (R == -INFINITY || !(R < INFINITY)) R = uy;
      float sa = 0.f, wa = 0.f;
      for (int j = tid; j < nvec; j += NTC) {
        float x[EPV];
        Vec<Tin>::unpack(coh ? ld_stream_coherent(grow + int64_t(j) * 16) : ld_stream(grow + int64_t(j) * 16), x);
        fix_special<EPV>(x, j, vy, yoff, V);
        acc_vec<EPV, true>(x, lamL, -R, sa, wa);
      }
      S = sa;
      W = wa;
      block_sum2_named<NTC>(S, W, s_red);
    }
    float nlseL, qv;
    fg_stats(R, float(S), float(W), uy, p.ws, p.row_begin + rec.r, tid == 0, nlseL, qv);

    // ---- pass 2
    BwdRec g;
    g.ng = -1.f;
    g.nlseL = nlseL;
    g.gq = qv;
    // the stash holds 2^(u − u_y); p = that · 2^(u_y − lse) (= p_y ≤ 1). Not after the slow
    // path (its reference moved off u_y and the stash may hold overflowed values).
    const bool use_stash = TM && stash_ok && R == uy;
    const float py2 = ex2(uy + nlseL);
    for (int c = 0; c < nch; ++c) {
      take(slot);
      if (TM && use_stash && c < CT) {
        release(slot);                          // the logits are not needed: p from TMEM
#pragma unroll
        for (int u = 0; u < VPT; ++u) {
          const int j = c * VPC + u * NTC + tid;
          float e[EPV];
          tmem_ld8<EPV>(tcol + uint32_t((c * VPT + u) * EPV), e);
          float d[EPV];
          const float2 P2 = make_float2(-py2, -py2);
#pragma unroll
          for (int q2 = 0; q2 < EPV; q2 += 2) {
            const float2 o = __fmul2_rn(P2, make_float2(e[q2], e[q2 + 1]));
            d[q2] = o.x;
            d[q2 + 1] = o.y;
          }
          if (j == vy) {
#pragma unroll
            for (int q2 = 0; q2 < EPV; ++q2)
              if (q2 == yoff) d[q2] = qv;
          }
          store_out<Tin, Tout>(orow, j, d, V);
        }
        continue;
      }
      uint4 v[VPT];
#pragma unroll
      for (int u = 0; u < VPT; ++u)
        v[u] = lds128(ring + size_t(slot) * CH + size_t(u * NTC + tid) * 16);
      release(slot);
#pragma unroll
      for (int u = 0; u < VPT; ++u) {
        const int j = c * VPC + u * NTC + tid;
        if (j >= nvec) continue;
        float d[EPV];
        dz_vec<Tin>(v[u], j, vy, yoff, lamL, g, d);
        store_out<Tin, Tout>(orow, j, d, V);
      }
    }
  }
  if (TM) {                                    // all consumer warps are done with TMEM
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    bar_consumers(NTC);
    if (warp == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "r"(512)
                   : "memory");
    }
  }
}

template <typename Tin, typename Tout, int NC, int STAGES, int CH, int TM = 0>
cudaError_t launch_fwd_grad_ring(const FwdParams& p, const FwdRec* list, const int32_t* zlist,
                                 const int* count, void* grad, int64_t ldg, int aliased,
                                 int num_sms, cudaStream_t s, int ctas_per_sm = 1) {
  static unsigned long long attr_mask = 0;
  auto k = k_fwd_grad_ring<Tin, Tout, NC, STAGES, CH, TM>;
  constexpr size_t smem = size_t(STAGES) * CH + size_t(STAGES) * 16 + size_t(STAGES + 1) * 4 + 8 +
                          size_t(NC) * 16 + 64;
  cudaError_t e = ensure_smem_attr(k, int(smem), attr_mask);
  if (e != cudaSuccess) return e;
  k<<<num_sms * ctas_per_sm, (NC + 1) * 32, smem, s>>>(p, list, zlist, count, grad, ldg, aliased);
  return cudaGetLastError();
}

// Rolling variant: the producer interleaves pass 2 of the previous row with pass 1 of the
// current one chunk by chunk — P2(k−1, 0), P1(k, 0), P2(k−1, 1), P1(k, 1), … — so each SM
// keeps HBM reads (the new row) and writes (the old row's G) in flight together all the time,
// including while the consumers reduce a finished row. Slot headers carry (row, pass, chunk);
// the consumers follow them. Measured slower than k_fwd_grad_ring (A/B option only): a
// chunk's L2 reuse distance grows to ~2 row-volumes and the re-reads start missing.
template <typename Tin, typename Tout, int NC, int STAGES, int CH>
__global__ void __launch_bounds__((NC + 1) * 32, 1) k_fwd_grad_roll(const FwdParams p,
                                                                   const FwdRec* list,
                                                                   const int32_t* zlist,
                                                                   const int* count, void* grad,
                                                                   int64_t ldg, int aliased) {
  constexpr int EPV = Vec<Tin>::EPV;
  constexpr int VPC = CH / 16;
  constexpr int NTC = NC * 32;
  static_assert(VPC % NTC == 0, "chunk must hold whole vectors per consumer thread");
  constexpr int VPT = VPC / NTC;
  constexpr int kZero = -1;                    // slot_meta of a zero-fill row
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(STAGES) * CH);
  uint64_t* empty = full + STAGES;
  int* slot_row = reinterpret_cast<int*>(empty + STAGES);
  int* slot_meta = slot_row + STAGES;
  double* s_red = reinterpret_cast<double*>(slot_meta + STAGES);   // 2·STAGES ints: 8-B aligned
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int k = 0; k < STAGES; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], NC);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int n = count[0], nz = count[1];
  const int V = p.V;
  const int nvec = (V + EPV - 1) / EPV;
  const uint32_t rowbytes = uint32_t(nvec) * 16u;
  const int nch = static_cast<int>((rowbytes + CH - 1) / CH);
  const int64_t pitch = p.ld * int64_t(sizeof(Tin));

  if (warp == NC) {                            // ---------------- producer
    if (lane != 0) return;
    int* claim = const_cast<int*>(count) + 2;
    const char* base = static_cast<const char*>(p.logits);
    const uint64_t pol1 = policy_evict_normal(), pol2 = policy_evict_first();
    uint32_t q = 0;
    auto next_slot = [&]() {
      const int slot = q % STAGES;
      if (q >= STAGES) mbar_wait(&empty[slot], ((q / STAGES) - 1) & 1u);
      ++q;
      return slot;
    };
    auto emit = [&](int k, const char* row, int pass, int c) {
      const int slot = next_slot();
      const uint32_t off = uint32_t(c) * CH;
      const uint32_t bytes = min(uint32_t(CH), rowbytes - off);
      slot_row[slot] = k;
      slot_meta[slot] = pass | (c << 1);
      mbar_arrive_tx(&full[slot], bytes);
      bulk_g2s(ring + size_t(slot) * CH, row + off, bytes, &full[slot], pass ? pol2 : pol1);
    };
    int prevk = -1;
    const char* prow = nullptr;
    for (;;) {
      const int k = atomicAdd(claim, 1);
      if (k >= n) {
        if (k < n + nz) {                      // zero-fill row: a slot without data
          const int slot = next_slot();
          slot_row[slot] = k;
          slot_meta[slot] = kZero;
          mbar_arrive(&full[slot]);
          continue;
        }
        if (prevk >= 0)
          for (int c = 0; c < nch; ++c) emit(prevk, prow, 1, c);
        const int slot = next_slot();          // the end
        slot_row[slot] = INT_MAX;
        slot_meta[slot] = kZero;
        mbar_arrive(&full[slot]);
        return;
      }
      const char* row = base + int64_t(list[k].r) * pitch;
      for (int c = 0; c < nch; ++c) {
        if (prevk >= 0) emit(prevk, prow, 1, c);
        emit(k, row, 0, c);
      }
      prevk = k;
      prow = row;
    }
  }

  // ------------------------------------------------------------------ consumers
  const int tid = threadIdx.x;
  const int jrag = (V % EPV) ? nvec - 1 : -1;
  const float lamL = p.lam_log2e;
  const int64_t gpitch = ldg * int64_t(sizeof(Tout));
  const bool coh = aliased != 0;
  const float2 L2 = make_float2(lamL, lamL);
  uint32_t q = 0;
  // current row (pass 1 in progress) and previous row (pass 2 pending)
  int cvy = 0, cyoff = 0, cr = 0;
  float cuy = 0.f;
  double S = 0.0, W = 0.0;
  int pvy = 0, pyoff = 0;
  char* porow = nullptr;
  BwdRec g;
  g.ng = -1.f;
  for (;;) {
    const int slot = q % STAGES;
    mbar_wait(&full[slot], (q / STAGES) & 1u);
    ++q;
    const int k = slot_row[slot], meta = slot_meta[slot];
    if (meta == kZero) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (k == INT_MAX) return;
      char* orow = static_cast<char*>(grad) + int64_t(zlist[k - n]) * gpitch;
      constexpr int EPO = Out<Tout>::EPV;
      const int nfull = V / EPO;
      const uint4 z = make_uint4(0, 0, 0, 0);
      for (int j = tid; j < nfull; j += NTC) st_stream(orow + int64_t(j) * 16, z);
      for (int c = nfull * EPO + tid; c < V; c += NTC) {
        if (sizeof(Tout) == 4) reinterpret_cast<float*>(orow)[c] = 0.f;
        else reinterpret_cast<uint16_t*>(orow)[c] = 0;
      }
      continue;
    }
    const int pass = meta & 1, c = meta >> 1;
    uint4 v[VPT];
#pragma unroll
    for (int u = 0; u < VPT; ++u) v[u] = lds128(ring + size_t(slot) * CH + size_t(u * NTC + tid) * 16);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (pass == 1) {                           // ---- G of the previous row
#pragma unroll
      for (int u = 0; u < VPT; ++u) {
        const int j = c * VPC + u * NTC + tid;
        if (j >= nvec) continue;
        float d[EPV];
        dz_vec<Tin>(v[u], j, pvy, pyoff, lamL, g, d);
        store_out<Tin, Tout>(porow, j, d, V);
      }
      continue;
    }
    // ---- pass 1 of the current row
    if (c == 0) {
      const FwdRec rec = list[k];
      cr = rec.r;
      cvy = rec.y / EPV;
      cyoff = rec.y % EPV;
      cuy = rec.uy;
      S = 0.0;
      W = 0.0;
    }
    {
      const float2 N2 = make_float2(-cuy, -cuy);
      float2 s2 = make_float2(0.f, 0.f), w2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int u = 0; u < VPT; ++u) {
        const int j = c * VPC + u * NTC + tid;
        if (j >= nvec) continue;
        float x[EPV];
        Vec<Tin>::unpack(v[u], x);
        if (j == cvy || j == jrag) {
          fix_special<EPV>(x, j, cvy, cyoff, V);
          float s = 0.f, w = 0.f;
          acc_vec<EPV, true>(x, lamL, -cuy, s, w);
          s2.x += s;
          w2.x += w;
        } else {
#pragma unroll
          for (int e = 0; e < EPV; e += 2) {
            const float2 tt = __ffma2_rn(make_float2(x[e], x[e + 1]), L2, N2);
            const float2 ex = make_float2(ex2(tt.x), ex2(tt.y));
            s2 = __fadd2_rn(s2, ex);
            w2 = __ffma2_rn(ex, tt, w2);
          }
        }
      }
      S += double(s2.x) + double(s2.y);
      W += double(w2.x) + double(w2.y);
    }
    if (c != nch - 1) continue;
    // ---- the row's last chunk: reduce, statistics, it becomes the pass-2 row
    const char* grow = static_cast<const char*>(p.logits) + int64_t(cr) * pitch;
    block_sum2_named<NTC>(S, W, s_red);
    float R = cuy;
    if (!(S < 0x1p100) || !(fabs(W) < 0x1p110)) {   // rare: see k_fwd_grad
      float m = -INFINITY;
      bool bad = false;
      for (int j = tid; j < nvec; j += NTC) {
        float x[EPV];
        Vec<Tin>::unpack(coh ? ld_stream_coherent(grow + int64_t(j) * 16) : ld_stream(grow + int64_t(j) * 16), x);
#pragma unroll
        for (int e = 0; e < EPV; ++e) {
          if (j * EPV + e >= V) continue;
          bad |= isnan(x[e]) || x[e] == INFINITY;
          m = fmaxf(m, x[e] * lamL);
        }
      }
      if (bad) set_error(p.ws.err, ESPO_ERR_NONFINITE_INPUT);
      R = block_max_named<NTC>(m, reinterpret_cast<float*>(s_red));
      if (R == -INFINITY || !(R < INFINITY)) R = cuy;
      float sa = 0.f, wa = 0.f;
      for (int j = tid; j < nvec; j += NTC) {
        float x[EPV];
        Vec<Tin>::unpack(coh ? ld_stream_coherent(grow + int64_t(j) * 16) : ld_stream(grow + int64_t(j) * 16), x);
        fix_special<EPV>(x, j, cvy, cyoff, V);
        acc_vec<EPV, true>(x, lamL, -R, sa, wa);
      }
      S = sa;
      W = wa;
      block_sum2_named<NTC>(S, W, s_red);
    }
    float nlseL, qv;
    fg_stats(R, float(S), float(W), cuy, p.ws, p.row_begin + cr, tid == 0, nlseL, qv);
    g.nlseL = nlseL;
    g.gq = qv;
    pvy = cvy;
    pyoff = cyoff;
    porow = static_cast<char*>(grad) + int64_t(cr) * gpitch;
  }
}

template <typename Tin, typename Tout, int NC, int STAGES, int CH>
cudaError_t launch_fwd_grad_roll(const FwdParams& p, const FwdRec* list, const int32_t* zlist,
                                 const int* count, void* grad, int64_t ldg, int aliased,
                                 int num_sms, cudaStream_t s) {
  static unsigned long long attr_mask = 0;
  auto k = k_fwd_grad_roll<Tin, Tout, NC, STAGES, CH>;
  constexpr size_t smem = size_t(STAGES) * CH + size_t(STAGES) * 16 + size_t(STAGES) * 8 +
                          size_t(NC) * 16 + 64;
  cudaError_t e = ensure_smem_attr(k, int(smem), attr_mask);
  if (e != cudaSuccess) return e;
  k<<<num_sms, (NC + 1) * 32, smem, s>>>(p, list, zlist, count, grad, ldg, aliased);
  return cudaGetLastError();
}

// scale_t = λ·g_t = −grad·(λ/D)·c_t for valid rows, 0 otherwise (dlogits_t = scale_t·G_t).
__global__ void __launch_bounds__(256) k_row_scale(int64_t row_begin, int64_t n_rows,
                                                   const float* grad_loss, Workspace ws,
                                                   float* out) {
  const float gl = grad_loss ? *grad_loss : 1.f;
  const float gscale = -gl * *ws.bwd_scale;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = row_begin + r;
    out[r] = ws.flag[t] ? gscale * ws.coef[t] : 0.f;
  }
}

}  // namespace espo
