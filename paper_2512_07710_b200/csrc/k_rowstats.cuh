// k_rowstats.cuh — K2: the forward vocab sweep.
//
// For every valid row t of an active rollout, one pass over λ·z_t computes, in base-2
// units u = λ·log2(e)·z and relative to a per-lane reference r (initially u_y, the target):
//   S = Σ_{v≠y} 2^{u_v − r},   W = Σ_{v≠y} 2^{u_v − r}·(u_v − r)
// and then lse = log Σ e^{λz}, lp = log p_y (Eq. 1 numerator),
// H = −Σ p log p (Eq. 3's e_t) and q = 1 − p_y.
// Choosing r = u_y makes e_y = 1 exactly, so lp = −log1p(S) and q = S/(1+S) are accurate
// for near-deterministic rows (no 1 − p cancellation). A batch whose sum leaves the safe
// range (lp < −69, NaN/+inf input) is recomputed with a max-based reference (rare path).
// No tensor cores: this is a streaming reduction (K2).
#pragma once
#include "common.cuh"
#include "workspace.cuh"
#include "k_rowlist.cuh"

namespace espo {

struct FwdParams {
  const void* logits;
  int64_t ld;           // elements
  const int32_t* tokens;
  const float* old_logp;
  const uint8_t* mask;  // nullable
  int64_t row_begin, n_rows;
  int V;                // columns of a logits row held here (the shard width if sharded)
  float lam_log2e;      // λ·log2(e)
  float* partial;       // vocabulary-parallel: per-row {R, S, W, u_y} instead of statistics
  // vocabulary-parallel over peer memory: the partial of chunk row r goes straight to
  // xbase[k][xoff + r] for every TP rank k (NVLink stores into the peers' exchange buffers)
  float4* const* xbase = nullptr;
  int nx = 0;
  int64_t xoff = 0;
  Workspace ws;
};

__device__ __forceinline__ float max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// Accumulates EPV elements (already unpacked) into (s, w) relative to reference nref = −r.
// Fast form: a −inf logit gives e·t = 0·(−inf) = NaN, which routes the batch to the slow
// path (SAFE form: t clamped at −127 with NaN propagation, so −inf contributes exactly 0).
template <int EPV, bool SAFE = false>
__device__ __forceinline__ void acc_vec(const float* x, float lamL, float nref, float& s,
                                        float& w) {
#pragma unroll
  for (int e = 0; e < EPV; ++e) {
    float t = fmaf(x[e], lamL, nref);
    if (SAFE) t = max_nan(t, -127.f);
    const float ex = ex2(t);
    s += ex;
    w = fmaf(ex, t, w);
  }
}

// Sets the target element and the elements past V of a vector to −inf (they contribute 0).
template <int EPV>
__device__ __forceinline__ void fix_special(float* x, int j, int vy, int yoff, int V) {
  // compile-time element indices only (a runtime index would put x in local memory)
#pragma unroll
  for (int e = 0; e < EPV; ++e)
    if ((j == vy && e == yoff) || j * EPV + e >= V) x[e] = -INFINITY;
}

// Compensated (Kahan) accumulation of the per-batch sums into the per-lane row sums:
// a lane adds ~150 batch sums per row, so a plain running sum would lose ~1e-5 relative.
__device__ __forceinline__ void kahan_add(float& s, float& c, float x) {
  const float y = x - c;
  const float t = s + y;
  c = (t - s) - y;
  s = t;
}

// Final statistics from (R, S, W) = (reference, Σ_{v≠y} 2^{u_v−R}, Σ 2^{u_v−R}(u_v−R)) and
// the target's u_y ≤ R: lse, lp = log p_y, H, q = 1 − p_y.
__device__ __forceinline__ void finish_stats(float R, float S, float W, float uy,
                                             const Workspace& ws, int64_t t) {
  {
    const float ty = uy - R;               // ≤ 0
    const float ey = ex2(ty);              // = 1 when no lane moved its reference
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
    const float Wt = fmaf(ey, ty, W);      // add the target's own e·t term
    float H = lnS - kLn2 * (Wt / Stot);
    H = H > 0.f ? H : 0.f;                 // also maps −0 and tiny negative rounding to +0
    ws.lse[t] = fmaf(R, kLn2, lnS);
    ws.lp[t] = lp;
    ws.H[t] = H;
    ws.q[t] = S / Stot;
  }
}

// Rescales (S, W) from reference r to R ≥ r (r = −inf: nothing accumulated yet).
__device__ __forceinline__ void rebase(float r, float R, float& S, float& W) {
  if (r == R) return;
  if (r == -INFINITY || (S == 0.f && W == 0.f)) {
    S = 0.f;
    W = 0.f;
    return;
  }
  const float d = r - R;
  const float sc = ex2(d);
  W = sc * fmaf(d, S, W);
  S = sc * S;
}

// Row epilogue: combine lanes (each lane may hold its own reference r), then write the row
// statistics — or, for a vocabulary shard, the row's partial {R, S, W, u_y}.
__device__ __forceinline__ void row_finish(float r, float S, float W, float uy, const Workspace& ws,
                                           int64_t t, int lane, float* partial = nullptr,
                                           int64_t pr = 0, float4* const* xbase = nullptr,
                                           int nx = 0, int64_t xoff = 0) {
  const float R = warp_max(r);
  if (R == -INFINITY) {
    S = 0.f;
    W = 0.f;
  } else {
    rebase(r, R, S, W);
  }
  S = warp_sum(S);
  W = warp_sum(W);
  if (lane == 0) {
    if (nx > 0) {            // fused exchange: the partial goes to every TP rank's buffer
      const float4 v = make_float4(R, S, W, uy);
      for (int k = 0; k < nx; ++k) xbase[k][xoff + pr] = v;
    } else if (partial) {
      reinterpret_cast<float4*>(partial)[pr] = make_float4(R, S, W, uy);
    } else {
      finish_stats(R, S, W, uy, ws, t);
    }
  }
}

// Vocabulary-parallel combine: one thread per valid row merges the shards' partials
// {R_k, S_k, W_k, u_y (owner only)} laid out [n_shards][n_rows] into the row statistics.
__global__ void __launch_bounds__(256) k_fwd_combine(const float4* partials, int n_shards,
                                                     int64_t row_begin, int64_t n_rows,
                                                     Workspace ws) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = row_begin + r;
    if (!ws.flag[t]) continue;
    float R = -INFINITY, uy = __int_as_float(0x7fc00000);
    for (int k = 0; k < n_shards; ++k) {
      const float4 a = partials[int64_t(k) * n_rows + r];
      R = fmaxf(R, a.x);
      if (!isnan(a.w)) uy = a.w;
    }
    float S = 0.f, W = 0.f;
    for (int k = 0; k < n_shards; ++k) {
      const float4 a = partials[int64_t(k) * n_rows + r];
      float s = a.y, w = a.z;
      rebase(a.x, R, s, w);
      S += s;
      W += w;
    }
    if (isnan(uy)) set_error(ws.err, ESPO_ERR_INVALID_ARGUMENT);  // no shard owns the target
    finish_stats(R, S, W, uy, ws, t);
  }
}

// The same merge for many partials per row (the LM head on the GEMM core: two per 512-column
// vocabulary tile, ~600 at V = 151,936): one warp per row with the lanes striding over the
// partials (a thread per row left most SMs idle: 315 µs per 8192 rows), the rebased terms
// 2^(R_k − R)·S_k summed in fp64 (one rounding at the end: no error growth with the count).
__global__ void __launch_bounds__(256) k_fwd_combine64(const float4* partials, int n_shards,
                                                       int64_t row_begin, int64_t n_rows,
                                                       Workspace ws) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < n_rows; r += nw) {
    const int64_t t = row_begin + r;
    if (!ws.flag[t]) continue;                       // warp-uniform
    float R = -INFINITY, uy = __int_as_float(0x7fc00000);
    for (int k = lane; k < n_shards; k += 32) {
      const float4 a = partials[int64_t(k) * n_rows + r];
      R = fmaxf(R, a.x);
      if (!isnan(a.w)) uy = a.w;
    }
    R = warp_max(R);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {             // the one owner's u_y to every lane
      const float u = __shfl_xor_sync(0xffffffffu, uy, o);
      if (isnan(uy)) uy = u;
    }
    double S = 0.0, W = 0.0;
    for (int k = lane; k < n_shards; k += 32) {
      const float4 a = partials[int64_t(k) * n_rows + r];
      if (a.x == -INFINITY || (a.y == 0.f && a.z == 0.f)) continue;
      const float d = a.x - R;                       // ≤ 0
      const float sc = ex2(d);
      W += double(sc) * (double(d) * double(a.y) + double(a.z));
      S += double(sc) * double(a.y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      S += __shfl_xor_sync(0xffffffffu, S, o);
      W += __shfl_xor_sync(0xffffffffu, W, o);
    }
    if (lane == 0) {
      if (isnan(uy)) set_error(ws.err, ESPO_ERR_INVALID_ARGUMENT);  // no tile holds the target
      finish_stats(R, float(S), float(W), uy, ws, t);
    }
  }
}

// Slow path for one batch: NaN/+inf detection and a max-based reference. Re-unpacks the
// packed vectors (kept in registers) instead of holding U·EPV floats.
template <typename Tin, int U, int STRIDE = 32>   // vector k of the batch is j0 + STRIDE·k
__device__ __forceinline__ void batch_slow(const uint4* v, int j0, int nvec, int vy, int yoff,
                                           int jrag, int V, float lamL, float& r, float& S,
                                           float& W, float& bS, float& bW, int* err) {
  constexpr int EPV = Vec<Tin>::EPV;
  float bm = -INFINITY;
  bool bad = false;
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const int j = j0 + STRIDE * k;
    if (j >= nvec) continue;
    float x[EPV];
    Vec<Tin>::unpack(v[k], x);
    fix_special<EPV>(x, j, vy, yoff, V);
#pragma unroll
    for (int e = 0; e < EPV; ++e) {
      const float u = x[e] * lamL;
      bad |= isnan(u) || u == INFINITY;
      bm = fmaxf(bm, u);
    }
  }
  if (bad) {
    set_error(err, ESPO_ERR_NONFINITE_INPUT);
    bS = __int_as_float(0x7fc00000);
    bW = bS;
    return;
  }
  if (bm > r + 60.f) {  // keep r = u_y (exact e_y = 1) unless the batch could overflow
    rebase(r, bm, S, W);
    r = bm;
  }
  bS = 0.f;
  bW = 0.f;
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const int j = j0 + STRIDE * k;
    if (j >= nvec) continue;
    float x[EPV];
    Vec<Tin>::unpack(v[k], x);
    fix_special<EPV>(x, j, vy, yoff, V);
    acc_vec<EPV, true>(x, lamL, -r, bS, bW);
  }
}

// Special batch (holds the target vector, the ragged vocabulary end or vectors past the row
// end): one pass with the target / out-of-range elements set to −inf and the SAFE form
// (t clamped at −127: −inf contributes exactly 0 under ftz), relative to the current
// reference. The caller falls back to batch_slow if the sums overflow or carry NaN/+inf.
template <typename Tin, int U, int STRIDE = 32>
__device__ __forceinline__ void batch_safe(const uint4* v, int j0, int nvec, int vy, int yoff,
                                           int V, float lamL, float r, float& bS, float& bW) {
  constexpr int EPV = Vec<Tin>::EPV;
  bS = 0.f;
  bW = 0.f;
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const int j = j0 + STRIDE * k;
    if (j >= nvec) continue;
    float x[EPV];
    Vec<Tin>::unpack(v[k], x);
    fix_special<EPV>(x, j, vy, yoff, V);
    acc_vec<EPV, true>(x, lamL, -r, bS, bW);
  }
}

// Fast path: U vectors into the batch sums with no per-vector checks. The batch that
// holds the target element or the ragged end of the row (at most two per lane and row)
// is routed to batch_slow instead (see `special`).
// NPOLY elements of every 8 (the odd slots 7, then 3) take 2^t from ex2_poly on the FMA
// pipe instead of MUFU.EX2, balancing the two pipes (K2).
template <int NPOLY>
__device__ __forceinline__ float ex2_mix(float t, int e) {
  const bool poly = (NPOLY >= 1 && (e & 7) == 7) || (NPOLY >= 2 && (e & 7) == 3);
  return poly ? ex2_poly(t) : ex2(t);
}

template <typename Tin, int U, int NPOLY = 0>
__device__ __forceinline__ void acc_batch(const uint4* v, float lamL, float nref, float& bS,
                                          float& bW) {
  constexpr int EPV = Vec<Tin>::EPV;
  if constexpr (NPOLY < 0) {
    // packed variant: the same two (s, w) chains as below, issued as sm_100 f32x2 FFMA2 /
    // FADD2 pairs (bitwise the same per-lane arithmetic, half the FP32 instructions)
    const float2 L2 = make_float2(lamL, lamL), N2 = make_float2(nref, nref);
    float2 s, w;
    {
      float x[EPV];
      Vec<Tin>::unpack(v[0], x);
      const float2 t = __ffma2_rn(make_float2(x[0], x[1]), L2, N2);
      const float2 e = make_float2(ex2(t.x), ex2(t.y));
      s = e;
      w = __fmul2_rn(e, t);
#pragma unroll
      for (int k = 2; k < EPV; k += 2) {
        const float2 tk = __ffma2_rn(make_float2(x[k], x[k + 1]), L2, N2);
        const float2 ek = make_float2(ex2(tk.x), ex2(tk.y));
        s = __fadd2_rn(s, ek);
        w = __ffma2_rn(ek, tk, w);
      }
    }
#pragma unroll
    for (int u = 1; u < U; ++u) {
      float x[EPV];
      Vec<Tin>::unpack(v[u], x);
#pragma unroll
      for (int k = 0; k < EPV; k += 2) {
        const float2 tk = __ffma2_rn(make_float2(x[k], x[k + 1]), L2, N2);
        const float2 ek = make_float2(ex2(tk.x), ex2(tk.y));
        s = __fadd2_rn(s, ek);
        w = __ffma2_rn(ek, tk, w);
      }
    }
    bS = s.x + s.y;
    bW = w.x + w.y;
    return;
  }
  // two (s, w) chains, seeded by the first vector (no 0 + x instructions)
  float s0, s1, w0, w1;
  {
    float x[EPV];
    Vec<Tin>::unpack(v[0], x);
    const float t0 = fmaf(x[0], lamL, nref), t1 = fmaf(x[1], lamL, nref);
    const float e0 = ex2_mix<NPOLY>(t0, 0), e1 = ex2_mix<NPOLY>(t1, 1);
    s0 = e0; s1 = e1; w0 = e0 * t0; w1 = e1 * t1;
#pragma unroll
    for (int e = 2; e < EPV; e += 2) {
      const float ta = fmaf(x[e], lamL, nref), tb = fmaf(x[e + 1], lamL, nref);
      const float ea = ex2_mix<NPOLY>(ta, e), eb = ex2_mix<NPOLY>(tb, e + 1);
      s0 += ea; s1 += eb; w0 = fmaf(ea, ta, w0); w1 = fmaf(eb, tb, w1);
    }
  }
#pragma unroll
  for (int k = 1; k < U; ++k) {
    float x[EPV];
    Vec<Tin>::unpack(v[k], x);
#pragma unroll
    for (int e = 0; e < EPV; e += 2) {
      const float ta = fmaf(x[e], lamL, nref), tb = fmaf(x[e + 1], lamL, nref);
      const float ea = ex2_mix<NPOLY>(ta, e), eb = ex2_mix<NPOLY>(tb, e + 1);
      s0 += ea; s1 += eb; w0 = fmaf(ea, ta, w0); w1 = fmaf(eb, tb, w1);
    }
  }
  bS = s0 + s1;
  bW = w0 + w1;
}

// A row with no target in this vocabulary shard starts without a reference (−inf), which would
// send its first batch through batch_slow on every lane (measured: 15 % of the sweep's
// instructions at 1/8-vocabulary shard rows). Instead each lane takes the largest element of
// its first vector as its reference when that is finite (the element itself contributes
// 2^0, so the lane's sums never underflow; elements up to ~90 above it stay in range, and
// anything else still falls back to batch_slow). Lanes combine with rebasing (row_finish).
template <typename Tin>
__device__ __forceinline__ void seed_ref(float& ref, const uint4& v0, float lamL) {
  if (ref != -INFINITY) return;
  float x[Vec<Tin>::EPV];
  Vec<Tin>::unpack(v0, x);
  float m = x[0];
#pragma unroll
  for (int e = 1; e < Vec<Tin>::EPV; ++e) m = fmaxf(m, x[e]);
  const float u = m * lamL;
  if (fabsf(u) < 1e30f) ref = u;         // not the −1e30 padding, not ±inf / NaN
}

// True if the batch j0 + 32k (k < U) contains vector vy or the ragged last vector jrag.
template <int U>
__device__ __forceinline__ bool special_batch(int j0, int vy, int jrag) {
  const unsigned dy = static_cast<unsigned>(vy - j0);
  const unsigned dr = static_cast<unsigned>(jrag - j0);
  return (dy < 32u * U && (dy & 31u) == 0) || (jrag >= 0 && dr < 32u * U && (dr & 31u) == 0);
}

// ---------------------------------------------------------------------------------------
// Variant LDG: warp per row, 128-bit LDG (L1::no_allocate), U vectors in flight per lane.
// ---------------------------------------------------------------------------------------
template <typename Tin, int U>
__global__ void __launch_bounds__(256) k_rowstats_ldg(const FwdParams p, const FwdRec* list,
                                                      const int* count) {
  constexpr int EPV = Vec<Tin>::EPV;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int n = *count;
  const int nvec = (p.V + EPV - 1) / EPV;
  const int jrag = (p.V % EPV) ? nvec - 1 : -1;
  const float lamL = p.lam_log2e;
  const uint4 ninf = make_uint4(Vec<Tin>::kNegInfWord, Vec<Tin>::kNegInfWord, Vec<Tin>::kNegInfWord,
                                Vec<Tin>::kNegInfWord);
  for (int k = gw; k < n; k += nw) {
    const FwdRec rec = list[k];
    const char* row = static_cast<const char*>(p.logits) + int64_t(rec.r) * p.ld * int64_t(sizeof(Tin));
    const int vy = rec.yl >= 0 ? rec.yl / EPV : -1, yoff = rec.yl >= 0 ? rec.yl % EPV : 0;
    float ref = rec.yl >= 0 ? rec.uy : -INFINITY, S = 0.f, W = 0.f, cS = 0.f, cW = 0.f;
    for (int j0 = lane; j0 < nvec; j0 += 32 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + 32 * u;
        v[u] = (j < nvec) ? ld_stream(row + int64_t(j) * 16) : ninf;
      }
      if (j0 == lane && vy < 0 && jrag != lane) seed_ref<Tin>(ref, v[0], lamL);
      float bS, bW;
      acc_batch<Tin, U>(v, lamL, -ref, bS, bW);
      if (special_batch<U>(j0, vy, jrag) || !(bS < 0x1p100f) || !(fabsf(bW) < 0x1p110f)) {
        S -= cS;
        W -= cW;
        cS = cW = 0.f;
        batch_slow<Tin, U>(v, j0, nvec, vy, yoff, jrag, p.V, lamL, ref, S, W, bS, bW, p.ws.err);
      }
      kahan_add(S, cS, bS);
      kahan_add(W, cW, bW);
    }
    row_finish(ref, S - cS, W - cW, rec.uy, p.ws, p.row_begin + rec.r, lane, p.partial, rec.r,
               p.xbase, p.nx, p.xoff);
  }
  // peer-memory exchange: lane 0 issued this warp's partial stores; one system-scope fence
  // orders them before k_tpx_signal's release of the ready flags
  if (p.nx > 0 && lane == 0) __threadfence_system();
}

// ---------------------------------------------------------------------------------------
// Variant TMA: warp per row; each warp owns a STAGES-deep ring of CHUNK-byte shared-memory
// slots filled by cp.async.bulk (the TMA engine; completion on one mbarrier per slot).
// Steady state per chunk: wait on the slot, read it with conflict-free 128-bit LDS in
// sub-batches of 8 vectors per lane (computing as it goes), release the slot and have lane 0
// issue the chunk STAGES ahead (same row or the next one) into it. The first STAGES chunks
// of a warp are issued up front; the ring then runs across row boundaries.
// ---------------------------------------------------------------------------------------
template <typename Tin, int NW, int STAGES, int CHUNK, int SUB, int NPOLY>
__global__ void __launch_bounds__(NW * 32, 1) k_rowstats_tma(const FwdParams p,
                                                             const FwdRec* list, const int* count) {
  constexpr int EPV = Vec<Tin>::EPV;
  constexpr int VPC = CHUNK / 16;  // vectors per chunk; SUB = vectors per lane per sub-batch
  constexpr int NSUB = VPC / (32 * SUB);
  static_assert(VPC % (32 * SUB) == 0, "chunk must hold whole sub-batches");
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + size_t(warp) * STAGES * CHUNK;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(NW) * STAGES * CHUNK) + warp * STAGES;
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int n = *count;
  const int nw = gridDim.x * NW;
  const int gw = blockIdx.x * NW + warp;
  if (gw >= n) return;
  const int nvec = (p.V + EPV - 1) / EPV;
  const uint32_t rowbytes = uint32_t(nvec) * 16u;
  const int nch = static_cast<int>((rowbytes + CHUNK - 1) / CHUNK);
  const int jrag = (p.V % EPV) ? nvec - 1 : -1;
  const float lamL = p.lam_log2e;
  const int64_t pitch = p.ld * int64_t(sizeof(Tin));
  const char* base = static_cast<const char*>(p.logits);
  const uint64_t pol = policy_evict_first();
  const uint4 ninf = make_uint4(Vec<Tin>::kNegInfWord, Vec<Tin>::kNegInfWord, Vec<Tin>::kNegInfWord,
                                Vec<Tin>::kNegInfWord);
  // General chunks (target vector, ragged end, past the row end) on the packed fast path:
  // the excluded elements are replaced in registers by the finite −1e30 (2^(−1e30·λ·log2e
  // − r) = 0 and 0·t = 0 exactly, where −inf would give 0·(−inf) = NaN), by the one lane
  // holding the target / ragged vector; vectors past the row end load as −1e30. Valid while
  // −1e30·λ·log2e stays finite (λ < 1e6; otherwise the SAFE batch form is used).
  const bool bigneg = lamL < 1e6f;
  const uint4 nbig = make_uint4(Vec<Tin>::kBigNegWord, Vec<Tin>::kBigNegWord,
                                Vec<Tin>::kBigNegWord, Vec<Tin>::kBigNegWord);
  const int keep_rag = p.V % EPV;          // valid elements of the ragged vector jrag

  // Row assignment: the first row of every warp is static (gw); after that, for rows of ≥ 16
  // ring chunks, warps CLAIM rows dynamically (atomic counter count[1], one row ahead) so
  // faster warps take more rows and the sweep does not wait for the slowest warp's static
  // share (C1 fwd +2.3 %); shorter rows keep the static stride nw (TP8 shards: −3.8 % with
  // claims).
  const bool dyn = nch >= STAGES + 2 && nch >= 16;   // short rows: the claim costs more than it saves
  int* claim = const_cast<int*>(count) + 1;
  auto next_index = [&](int cur) {   // warp-uniform
    if (!dyn) return cur + nw;
    int v = 0;
    if (lane == 0) v = atomicAdd(claim, 1);
    return nw + __shfl_sync(0xffffffffu, v, 0);
  };
  // producer cursor: (row pk with record prec, chunk pc); the next row (pk_next, prec_next)
  // is fetched one row ahead. With nch ≥ STAGES + 2 the producer is never more than one row
  // ahead of the consumer, so the consumer's next row is the producer's current one.
  int pk = gw, pc = 0;
  FwdRec prec = list[pk];
  int pk_next = next_index(pk);
  FwdRec prec_next = (pk_next < n) ? list[pk_next] : prec;
  auto issue_one = [&](int slot) {  // issues the cursor's chunk into `slot`, advances cursor
    const uint32_t off = uint32_t(pc) * CHUNK;
    const uint32_t bytes = min(uint32_t(CHUNK), rowbytes - off);
    if (lane == 0) {
      mbar_arrive_tx(&bars[slot], bytes);
      bulk_g2s(ring + slot * CHUNK, base + int64_t(prec.r) * pitch + off, bytes, &bars[slot], pol);
    }
    if (++pc == nch) {
      pc = 0;
      pk = pk_next;
      prec = prec_next;
      if (pk < n) {
        pk_next = next_index(pk);
        if (pk_next < n) prec_next = list[pk_next];
      }
    }
  };
  for (int s = 0; s < STAGES && pk < n; ++s) issue_one(s);

  uint32_t q = 0;  // chunks consumed by this warp
  FwdRec rec_next = list[gw];
  for (int k = gw; k < n;) {
    const FwdRec rec = rec_next;
    if (!dyn && k + nw < n) rec_next = list[k + nw];
    const int vy = rec.yl >= 0 ? rec.yl / EPV : -1, yoff = rec.yl >= 0 ? rec.yl % EPV : 0;
    float ref = rec.yl >= 0 ? rec.uy : -INFINITY, S = 0.f, W = 0.f, cS = 0.f, cW = 0.f;
    const int cy = vy >= 0 ? vy / VPC : -1;  // chunk holding the target; the ragged vector is in the last
    for (int c = 0; c < nch; ++c, ++q) {
      const int slot = q % STAGES;
      mbar_wait(&bars[slot], (q / STAGES) & 1u);
      const uint8_t* buf = ring + slot * CHUNK;
      if (c != cy && c != nch - 1) {
        // ---- fast chunk: full, no target, no ragged end (all but ≤ 2 chunks of a row)
        const uint8_t* lbuf = buf + lane * 16;
        float cSum = 0.f, cWsum = 0.f;
#pragma unroll
        for (int h = 0; h < NSUB; ++h) {
          uint4 v[SUB];
#pragma unroll
          for (int u = 0; u < SUB; ++u) v[u] = lds128(lbuf + (h * 32 * SUB + 32 * u) * 16);
          if (h == NSUB - 1) {
            __syncwarp();                        // every lane has read the slot
            if (pk < n) issue_one(slot);         // refill it STAGES chunks ahead
          }
          if (h == 0 && c == 0) seed_ref<Tin>(ref, v[0], lamL);
          float bS, bW;
          acc_batch<Tin, SUB, NPOLY>(v, lamL, -ref, bS, bW);
          if (!(bS < 0x1p100f) || !(fabsf(bW) < 0x1p110f)) {
            kahan_add(S, cS, cSum);
            kahan_add(W, cW, cWsum);
            cSum = cWsum = 0.f;
            S -= cS;
            W -= cW;
            cS = cW = 0.f;
            batch_slow<Tin, SUB>(v, c * VPC + h * 32 * SUB + lane, nvec, vy, yoff, jrag, p.V,
                                 lamL, ref, S, W, bS, bW, p.ws.err);
          }
          cSum += bS;
          cWsum += bW;
        }
        kahan_add(S, cS, cSum);
        kahan_add(W, cW, cWsum);
        continue;
      }
      // ---- general chunk: partial end of row, target vector, ragged vocabulary end
      const int vlim = min(VPC, nvec - c * VPC);
#pragma unroll
      for (int h = 0; h < NSUB; ++h) {
        if (h * 32 * SUB >= vlim) {            // past the row's end for every lane: nothing
          if (h == NSUB - 1) {                 // to add (warp-uniform), just refill the slot
            __syncwarp();
            if (pk < n) issue_one(slot);
          }
          continue;
        }
        uint4 v[SUB];
#pragma unroll
        for (int u = 0; u < SUB; ++u) {
          const int jl = h * 32 * SUB + lane + 32 * u;
          v[u] = (jl < vlim) ? lds128(buf + jl * 16) : (bigneg ? nbig : ninf);
        }
        if (h == NSUB - 1) {
          __syncwarp();
          if (pk < n) issue_one(slot);
        }
        const int j0 = c * VPC + h * 32 * SUB + lane;
        if (h == 0 && c == 0 && j0 < nvec && j0 != jrag) seed_ref<Tin>(ref, v[0], lamL);
        float bS, bW;
        if (bigneg) {
#pragma unroll
          for (int u = 0; u < SUB; ++u) {
            const int j = j0 + 32 * u;
            if (j == vy || j == jrag)              // one lane, one vector: patch in registers
              v[u] = Vec<Tin>::patch(v[u], j == vy ? yoff : -1, j == jrag ? keep_rag : EPV);
          }
          acc_batch<Tin, SUB, NPOLY>(v, lamL, -ref, bS, bW);
        } else if (special_batch<SUB>(j0, vy, jrag) || j0 + 32 * (SUB - 1) >= nvec) {
          batch_safe<Tin, SUB>(v, j0, nvec, vy, yoff, p.V, lamL, ref, bS, bW);
        } else {
          acc_batch<Tin, SUB, NPOLY>(v, lamL, -ref, bS, bW);
        }
        if (!(bS < 0x1p100f) || !(fabsf(bW) < 0x1p110f)) {
          S -= cS;
          W -= cW;
          cS = cW = 0.f;
          batch_slow<Tin, SUB>(v, j0, nvec, vy, yoff, jrag, p.V, lamL, ref, S, W, bS, bW, p.ws.err);
        }
        kahan_add(S, cS, bS);
        kahan_add(W, cW, bW);
      }
    }
    row_finish(ref, S - cS, W - cW, rec.uy, p.ws, p.row_begin + rec.r, lane, p.partial, rec.r,
               p.xbase, p.nx, p.xoff);
    if (dyn) {           // the producer already moved on to the next claimed row
      k = pk;
      rec_next = prec;
    } else {
      k += nw;
    }
  }
  // peer-memory exchange: lane 0 issued this warp's partial stores; one system-scope fence
  // orders them before k_tpx_signal's release of the ready flags
  if (p.nx > 0 && lane == 0) __threadfence_system();
}

// ---------------------------------------------------------------------------------------
// Variant TILE: a non-persistent grid of (listed row, tile) blocks — the K5 access pattern,
// which reaches the part's streaming ceiling. Block = 256 threads × VPT 16-byte vectors (32 KB
// of bf16 at VPT = 8), all loads in flight; each thread reduces its VPT vectors relative to
// the row's target logit (batch_slow for the target / ragged vector or an overflow), the
// block merges its threads (max reference, rebase, tree sums) and writes the tile's partial
// {R, S, W, u_y} to part[tile][row]; k_fwd_combine merges the tiles exactly like vocabulary
// shards.
// ---------------------------------------------------------------------------------------
template <typename Tin, int VPT, int MINB>
__global__ void __launch_bounds__(256, MINB) k_rowstats_tile(const FwdParams p, const FwdRec* list,
                                                       const int* count, int ntiles,
                                                       float4* part) {
  constexpr int EPV = Vec<Tin>::EPV;
  __shared__ float sh_r[8], sh_s[8], sh_w[8];
  const int i = blockIdx.x / ntiles;
  const int tile = blockIdx.x - i * ntiles;
  if (i >= *count) return;
  const FwdRec rec = list[i];
  const char* row = static_cast<const char*>(p.logits) + int64_t(rec.r) * p.ld * int64_t(sizeof(Tin));
  const int nvec = (p.V + EPV - 1) / EPV;
  const int jrag = (p.V % EPV) ? nvec - 1 : -1;
  const int vy = rec.yl >= 0 ? rec.yl / EPV : -1, yoff = rec.yl >= 0 ? rec.yl % EPV : 0;
  const float lamL = p.lam_log2e;
  const int j0 = tile * (256 * VPT) + threadIdx.x;
  const uint4 ninf = make_uint4(Vec<Tin>::kNegInfWord, Vec<Tin>::kNegInfWord, Vec<Tin>::kNegInfWord,
                                Vec<Tin>::kNegInfWord);
  uint4 v[VPT];
#pragma unroll
  for (int u = 0; u < VPT; ++u) {
    const int j = j0 + 256 * u;
    v[u] = (j < nvec) ? ld_stream(row + int64_t(j) * 16) : ninf;
  }
  float ref = rec.yl >= 0 ? rec.uy : -INFINITY, bS, bW;
  if (j0 < nvec && j0 != jrag) seed_ref<Tin>(ref, v[0], lamL);
  acc_batch<Tin, VPT, -1>(v, lamL, -ref, bS, bW);
  const unsigned dy = static_cast<unsigned>(vy - j0), dr = static_cast<unsigned>(jrag - j0);
  const bool special = (vy >= 0 && dy < 256u * VPT && (dy & 255u) == 0) ||
                       (jrag >= 0 && dr < 256u * VPT && (dr & 255u) == 0);
  if (special || !(bS < 0x1p100f) || !(fabsf(bW) < 0x1p110f)) {
    float S = 0.f, W = 0.f;
    batch_slow<Tin, VPT, 256>(v, j0, nvec, vy, yoff, jrag, p.V, lamL, ref, S, W, bS, bW, p.ws.err);
  }
  // block merge: max reference, rebase, fixed-order tree sums
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float R = warp_max(ref);
  if (lane == 0) sh_r[w] = R;
  __syncthreads();
  R = sh_r[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) R = fmaxf(R, sh_r[k]);
  if (R == -INFINITY) {
    bS = 0.f;
    bW = 0.f;
  } else {
    rebase(ref, R, bS, bW);
  }
  bS = warp_sum(bS);
  bW = warp_sum(bW);
  if (lane == 0) {
    sh_s[w] = bS;
    sh_w[w] = bW;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float S = 0.f, W = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      S += sh_s[k];
      W += sh_w[k];
    }
    part[int64_t(tile) * p.n_rows + rec.r] = make_float4(R, S, W, rec.uy);
  }
}

template <typename Tin, int NW, int STAGES, int CHUNK, int SUB, int NPOLY>
inline cudaError_t launch_rowstats_tma_cfg(const FwdParams& p, const FwdRec* list, const int* count,
                                           int num_sms, int blocks_per_sm, cudaStream_t s) {
  constexpr size_t smem = size_t(NW) * STAGES * CHUNK + size_t(NW) * STAGES * 8;
  auto k = k_rowstats_tma<Tin, NW, STAGES, CHUNK, SUB, NPOLY>;
  static unsigned long long attr_mask = 0;
  cudaError_t e = ensure_smem_attr(k, int(smem), attr_mask);
  if (e != cudaSuccess) return e;
  const int bps = blocks_per_sm > 0 ? blocks_per_sm : 1;
  k<<<num_sms * bps, NW * 32, smem, s>>>(p, list, count);
  return cudaGetLastError();
}

// variant → (warps, stages, chunk bytes, vectors per lane per sub-batch)
template <typename Tin>
inline cudaError_t launch_rowstats_tma(const FwdParams& p, const FwdRec* list, const int* count,
                                       int num_sms, int blocks_per_sm, int variant, cudaStream_t s) {
#define ESPO_FWD_CFG(NW, ST, CH, SB, NP) \
  launch_rowstats_tma_cfg<Tin, NW, ST, CH, SB, NP>(p, list, count, num_sms, blocks_per_sm, s)
  switch (variant) {
    case 2: return ESPO_FWD_CFG(16, 2, 7168, 2, -1);
    case 3: return ESPO_FWD_CFG(14, 2, 7168, 2, -1);
    case 4: return ESPO_FWD_CFG(20, 2, 5120, 2, -1);
    case 5: return ESPO_FWD_CFG(16, 3, 4096, 4, -1);   // the previous default (3 × 4 KB ring)
    case 6: return ESPO_FWD_CFG(16, 2, 6144, 4, 1);    // 1 element in 8 by polynomial exp2
    case 7: return ESPO_FWD_CFG(18, 2, 6144, 4, -1);
    case 8:    // the default geometries, scalar FP32
      if (int64_t(p.V) * int64_t(sizeof(Tin)) >= 65536) return ESPO_FWD_CFG(16, 2, 6144, 4, 0);
      return ESPO_FWD_CFG(16, 3, 4096, 4, 0);
    default:   // packed f32x2; ring geometry by row width (measured: C1 / C3 vs 1/8-vocab shards)
      if (int64_t(p.V) * int64_t(sizeof(Tin)) >= 65536) return ESPO_FWD_CFG(16, 2, 6144, 4, -1);
      return ESPO_FWD_CFG(16, 3, 4096, 4, -1);
  }
#undef ESPO_FWD_CFG
}

}  // namespace espo
