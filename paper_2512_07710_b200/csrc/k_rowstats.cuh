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
  int V;
  float lam_log2e;      // λ·log2(e)
  Workspace ws;
};

__device__ __forceinline__ float max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// Accumulates EPV elements (already unpacked) into (s, w) relative to reference nref = −r.
template <int EPV>
__device__ __forceinline__ void acc_vec(const float* x, float lamL, float nref, float& s,
                                        float& w) {
  float s0 = 0.f, s1 = 0.f, w0 = 0.f, w1 = 0.f;
#pragma unroll
  for (int e = 0; e < EPV; e += 2) {
    const float t0 = max_nan(fmaf(x[e], lamL, nref), -127.f);
    const float t1 = max_nan(fmaf(x[e + 1], lamL, nref), -127.f);
    const float e0 = ex2(t0), e1 = ex2(t1);
    s0 += e0;
    s1 += e1;
    w0 = fmaf(e0, t0, w0);
    w1 = fmaf(e1, t1, w1);
  }
  s += s0 + s1;
  w += w0 + w1;
}

// Sets the target element and the elements past V of a vector to −inf (they contribute 0).
template <int EPV>
__device__ __forceinline__ void fix_special(float* x, int j, int vy, int yoff, int V) {
  if (j == vy) x[yoff] = -INFINITY;
#pragma unroll
  for (int e = 0; e < EPV; ++e)
    if (j * EPV + e >= V) x[e] = -INFINITY;
}

// Row epilogue: combine lanes (each lane may hold its own reference r), write lse/lp/H/q.
__device__ __forceinline__ void row_finish(float r, float S, float W, float uy, const Workspace& ws,
                                           int64_t t, int lane) {
  const float R = warp_max(r);
  const float d = r - R;
  const float sc = ex2(d);
  W = sc * fmaf(d, S, W);
  S = sc * S;
  S = warp_sum(S);
  W = warp_sum(W);
  if (lane == 0) {
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

// Slow path for one batch: NaN/+inf detection and a max-based reference.
template <int EPV, int U>
__device__ __noinline__ void batch_slow(const uint4* v, int j0, int nvec, int vy, int yoff, int V,
                                        float lamL, float& r, float& S, float& W, float& bS,
                                        float& bW, int* err, bool is_bf16) {
  float bm = -INFINITY;
  bool bad = false;
  float xs[U][EPV];
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const int j = j0 + 32 * k;
    if (is_bf16) Vec<__nv_bfloat16>::unpack(v[k], xs[k]);
    else Vec<float>::unpack(v[k], xs[k]);
    if (j >= nvec) {
#pragma unroll
      for (int e = 0; e < EPV; ++e) xs[k][e] = -INFINITY;
    } else {
      fix_special<EPV>(xs[k], j, vy, yoff, V);
    }
#pragma unroll
    for (int e = 0; e < EPV; ++e) {
      const float u = xs[k][e] * lamL;
      if (isnan(u) || u == INFINITY) bad = true;
      bm = fmaxf(bm, u);
    }
  }
  if (bad) {
    set_error(err, ESPO_ERR_NONFINITE_INPUT);
    bS = __int_as_float(0x7fc00000);
    bW = bS;
    return;
  }
  if (bm > r) {
    const float d = r - bm;
    const float sc = ex2(d);
    W = sc * fmaf(d, S, W);
    S = sc * S;
    r = bm;
  }
  bS = 0.f;
  bW = 0.f;
#pragma unroll
  for (int k = 0; k < U; ++k) acc_vec<EPV>(xs[k], lamL, -r, bS, bW);
}


// Processes U vectors (global vector index j0 + 32k) into the batch sums (bS, bW).
template <typename Tin, int U>
__device__ __forceinline__ void acc_batch(const uint4* v, int j0, int vy, int yoff, int jrag, int V,
                                          float lamL, float nref, float& bS, float& bW) {
  constexpr int EPV = Vec<Tin>::EPV;
#pragma unroll
  for (int k = 0; k < U; ++k) {
    float x[EPV];
    Vec<Tin>::unpack(v[k], x);
    const int j = j0 + 32 * k;
    if (j == vy || j == jrag) fix_special<EPV>(x, j, vy, yoff, V);
    acc_vec<EPV>(x, lamL, nref, bS, bW);
  }
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
    const int vy = rec.y / EPV, yoff = rec.y % EPV;
    float ref = rec.uy, S = 0.f, W = 0.f;
    for (int j0 = lane; j0 < nvec; j0 += 32 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + 32 * u;
        v[u] = (j < nvec) ? ld_stream(row + int64_t(j) * 16) : ninf;
      }
      float bS = 0.f, bW = 0.f;
      acc_batch<Tin, U>(v, j0, vy, yoff, jrag, p.V, lamL, -ref, bS, bW);
      if (!(bS < 0x1p100f) || !(fabsf(bW) < 0x1p110f))
        batch_slow<EPV, U>(v, j0, nvec, vy, yoff, p.V, lamL, ref, S, W, bS, bW, p.ws.err,
                           sizeof(Tin) == 2);
      S += bS;
      W += bW;
    }
    row_finish(ref, S, W, rec.uy, p.ws, p.row_begin + rec.r, lane);
  }
}

// ---------------------------------------------------------------------------------------
// Variant TMA: warp per row; each warp owns a STAGES-deep ring of CHUNK-byte shared-memory
// slots filled by cp.async.bulk (the TMA engine, completion on one mbarrier per slot).
// Lane 0 keeps STAGES chunks in flight across row boundaries; all lanes consume a slot
// with conflict-free 128-bit LDS, then release it (__syncwarp) for the next copy.
// ---------------------------------------------------------------------------------------
template <typename Tin, int NW, int STAGES, int CHUNK>
__global__ void __launch_bounds__(NW * 32, 1) k_rowstats_tma(const FwdParams p,
                                                             const FwdRec* list, const int* count) {
  constexpr int EPV = Vec<Tin>::EPV;
  constexpr int VPC = CHUNK / 16;  // vectors per chunk
  constexpr int VPL = VPC / 32;    // vectors per lane per chunk
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

  // producer cursor (row records prefetched one row ahead)
  int pk = gw, pc = 0;
  int pr = (pk < n) ? list[pk].r : 0;
  int pr_next = (pk + nw < n) ? list[pk + nw].r : 0;
  uint32_t issued = 0, consumed = 0;
  auto refill = [&]() {
    while (issued - consumed < STAGES && pk < n) {
      const int slot = issued % STAGES;
      const uint32_t off = uint32_t(pc) * CHUNK;
      const uint32_t bytes = min(uint32_t(CHUNK), rowbytes - off);
      if (lane == 0) {
        mbar_arrive_tx(&bars[slot], bytes);
        bulk_g2s(ring + slot * CHUNK, base + int64_t(pr) * pitch + off, bytes, &bars[slot], pol);
      }
      ++issued;
      if (++pc == nch) {
        pc = 0;
        pk += nw;
        pr = pr_next;
        pr_next = (pk + nw < n) ? list[pk + nw].r : 0;
      }
    }
  };
  refill();
  FwdRec rec_next = (gw < n) ? list[gw] : FwdRec{};
  for (int k = gw; k < n; k += nw) {
    const FwdRec rec = rec_next;
    if (k + nw < n) rec_next = list[k + nw];
    const int vy = rec.y / EPV, yoff = rec.y % EPV;
    float ref = rec.uy, S = 0.f, W = 0.f;
    for (int c = 0; c < nch; ++c) {
      const int slot = consumed % STAGES;
      mbar_wait(&bars[slot], (consumed / STAGES) & 1u);
      const uint8_t* buf = ring + slot * CHUNK;
      const int vlim = min(VPC, nvec - c * VPC);
      uint4 v[VPL];
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        const int jl = lane + 32 * u;
        v[u] = (jl < vlim) ? lds128(buf + jl * 16) : ninf;
      }
      __syncwarp();
      ++consumed;
      refill();  // the slot's data is in registers: reuse it right away
      const int j0 = c * VPC + lane;
      float bS = 0.f, bW = 0.f;
      acc_batch<Tin, VPL>(v, j0, vy, yoff, jrag, p.V, lamL, -ref, bS, bW);
      if (!(bS < 0x1p100f) || !(fabsf(bW) < 0x1p110f))
        batch_slow<EPV, VPL>(v, j0, nvec, vy, yoff, p.V, lamL, ref, S, W, bS, bW, p.ws.err,
                             sizeof(Tin) == 2);
      S += bS;
      W += bW;
    }
    row_finish(ref, S, W, rec.uy, p.ws, p.row_begin + rec.r, lane);
  }
}

template <typename Tin>
struct RowstatsTmaCfg {
  static constexpr int NW = 8, STAGES = 4, CHUNK = 4096;
  static constexpr size_t smem() { return size_t(NW) * STAGES * CHUNK + size_t(NW) * STAGES * 8; }
};

template <typename Tin>
inline cudaError_t launch_rowstats_tma(const FwdParams& p, const FwdRec* list, const int* count,
                                       int num_sms, int blocks_per_sm, cudaStream_t s) {
  using C = RowstatsTmaCfg<Tin>;
  auto k = k_rowstats_tma<Tin, C::NW, C::STAGES, C::CHUNK>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::smem()));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int bps = blocks_per_sm > 0 ? blocks_per_sm : 1;
  k<<<num_sms * bps, C::NW * 32, C::smem(), s>>>(p, list, count);
  return cudaGetLastError();
}

}  // namespace espo
