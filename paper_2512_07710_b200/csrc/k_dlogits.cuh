// k_dlogits.cuh — K5: the backward vocab sweep.
//
// d loss/d z_{t,v} = λ·g_t·(1[v = y_t] − p_v) with g_t = −grad_loss·c_t/D: only the Eq. 1
// numerator log π_θ(y_t) carries gradient (stop-gradient). The target
// entry is written as λ·g_t·q_t (q = 1 − p_y from K2, no cancellation). Rows that carry
// no gradient (masked, eliminated group, inactive rollout, clipped token) are zero-filled
// without reading the logits.
#pragma once
#include "common.cuh"
#include "workspace.cuh"
#include "k_rowlist.cuh"

namespace espo {

struct BwdParams {
  const void* logits;
  int64_t ld;
  void* dlogits;
  int64_t ldg;
  const float* grad_loss;  // nullable = 1
  int64_t row_begin, n_rows;
  int V;
  float lam_log2e;
  int zero_fill;
  int aliased;             // dlogits == logits (in place)
  Workspace ws;
};

// Writes the EPV_in outputs of one input vector j (handles the f32-out-of-bf16 split and
// the ragged last vector).
template <typename Tin, typename Tout>
__device__ __forceinline__ void store_out(char* orow, int j, const float* d, int V) {
  constexpr int EPI = Vec<Tin>::EPV;
  constexpr int EPO = Out<Tout>::EPV;
  if ((j + 1) * EPI <= V) {
    if constexpr (EPI < EPO) {   // f32 in → bf16 out: 4 values → one 8-byte store
      st_stream2(orow + int64_t(j) * EPI * sizeof(Tout), pack_bf16x2(d[0], d[1]),
                 pack_bf16x2(d[2], d[3]));
    } else {
#pragma unroll
      for (int h = 0; h < EPI / EPO; ++h)
        st_stream(orow + (int64_t(j) * EPI + h * EPO) * sizeof(Tout), Out<Tout>::pack(d + h * EPO));
    }
  } else {
#pragma unroll
    for (int e = 0; e < EPI; ++e) {
      const int c = j * EPI + e;
      if (c < V) {
        if (sizeof(Tout) == 4) reinterpret_cast<float*>(orow)[c] = d[e];
        else reinterpret_cast<__nv_bfloat16*>(orow)[c] = __float2bfloat16_rn(d[e]);
      }
    }
  }
}

template <typename Tout>
__device__ __forceinline__ void zero_row(char* orow, int V, int lane) {
  constexpr int EPO = Out<Tout>::EPV;
  const int nfull = V / EPO;
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int j = lane; j < nfull; j += 32) st_stream(orow + int64_t(j) * 16, z);
  for (int c = nfull * EPO + lane; c < V; c += 32) {
    if (sizeof(Tout) == 4) reinterpret_cast<float*>(orow)[c] = 0.f;
    else reinterpret_cast<uint16_t*>(orow)[c] = 0;
  }
}

// Computes the EPV outputs of one input vector j of a swept row.
// P2: the FFMA and FMUL of element pairs issued as sm_100 packed f32x2 (bitwise the same).
template <typename Tin, bool P2 = true>
__device__ __forceinline__ void dz_vec(const uint4& v, int j, int vy, int yoff, float lamL,
                                       const BwdRec& rec, float* d) {
  constexpr int EPV = Vec<Tin>::EPV;
  float x[EPV];
  Vec<Tin>::unpack(v, x);
  if constexpr (P2) {
    const float2 L2 = make_float2(lamL, lamL), N2 = make_float2(rec.nlseL, rec.nlseL);
    const float2 G2 = make_float2(rec.ng, rec.ng);
#pragma unroll
    for (int e = 0; e < EPV; e += 2) {
      const float2 t = __ffma2_rn(make_float2(x[e], x[e + 1]), L2, N2);
      const float2 o = __fmul2_rn(G2, make_float2(ex2(t.x), ex2(t.y)));
      d[e] = o.x;
      d[e + 1] = o.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < EPV; ++e) d[e] = rec.ng * ex2(fmaf(x[e], lamL, rec.nlseL));
  }
  if (j == vy) {
#pragma unroll
    for (int e = 0; e < EPV; ++e)
      if (e == yoff) d[e] = rec.gq;
  }
}

// zero-fill records: processed by the same warps after their sweep rows
template <typename Tout>
__device__ __forceinline__ void zero_rows(const BwdParams& p, const int32_t* zlist, int nz, int gw,
                                          int nw, int lane) {
  for (int k = gw; k < nz; k += nw) {
    char* orow = static_cast<char*>(p.dlogits) + int64_t(zlist[k]) * p.ldg * int64_t(sizeof(Tout));
    zero_row<Tout>(orow, p.V, lane);
  }
}

template <typename Tin, typename Tout, int U>
__global__ void __launch_bounds__(256) k_dlogits_ldg(const BwdParams p, const BwdRec* list,
                                                     const int32_t* zlist, const int* count) {
  constexpr int EPV = Vec<Tin>::EPV;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int n = count[0], nz = count[1];
  const int nvec = (p.V + EPV - 1) / EPV;
  const float lamL = p.lam_log2e;
  for (int k = gw; k < n; k += nw) {
    const BwdRec rec = list[k];
    const char* row = static_cast<const char*>(p.logits) + int64_t(rec.r) * p.ld * int64_t(sizeof(Tin));
    char* orow = static_cast<char*>(p.dlogits) + int64_t(rec.r) * p.ldg * int64_t(sizeof(Tout));
    const int vy = rec.yl >= 0 ? rec.yl / EPV : -1, yoff = rec.yl >= 0 ? rec.yl % EPV : 0;
    for (int j0 = lane; j0 < nvec; j0 += 32 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + 32 * u;
        if (j < nvec)
          v[u] = p.aliased ? ld_stream_coherent(row + int64_t(j) * 16) : ld_stream(row + int64_t(j) * 16);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + 32 * u;
        if (j < nvec) {
          float d[EPV];
          dz_vec<Tin>(v[u], j, vy, yoff, lamL, rec, d);
          store_out<Tin, Tout>(orow, j, d, p.V);
        }
      }
    }
  }
  zero_rows<Tout>(p, zlist, nz, gw, nw, lane);
}

// TMA variant: the same per-warp bulk-copy ring as k_rowstats_tma for the logits; the
// gradient is written from registers with 128-bit streaming stores (st.global.cs).
// In place is safe: a chunk is in registers before its own addresses are written, and
// the ring only runs ahead (to addresses not yet written).
template <typename Tin, typename Tout, int NW, int STAGES, int CHUNK>
__global__ void __launch_bounds__(NW * 32, 1) k_dlogits_tma(const BwdParams p, const BwdRec* list,
                                                            const int32_t* zlist, const int* count) {
  constexpr int EPV = Vec<Tin>::EPV;
  constexpr int VPC = CHUNK / 16;
  constexpr int VPL = VPC / 32;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + size_t(warp) * STAGES * CHUNK;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(NW) * STAGES * CHUNK) + warp * STAGES;
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int n = count[0], nz = count[1];
  const int nw = gridDim.x * NW;
  const int gw = blockIdx.x * NW + warp;
  const int nvec = (p.V + EPV - 1) / EPV;
  const uint32_t rowbytes = uint32_t(nvec) * 16u;
  const int nch = static_cast<int>((rowbytes + CHUNK - 1) / CHUNK);
  const float lamL = p.lam_log2e;
  const int64_t pitch = p.ld * int64_t(sizeof(Tin));
  const char* base = static_cast<const char*>(p.logits);
  const uint64_t pol = policy_evict_first();

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
  BwdRec rec_next = (gw < n) ? list[gw] : BwdRec{};
  for (int k = gw; k < n; k += nw) {
    const BwdRec rec = rec_next;
    if (k + nw < n) rec_next = list[k + nw];
    char* orow = static_cast<char*>(p.dlogits) + int64_t(rec.r) * p.ldg * int64_t(sizeof(Tout));
    const int vy = rec.yl >= 0 ? rec.yl / EPV : -1, yoff = rec.yl >= 0 ? rec.yl % EPV : 0;
    for (int c = 0; c < nch; ++c) {
      const int slot = consumed % STAGES;
      mbar_wait(&bars[slot], (consumed / STAGES) & 1u);
      const uint8_t* buf = ring + slot * CHUNK;
      const int vlim = min(VPC, nvec - c * VPC);
      uint4 v[VPL];
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        const int jl = lane + 32 * u;
        if (jl < vlim) v[u] = lds128(buf + jl * 16);
      }
      __syncwarp();
      ++consumed;
      refill();
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        const int jl = lane + 32 * u;
        if (jl < vlim) {
          const int j = c * VPC + jl;
          float d[EPV];
          dz_vec<Tin>(v[u], j, vy, yoff, lamL, rec, d);
          store_out<Tin, Tout>(orow, j, d, p.V);
        }
      }
    }
  }
  zero_rows<Tout>(p, zlist, nz, gw, nw, lane);
}

// Tiled variant: a non-persistent grid of (row, tile) blocks in row-major order, 256 threads,
// VPT 16-byte input vectors per thread (16 KB bf16 tile): every block reads its tile with all
// loads in flight, computes and writes it back — the access pattern of the fastest copy
// measured on this part (tools/bwprobe.cu: 6.9 TB/s vs 6.3 for per-warp rings), and a
// zero-fill tile is a pure write.
// Tiled variant over the compact row lists of k_bwd_rows: block b handles tile b % ntiles of
// list entries [RPB·(b / ntiles), +RPB) — sweep rows first, then zero-fill rows. Blocks past
// the lists' end exit at once; with RPB rows per block there are RPB× fewer of them than in
// the per-row grid (compact mode, where most rows have no gradient and are not written).
template <typename Tin, typename Tout, int VPT, int RPB>
__global__ void __launch_bounds__(256) k_dlogits_tlist(const BwdParams p, const BwdRec* list,
                                                       const int32_t* zlist, const int* count,
                                                       int ntiles) {
  constexpr int EPV = Vec<Tin>::EPV;
  const int g = blockIdx.x / ntiles;
  const int tile = blockIdx.x - g * ntiles;
  const int n_sweep = count[0], n_all = n_sweep + count[1];
  const int nvec = (p.V + EPV - 1) / EPV;
  const int j0 = tile * (256 * VPT) + threadIdx.x;
  const float lamL = p.lam_log2e;
  for (int k = 0; k < RPB; ++k) {
    const int idx = g * RPB + k;
    if (idx >= n_all) return;
    if (idx >= n_sweep) {   // zero-fill row: write only
      char* orow = static_cast<char*>(p.dlogits) + int64_t(zlist[idx - n_sweep]) * p.ldg * int64_t(sizeof(Tout));
      float z[EPV];
#pragma unroll
      for (int e = 0; e < EPV; ++e) z[e] = 0.f;
#pragma unroll
      for (int u = 0; u < VPT; ++u) {
        const int j = j0 + 256 * u;
        if (j < nvec) store_out<Tin, Tout>(orow, j, z, p.V);
      }
      continue;
    }
    const BwdRec rc = list[idx];
    const char* row = static_cast<const char*>(p.logits) + int64_t(rc.r) * p.ld * int64_t(sizeof(Tin));
    char* orow = static_cast<char*>(p.dlogits) + int64_t(rc.r) * p.ldg * int64_t(sizeof(Tout));
    const int vy = rc.yl >= 0 ? rc.yl / EPV : -1, yoff = rc.yl >= 0 ? rc.yl % EPV : 0;
    uint4 v[VPT];
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int j = j0 + 256 * u;
      if (j < nvec)
        v[u] = p.aliased ? ld_stream_coherent(row + int64_t(j) * 16) : ld_stream(row + int64_t(j) * 16);
    }
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int j = j0 + 256 * u;
      if (j < nvec) {
        float dd[EPV];
        dz_vec<Tin>(v[u], j, vy, yoff, lamL, rc, dd);
        store_out<Tin, Tout>(orow, j, dd, p.V);
      }
    }
  }
}

template <typename Tin, typename Tout, int VPT, bool P2 = true>
__global__ void __launch_bounds__(256) k_dlogits_tile(const BwdParams p, const BwdRec* rec,
                                                      int ntiles) {
  constexpr int EPV = Vec<Tin>::EPV;
  const int r = blockIdx.x / ntiles;
  const int tile = blockIdx.x - r * ntiles;
  const BwdRec rc = rec[r];
  if (rc.y == -2) return;
  const int nvec = (p.V + EPV - 1) / EPV;
  const int j0 = tile * (256 * VPT) + threadIdx.x;
  char* orow = static_cast<char*>(p.dlogits) + int64_t(rc.r) * p.ldg * int64_t(sizeof(Tout));
  if (rc.y < 0) {
    float z[EPV];
#pragma unroll
    for (int e = 0; e < EPV; ++e) z[e] = 0.f;
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int j = j0 + 256 * u;
      if (j < nvec) store_out<Tin, Tout>(orow, j, z, p.V);
    }
    return;
  }
  const char* row = static_cast<const char*>(p.logits) + int64_t(rc.r) * p.ld * int64_t(sizeof(Tin));
  const float lamL = p.lam_log2e;
  const int vy = rc.yl >= 0 ? rc.yl / EPV : -1, yoff = rc.yl >= 0 ? rc.yl % EPV : 0;
  uint4 v[VPT];
#pragma unroll
  for (int u = 0; u < VPT; ++u) {
    const int j = j0 + 256 * u;
    if (j < nvec)
      v[u] = p.aliased ? ld_stream_coherent(row + int64_t(j) * 16) : ld_stream(row + int64_t(j) * 16);
  }
#pragma unroll
  for (int u = 0; u < VPT; ++u) {
    const int j = j0 + 256 * u;
    if (j < nvec) {
      float dd[EPV];
      dz_vec<Tin, P2>(v[u], j, vy, yoff, lamL, rc, dd);
      store_out<Tin, Tout>(orow, j, dd, p.V);
    }
  }
}

template <typename Tin, typename Tout, int NW, int STAGES, int CHUNK>
inline cudaError_t launch_dlogits_tma_cfg(const BwdParams& p, const BwdRec* list,
                                          const int32_t* zlist, const int* count, int num_sms,
                                          int blocks_per_sm, cudaStream_t s) {
  constexpr size_t smem = size_t(NW) * STAGES * CHUNK + size_t(NW) * STAGES * 8;
  auto k = k_dlogits_tma<Tin, Tout, NW, STAGES, CHUNK>;
  static unsigned long long attr_mask = 0;
  cudaError_t e = ensure_smem_attr(k, int(smem), attr_mask);
  if (e != cudaSuccess) return e;
  const int bps = blocks_per_sm > 0 ? blocks_per_sm : 1;
  k<<<num_sms * bps, NW * 32, smem, s>>>(p, list, zlist, count);
  return cudaGetLastError();
}

// variant → (warps, stages, chunk bytes)
template <typename Tin, typename Tout>
inline cudaError_t launch_dlogits_tma(const BwdParams& p, const BwdRec* list, const int32_t* zlist,
                                      const int* count, int num_sms, int blocks_per_sm, int variant,
                                      cudaStream_t s) {
#define ESPO_BWD_CFG(NW, ST, CH) \
  launch_dlogits_tma_cfg<Tin, Tout, NW, ST, CH>(p, list, zlist, count, num_sms, blocks_per_sm, s)
  switch (variant) {
    case 2: return ESPO_BWD_CFG(16, 3, 4096);
    case 3: return ESPO_BWD_CFG(16, 2, 4096);
    case 4: return ESPO_BWD_CFG(12, 4, 4096);
    case 5: return ESPO_BWD_CFG(8, 6, 4096);
    default: return ESPO_BWD_CFG(8, 4, 4096);
  }
#undef ESPO_BWD_CFG
}

}  // namespace espo
