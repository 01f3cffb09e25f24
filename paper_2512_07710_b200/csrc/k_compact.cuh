// k_compact.cuh — row compaction for the fused LM-head backward.
//
// A row whose coefficient c_t is 0 (clipped token, masked token, eliminated group, inactive
// rollout) has dz_t = 0 (only the Eq. 1 numerator carries gradient, and the
// clipped branch of the min has slope 0), so it contributes nothing to dh_t = dz_t·W (dh_t = 0)
// nor to dW = dzᵀ·h. The backward therefore recomputes logits, forms dz and runs both GEMMs
// only over the rows with gradient, gathered into a dense block: K5's "rows without gradient
// are not read" applied to the LM head. Order is stable (increasing row), so dh is bitwise the
// uncompacted result; dW sums the same non-zero products (fp32 accumulation order may differ).
//
//   k_cmp_count   one CTA per 1024 rows: rows with gradient per block
//   k_cmp_scatter prefix over the block counts, stable in-block scan → list[], total
//   k_cmp_gather  sub-chunk j: h rows list[base + i] → hc (bf16), records → rec_c; the tail up
//                 to a multiple of 256 rows is zero (rows and records), so tiles read zeros
//   k_zero_rows   rows without gradient of dhidden are written as zeros
#pragma once
#include "common.cuh"
#include "k_rowlist.cuh"

namespace espo {

constexpr int kCmpBlock = 1024;

__global__ void __launch_bounds__(kCmpBlock) k_cmp_count(const BwdRec* rec, int n, int* counts) {
  const int r = blockIdx.x * kCmpBlock + threadIdx.x;
  const int f = (r < n && rec[r].ng != 0.f) ? 1 : 0;
  const int c = __syncthreads_count(f);
  if (threadIdx.x == 0) counts[blockIdx.x] = c;
}

__global__ void __launch_bounds__(kCmpBlock) k_cmp_scatter(const BwdRec* rec, int n,
                                                          const int* counts, int nblocks,
                                                          int* list, int* total) {
  __shared__ int warp_off[kCmpBlock / 32];
  __shared__ int base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    int s = 0;
    for (int b = 0; b < int(blockIdx.x); ++b) s += counts[b];
    base = s;
    if (int(blockIdx.x) == nblocks - 1) *total = s + counts[blockIdx.x];
  }
  const int r = blockIdx.x * kCmpBlock + threadIdx.x;
  const bool f = r < n && rec[r].ng != 0.f;
  const unsigned m = __ballot_sync(0xffffffffu, f);
  if (lane == 0) warp_off[warp] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < kCmpBlock / 32; ++w) {
      const int c = warp_off[w];
      warp_off[w] = s;
      s += c;
    }
  }
  __syncthreads();
  if (f) list[base + warp_off[warp] + __popc(m & ((1u << lane) - 1u))] = r;
}

// rows i ∈ [0, cap) of sub-chunk `base`: count_i = clamp(total − base, 0, cap); rows
// i < count get h[list[base + i]] and its record, rows count ≤ i < round_up(count, 256) zeros
__global__ void __launch_bounds__(256) k_cmp_gather(const __nv_bfloat16* h, int64_t ldh, int d,
                                                    const BwdRec* rec, const int* list,
                                                    const int* total, int base, int cap,
                                                    __nv_bfloat16* hc, int64_t ldc, BwdRec* rec_c) {
  const int i = blockIdx.x;
  const int cnt = min(cap, max(0, *total - base));
  const int pad = min(cap, (cnt + 255) / 256 * 256);
  if (i >= pad) return;
  uint4* dst = reinterpret_cast<uint4*>(hc + int64_t(i) * ldc);
  const int nv = d / 8;                        // d % 8 == 0 (16-byte rows) checked on the host
  if (i < cnt) {
    const int src = list[base + i];
    const uint4* s = reinterpret_cast<const uint4*>(h + int64_t(src) * ldh);
    for (int v = threadIdx.x; v < nv; v += blockDim.x) dst[v] = s[v];
    if (threadIdx.x == 0) {
      BwdRec o = rec[src];
      o.r = i;
      rec_c[i] = o;
    }
  } else {
    for (int v = threadIdx.x; v < nv; v += blockDim.x) dst[v] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
      BwdRec o{};
      o.r = i;
      o.y = -1;
      rec_c[i] = o;
    }
  }
}

// dhidden rows without gradient (rec.ng == 0) → zeros (f32 or bf16 rows of d elements)
__global__ void __launch_bounds__(256) k_zero_rows(const BwdRec* rec, int n, void* out,
                                                   int64_t ld_bytes, int row_bytes) {
  const int r = blockIdx.x;
  if (r >= n || rec[r].ng != 0.f) return;
  uint8_t* row = static_cast<uint8_t*>(out) + int64_t(r) * ld_bytes;
  for (int b = threadIdx.x * 16; b < row_bytes; b += blockDim.x * 16)
    *reinterpret_cast<uint4*>(row + b) = make_uint4(0, 0, 0, 0);
}

}  // namespace espo

namespace espo {
// per block of `rows_per_block` chunk rows: 1 if any row is valid (flag) — the LM-head forward
// on the GEMM core skips M-tiles without a row to compute (eliminated groups, masked tails)
__global__ void __launch_bounds__(256) k_block_live(const uint8_t* flag, int n_rows,
                                                    int rows_per_block, uint8_t* live) {
  const int b = blockIdx.x;
  int any = 0;
  for (int r = b * rows_per_block + threadIdx.x; r < min(n_rows, (b + 1) * rows_per_block);
       r += blockDim.x)
    any |= flag[r];
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) live[b] = any ? 1 : 0;
}
}  // namespace espo
