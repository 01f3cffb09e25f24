// k_rowlist.cuh — per-chunk row scheduling for the two vocab sweeps.
//
// Before each sweep a light kernel classifies the chunk's rows and appends the rows that
// need the sweep to a compact list of fixed-size records (warp-aggregated atomics; the
// order of the list does not matter because every row's result depends only on its own
// data). The hot kernels then read one record per row instead of a chain of dependent
// metadata loads, never touch rows that need no work, and balance over the rows that do.
#pragma once
#include "common.cuh"
#include "workspace.cuh"

namespace espo {

struct __align__(16) FwdRec {
  int32_t r;   // chunk-relative row
  int32_t y;   // sampled token
  float uy;    // λ·log2(e)·z_y (the sweep's initial reference); NaN if y is not in the shard
  int32_t yl;  // column of y in the local (vocabulary-shard) row, −1 if not in the shard
};

struct __align__(16) BwdRec {
  int32_t r;   // chunk-relative row
  int32_t y;   // ≥ 0: sweep the row; −1: zero-fill it; −2: leave it untouched
  float ng;    // −λ·g_t : dz_v = ng·p_v
  float nlseL; // −lse_t·log2(e)
  float gq;    // λ·g_t·q_t : dz_y
  int32_t yl;  // column of y in the local (vocabulary-shard) row, −1 if not in the shard
  float pad[2];
};

__device__ __forceinline__ int warp_append(bool take, int* count) {
  const unsigned m = __ballot_sync(0xffffffffu, take);
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == 0 && m) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  return base + __popc(m & ((1u << lane) - 1u));
}

// Forward: copies tokens/old_logp into the workspace, sets flag[t], lists valid rows of
// active rollouts (and, given zlist, the other rows at count[1]). Errors: token ∉ [0,V) and a non-finite target logit.
template <typename Tin>
__global__ void __launch_bounds__(256) k_fwd_rows(const void* logits, int64_t ld,
                                                  const int32_t* tokens, const float* old_logp,
                                                  const uint8_t* mask, int64_t row_begin,
                                                  int64_t n_rows, int V, int v0, int Vl,
                                                  float lamL, Workspace ws, FwdRec* list,
                                                  int* count, int32_t* zlist = nullptr) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t n_round = (n_rows + 31) / 32 * 32;  // whole warps stay converged
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_round; r += stride) {
    bool valid = false;
    int y = 0, yl = -1;
    float uy = 0.f;
    if (r < n_rows) {
      const int64_t t = row_begin + r;
      y = tokens[r];
      const bool m = mask ? (mask[r] != 0) : true;
      ws.old[t] = old_logp[r];
      ws.y[t] = y;
      valid = m && ws.cand[ws.row_seq[t]];
      if (valid && (y < 0 || y >= V)) {
        set_error(ws.err, ESPO_ERR_TOKEN_OUT_OF_RANGE);
        valid = false;
      }
      if (valid) {
        yl = (y >= v0 && y < v0 + Vl) ? y - v0 : -1;   // target in this vocabulary shard?
        if (yl >= 0) {
          const char* row = static_cast<const char*>(logits) + r * ld * int64_t(sizeof(Tin));
          uy = Vec<Tin>::load1(row, yl) * lamL;
          if (!(fabsf(uy) <= 3.0e38f)) {
            set_error(ws.err, ESPO_ERR_NONFINITE_INPUT);
            valid = false;
          }
        } else {
          uy = __int_as_float(0x7fc00000);
        }
      }
      ws.flag[t] = valid ? 1 : 0;
    }
    if (zlist) {   // factored-gradient sweep: rows without gradient are zero-filled
      const bool zero = r < n_rows && !valid;
      const int pz = warp_append(zero, count + 1);
      if (zero) zlist[pz] = static_cast<int32_t>(r);
    }
    const int pos = warp_append(valid, count);
    if (valid) {
      FwdRec rec;
      rec.r = static_cast<int32_t>(r);
      rec.y = y;
      rec.uy = uy;
      rec.yl = yl;
      list[pos] = rec;
    }
  }
}

// Backward: rows with a nonzero coefficient get a sweep record; rows without gradient
// (masked, eliminated group, inactive rollout, clipped token) go to the zero-fill list when
// zero_fill is set and are left untouched otherwise. count[0] = sweeps, count[1] = zeros.
__global__ void __launch_bounds__(256) k_bwd_rows(int64_t row_begin, int64_t n_rows,
                                                  const float* grad_loss, int zero_fill, int v0,
                                                  int Vl, Workspace ws, BwdRec* list,
                                                  int32_t* zlist, int* count) {
  const float gl = grad_loss ? *grad_loss : 1.f;
  const float gscale = -gl * *ws.bwd_scale;  // λ·g_t = gscale·c_t
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t n_round = (n_rows + 31) / 32 * 32;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_round; r += stride) {
    bool sweep = false, zero = false;
    BwdRec rec;
    if (r < n_rows) {
      const int64_t t = row_begin + r;
      const float c = ws.flag[t] ? ws.coef[t] : 0.f;
      const float g = gscale * c;
      if (g != 0.f) {
        sweep = true;
        rec.r = static_cast<int32_t>(r);
        rec.y = ws.y[t];
        rec.ng = -g;
        rec.nlseL = -ws.lse[t] * kLog2e;
        rec.gq = g * ws.q[t];
        rec.yl = (rec.y >= v0 && rec.y < v0 + Vl) ? rec.y - v0 : -1;
        rec.pad[0] = rec.pad[1] = 0.f;
      } else {
        zero = zero_fill != 0;
      }
    }
    const int ps = warp_append(sweep, count);
    if (sweep) list[ps] = rec;
    const int pz = warp_append(zero, count + 1);
    if (zero) zlist[pz] = static_cast<int32_t>(r);
  }
}

// Backward, tiled variant: one record per chunk row, indexed by the row (no compaction):
// y ≥ 0 sweep, y = −1 zero-fill, y = −2 leave untouched (no gradient and zero_fill == 0).
__global__ void __launch_bounds__(256) k_bwd_recs(int64_t row_begin, int64_t n_rows,
                                                  const float* grad_loss, int zero_fill, int v0,
                                                  int Vl, Workspace ws, BwdRec* rec) {
  const float gl = grad_loss ? *grad_loss : 1.f;
  const float gscale = -gl * *ws.bwd_scale;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = row_begin + r;
    const float c = ws.flag[t] ? ws.coef[t] : 0.f;
    const float g = gscale * c;
    BwdRec o;
    o.r = static_cast<int32_t>(r);
    o.pad[0] = o.pad[1] = 0.f;
    o.yl = -1;
    if (g != 0.f) {
      o.y = ws.y[t];
      o.ng = -g;
      o.nlseL = -ws.lse[t] * kLog2e;
      o.gq = g * ws.q[t];
      o.yl = (o.y >= v0 && o.y < v0 + Vl) ? o.y - v0 : -1;
    } else {
      o.y = zero_fill ? -1 : -2;
      o.ng = o.nlseL = o.gq = 0.f;
    }
    rec[r] = o;
  }
}

}  // namespace espo
