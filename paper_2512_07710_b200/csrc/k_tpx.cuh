// k_tpx.cuh — vocabulary-parallel ESPO with the partial exchange fused into the forward sweep
// over peer memory (the Megatron vocab-parallel layout of PAPER.md:129).
//
// Every TP rank owns an exchange buffer (cudaMalloc, shared with the other ranks through CUDA
// IPC handles; NVLink/NVSwitch peer mappings):
//   flags: ready[2][tp_world] u32 (epoch at which rank k's partials of slot s are complete),
//          consumed[tp_world] u32 (last epoch rank k finished combining)
//   gath : [2 slots][tp_world][cap_rows] float4 partials {R, S, W, u_y}
// Chunk e (epoch e ≥ 1, slot e & 1) on rank j:
//   send: k_tpx_wait_consumed — slot e & 1 was read by every rank's combine of epoch e − 2;
//         K2 sweep whose row_finish stores each row's partial into gath[slot][j][r] of EVERY
//         rank (the all-gather is the sweep's own epilogue stores, no separate collective);
//         k_tpx_signal — system-scope release of ready[slot][j] = e on every rank.
//   recv: k_tpx_combine — acquire-wait until ready[slot][k] == e for all k, then the exact
//         merge of k_fwd_combine from the local buffer; k_tpx_post — consumed[j] = e on every
//         rank (the slot may be rewritten at epoch e + 2).
// Waits are bounded in wall time (ESPO_OPT_PEER_TIMEOUT_MS, default 120 s): a peer that never
// arrives sets ESPO_ERR_PEER_TIMEOUT instead of hanging the GPU; the step is then invalid
// (k_tpx_combine leaves the chunk's row statistics unwritten).
#pragma once
#include "common.cuh"
#include "k_rowstats.cuh"
#include "workspace.cuh"

namespace espo {

constexpr int kTpxFlagBytes = 4096;        // flags region at the start of an exchange buffer
constexpr int kTpxConsumedOff = 2048;      // byte offset of consumed[] inside it

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Bounded spin: true when pred() held; false once timeout_ns of wall time (the device's
// global timer) passed without it. The bound is ESPO_OPT_PEER_TIMEOUT_MS (default 120 s):
// generous enough for normal rank skew (host-side data work, GC), finite so a dead peer
// becomes ESPO_ERR_PEER_TIMEOUT instead of a hung GPU.
template <typename F>
__device__ __forceinline__ bool spin_until(F pred, uint64_t timeout_ns) {
  const uint64_t t0 = globaltimer_ns();
  for (uint32_t it = 0;; ++it) {
    if (pred()) return true;
    if ((it & 63) == 63 && globaltimer_ns() - t0 > timeout_ns) return pred();
    __nanosleep(it < 64 ? 32 : 256);
  }
}

struct TpxParams {
  uint8_t* const* peer;   // [tp_world] exchange buffer bases (peer k's, mapped here)
  uint8_t* local;         // this rank's exchange buffer
  int tp_rank, tp_world;
  int64_t cap;            // rows per (slot, rank) block
  uint32_t epoch;
  int slot;
  uint64_t timeout_ns;    // bound on every wait (ESPO_OPT_PEER_TIMEOUT_MS)
};

// wait until every rank consumed epoch − 2 (the last user of this slot)
__global__ void k_tpx_wait_consumed(const TpxParams x, int* err) {
  if (threadIdx.x != 0 || x.epoch <= 2) return;
  const uint32_t* consumed = reinterpret_cast<const uint32_t*>(x.local + kTpxConsumedOff);
  const uint32_t need = x.epoch - 2;
  for (int k = 0; k < x.tp_world; ++k)
    if (!spin_until([&] { return ld_acquire_sys(consumed + k) >= need; }, x.timeout_ns)) {
      set_error(err, ESPO_ERR_PEER_TIMEOUT);
      return;
    }
}

// ready[slot][tp_rank] = epoch on every rank (after this rank's sweep stores)
__global__ void k_tpx_signal(const TpxParams x) {
  const int k = threadIdx.x;
  if (k >= x.tp_world) return;
  __threadfence_system();
  uint32_t* ready = reinterpret_cast<uint32_t*>(x.peer[k]);
  st_release_sys(ready + x.slot * x.tp_world + x.tp_rank, x.epoch);
}

// wait for every rank's partials of this epoch, then merge them (as k_fwd_combine)
__global__ void __launch_bounds__(256) k_tpx_combine(const TpxParams x, int64_t row_begin,
                                                     int64_t n_rows, Workspace ws) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    const uint32_t* ready = reinterpret_cast<const uint32_t*>(x.local) + x.slot * x.tp_world;
    ok = 1;
    for (int k = 0; k < x.tp_world && ok; ++k)
      if (!spin_until([&] { return ld_acquire_sys(ready + k) == x.epoch; }, x.timeout_ns)) ok = 0;
    if (!ok) set_error(ws.err, ESPO_ERR_PEER_TIMEOUT);
  }
  __syncthreads();
  if (!ok) return;
  const float4* g = reinterpret_cast<const float4*>(x.local + kTpxFlagBytes) +
                    int64_t(x.slot) * x.tp_world * x.cap;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = row_begin + r;
    if (!ws.flag[t]) continue;
    float R = -INFINITY, uy = __int_as_float(0x7fc00000);
    for (int k = 0; k < x.tp_world; ++k) {
      const float4 a = g[int64_t(k) * x.cap + r];
      R = fmaxf(R, a.x);
      if (!isnan(a.w)) uy = a.w;
    }
    float S = 0.f, W = 0.f;
    for (int k = 0; k < x.tp_world; ++k) {
      const float4 a = g[int64_t(k) * x.cap + r];
      float s = a.y, w = a.z;
      rebase(a.x, R, s, w);
      S += s;
      W += w;
    }
    if (isnan(uy)) set_error(ws.err, ESPO_ERR_INVALID_ARGUMENT);  // no shard owns the target
    finish_stats(R, S, W, uy, ws, t);
  }
}

// consumed[tp_rank] = epoch on every rank (after this rank's combine read its buffer)
__global__ void k_tpx_post(const TpxParams x) {
  const int k = threadIdx.x;
  if (k >= x.tp_world) return;
  uint32_t* consumed = reinterpret_cast<uint32_t*>(x.peer[k] + kTpxConsumedOff);
  st_release_sys(consumed + x.tp_rank, x.epoch);
}

}  // namespace espo
