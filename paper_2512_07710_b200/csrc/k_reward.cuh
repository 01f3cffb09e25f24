// k_reward.cuh — ZVE stage 2 "reward reshaping" (concrete form SPEC.md:262-265):
// length penalty (linear ramp to −1 over the last `buffer` tokens before max_len) and
// repetition penalty −γ·max(0, f − thresh), f = fraction of n-gram positions whose n-gram
// occurred earlier in the same response. One CTA per rollout; the "occurred earlier" test
// uses a per-rollout open-addressing table in global scratch (64-bit n-gram hash → first
// position, atomicCAS / atomicMin) and verifies the tokens of the first occurrence, so a hit
// is never false; a miss could only come from a 64-bit hash collision between two distinct
// n-grams of one response.
#pragma once
#include "common.cuh"

namespace espo {

constexpr uint64_t kEmptyKey = ~0ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct ReshapeParams {
  const float* base;
  const int32_t* tokens;
  const int64_t* seq_off;
  int R;
  int max_len, buffer, ngram;
  float gamma_rep, rep_thresh;
  float* out;
  float* len_pen;   // nullable
  float* rep_pen;   // nullable
  uint64_t* keys;   // scratch [4·T]
  int32_t* first;   // scratch [4·T]
};

__global__ void __launch_bounds__(256) k_reshape_rewards(const ReshapeParams p) {
  __shared__ int s_cnt[8];
  const int i = blockIdx.x;
  const int64_t b = p.seq_off[i], e = p.seq_off[i + 1];
  const int n = static_cast<int>(e - b);
  const int g = p.ngram;
  const int m = n - g + 1;           // n-gram positions
  int cnt = 0;
  if (m > 0) {
    int cap = 1;
    while (cap < 2 * m) cap <<= 1;   // ≤ 4m ≤ 4n: fits the rollout's scratch region
    uint64_t* keys = p.keys + 4 * b;
    int32_t* first = p.first + 4 * b;
    for (int s = threadIdx.x; s < cap; s += blockDim.x) {
      keys[s] = kEmptyKey;
      first[s] = INT32_MAX;
    }
    __syncthreads();
    const int32_t* tok = p.tokens + b;
    auto key_of = [&](int pos) {
      uint64_t h = 0x243F6A8885A308D3ull;
      for (int k = 0; k < g; ++k) h = mix64(h ^ static_cast<uint32_t>(tok[pos + k]));
      return h == kEmptyKey ? h - 1 : h;
    };
    for (int pos = threadIdx.x; pos < m; pos += blockDim.x) {
      const uint64_t key = key_of(pos);
      int s = static_cast<int>(key & uint64_t(cap - 1));
      while (true) {
        const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(&keys[s]),
                                                  kEmptyKey, key);
        if (prev == kEmptyKey || prev == key) {
          atomicMin(&first[s], pos);
          break;
        }
        s = (s + 1) & (cap - 1);
      }
    }
    __syncthreads();
    for (int pos = threadIdx.x; pos < m; pos += blockDim.x) {
      const uint64_t key = key_of(pos);
      int s = static_cast<int>(key & uint64_t(cap - 1));
      while (keys[s] != key) s = (s + 1) & (cap - 1);
      const int f = first[s];
      if (f < pos) {
        bool same = true;
        for (int k = 0; k < g; ++k) same &= tok[f + k] == tok[pos + k];
        cnt += same ? 1 : 0;
      }
    }
  }
  // deterministic block sum of the integer count
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) s_cnt[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int rep = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) rep += s_cnt[w];
    const int buf = p.buffer > 0 ? p.buffer : (p.max_len + 7) / 8;
    const int start = p.max_len - buf;
    double lpen;
    if (n <= start) lpen = 0.0;
    else if (n >= p.max_len) lpen = -1.0;
    else lpen = -static_cast<double>(n - start) / static_cast<double>(buf);
    const double frac = m > 0 ? static_cast<double>(rep) / static_cast<double>(m) : 0.0;
    const double over = frac - static_cast<double>(p.rep_thresh);
    const double rpen = -static_cast<double>(p.gamma_rep) * (over > 0.0 ? over : 0.0);
    const double fin = (static_cast<double>(p.base[i]) + lpen) + rpen;
    p.out[i] = static_cast<float>(fin);
    if (p.len_pen) p.len_pen[i] = static_cast<float>(lpen);
    if (p.rep_pen) p.rep_pen[i] = static_cast<float>(rpen);
  }
}

}  // namespace espo
