// workspace.cuh — device workspace owned by an espo context (layout in DESIGN.md §HBM).
#pragma once
#include <cstdint>

namespace espo {

struct Workspace {
  // ---- per token [T] (SoA; ≈ 31 B/token) ----
  float* lse = nullptr;      // log Σ_v exp(λ z_v)                (K2)
  float* lp = nullptr;       // log π_θ(y_t)                      (K2)
  float* H = nullptr;        // entropy e_t (nats, ≥ 0)           (K2)
  float* q = nullptr;        // 1 − p_y = Σ_{v≠y} p_v             (K2)
  float* old = nullptr;      // log π_old(y_t) (copied at fwd)    (K2)
  float* coef = nullptr;     // c_t = Â·v·κ·w (∂J_i/∂lp_t)        (K3)
  int32_t* y = nullptr;      // token (copied at fwd)             (K2)
  int32_t* row_seq = nullptr;// rollout of each row               (K1)
  uint8_t* flag = nullptr;   // 1 = row read (active cand ∧ mask) (K2)
  uint8_t* bucket = nullptr; // stats bucket                      (K3)
  uint8_t* clip = nullptr;   // 1 = gradient clipped              (K3)
  uint8_t* pmask = nullptr;  // single-pass mode: copy of the batch mask (espo_set_mask)
  void* list = nullptr;      // per-chunk row records (FwdRec / BwdRec), 32 B × T
  int32_t* zlist = nullptr;  // per-chunk zero-fill rows (bwd), 4 B × T
  float* partial = nullptr;  // vocabulary shard: per-row {R, S, W, u_y}, 16 B × T
  float* gathered = nullptr; // TP all-gather target [tp_world][rows][4]
  // ---- per rollout [R] ----
  int64_t* seq_off = nullptr;  // [R+1] copy of seq_offsets       (K1)
  double* adv = nullptr;       // Â_i (0 for ZV)                  (K1)
  uint8_t* cand = nullptr;     // 1 = rows are read (group not eliminated) (K1)
  int8_t* zsign = nullptr;     // RL-ZVP: +1 / −1 reshaped ZV rollout, 0 otherwise (K1)
  uint8_t* ghead = nullptr;    // 1 = first rollout of a group, 2 = first of a ZV group
  uint8_t* active = nullptr;   // cand ∧ n_i ≥ 1                  (K3)
  int32_t* nb = nullptr;       // non-empty buckets               (K3)
  double* J = nullptr;         // J_i = Σ_t w_t ℓ_t               (K3)
  float* theta = nullptr;      // [R·(kMaxK−1)] entropy thresholds (K3)
  double* red_r = nullptr;     // [kRedLen·R] per-rollout reduction terms (K3), SoA
  // ---- scalars ----
  double* red = nullptr;       // [kRedLen] rank-local → all-reduced sums (K4)
  float* bwd_scale = nullptr;  // [1] λ/D (0 if D == 0)            (K4b; K0 in single-pass)
  double* dpre = nullptr;      // [2] single-pass: {N, T_active} counted from the mask (K0)
  int* err = nullptr;          // sticky device error word
  int* count = nullptr;        // [2] row-list lengths of the current sweep
};

}  // namespace espo
