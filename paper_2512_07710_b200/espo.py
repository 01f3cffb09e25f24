"""Thin Python binding of libespo (include/espo.h) — argument marshalling only.

Every step of the ESPO loss pass runs in the CUDA kernels of ``libespo.so`` (sm_100a);
this module only converts torch tensors to pointers/streams and status codes to
exceptions. PyTorch provides device memory, streams and process groups. There is no CPU
fallback: if ``libespo.so`` is missing or fails to load, every entry point raises.

C call → method:  espo_create → Espo(...), espo_prepare → Espo.prepare,
espo_loss_fwd → Espo.loss_fwd, espo_loss_finalize → Espo.loss_finalize,
espo_loss_bwd → Espo.loss_bwd, espo_get_error → Espo.get_error.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ESPO_LIB") or os.path.join(_HERE, "libespo.so")  # ESPO_LIB: A/B builds

ESPO_MAX_BUCKETS = 4
F32, BF16 = 0, 1
PART_QUANTILE, PART_WHOLE, PART_SINGLETON = 0, 1, 2
RATIO_GSPO_TOKEN, RATIO_LITERAL_OLD = 0, 1
NORM_SEQ, NORM_TOKEN = 0, 1
ZV_MASK, ZV_RLZVP = 0, 1
OPT_FWD_IMPL, OPT_BWD_IMPL, OPT_BLOCKS_PER_SM, OPT_LMHEAD_PARTS, OPT_LMHEAD_BWD_ROWS = 0, 1, 2, 3, 4
OPT_LMHEAD_2CTA = 5
OPT_FACTORED_IMPL = 6
OPT_PEER_TIMEOUT_MS = 7
OPT_LMHEAD_BWD_GEMM = 8
OPT_GEMM_GROUP_M = 9
OPT_GEMM_HINTS = 10
OPT_LMHEAD_COMPACT = 11
OPT_GEMM_SYNC = 12
OPT_LMHEAD_IMPL = 13
OPT_LMHEAD_RASTER = 14
REDUCE_LEN = 26          # ESPO_REDUCE_LEN: fp64 terms of espo_loss_reduce_local

STATUS = {
    0: "ESPO_OK", 1: "ESPO_ERR_INVALID_ARGUMENT", 2: "ESPO_ERR_ALIGNMENT",
    3: "ESPO_ERR_GROUPS_NOT_CONTIGUOUS", 4: "ESPO_ERR_BAD_STATE",
    5: "ESPO_ERR_NONFINITE_INPUT", 6: "ESPO_ERR_TOKEN_OUT_OF_RANGE",
    7: "ESPO_ERR_OUT_OF_MEMORY", 8: "ESPO_ERR_CUDA", 9: "ESPO_ERR_NCCL",
    10: "ESPO_ERR_UNSUPPORTED",
    11: "ESPO_ERR_BLAS", 12: "ESPO_ERR_PEER_TIMEOUT",
}
EXPORTED_SYMBOLS = [
    "espo_config_default", "espo_get_unique_id", "espo_create", "espo_destroy", "espo_prepare",
    "espo_loss_fwd", "espo_loss_finalize", "espo_loss_bwd", "espo_get_error",
    "espo_status_string", "espo_export_token_stats", "espo_export_rollout_stats",
    "espo_launch_count", "espo_set_option", "espo_set_entropies", "espo_loss_fwd_partial", "espo_loss_fwd_combine",
    "espo_attach_tp", "espo_lmhead_fwd", "espo_lmhead_bwd", "espo_set_mask", "espo_loss_fwd_bwd", "espo_tp_p2p_buffer", "espo_tp_p2p_open",
    "espo_tp_p2p_connect_local", "espo_tp_p2p_unmap", "espo_loss_fwd_p2p_send", "espo_loss_fwd_p2p_recv",
    "espo_attach_cp", "espo_cp_gather_local", "espo_reward_shaping_default",
    "espo_reshape_rewards", "espo_loss_fwd_factored", "espo_loss_row_scale",
    "espo_loss_reduce_local", "espo_loss_finalize_reduced", "espo_comm_size",
]


class EspoError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        self.code = STATUS.get(status, f"ESPO_ERR_{status}")
        super().__init__(f"{where}: {self.code}")


class Config(ctypes.Structure):
    _fields_ = [
        ("vocab", ctypes.c_int32), ("alpha", ctypes.c_float), ("eps_min", ctypes.c_float),
        ("n_buckets", ctypes.c_int32), ("split_num", ctypes.c_int32),
        ("split_den", ctypes.c_int32), ("partition", ctypes.c_int32),
        ("ratio_mode", ctypes.c_int32), ("norm", ctypes.c_int32),
        ("std_unbiased", ctypes.c_int32), ("adv_eps", ctypes.c_double),
        ("zv_var_eps", ctypes.c_double), ("logit_scale", ctypes.c_float),
        ("log_ratio_clamp", ctypes.c_float), ("logits_dtype", ctypes.c_int32),
        ("grad_dtype", ctypes.c_int32), ("zero_fill_inactive_rows", ctypes.c_int32),
        ("zv_mode", ctypes.c_int32), ("zvp_beta", ctypes.c_float),
        ("zvp_threshold", ctypes.c_float), ("vocab_begin", ctypes.c_int32),
        ("vocab_local", ctypes.c_int32), ("reserved", ctypes.c_int32 * 2),
    ]


class RewardShaping(ctypes.Structure):
    _fields_ = [("max_len", ctypes.c_int32), ("buffer", ctypes.c_int32),
                ("ngram", ctypes.c_int32), ("gamma_rep", ctypes.c_float),
                ("rep_thresh", ctypes.c_float), ("reserved", ctypes.c_int32 * 3)]


STATS_FIELDS = ["loss", "n_active_rollouts", "n_active_tokens", "n_zv_groups", "n_groups",
                "n_clipped_tokens", "mean_abs_logratio", "mean_entropy"]
STATS_ARRAYS = ["clip_frac", "mean_ratio", "mean_eps", "tokens_per_bucket"]
STATS_TAIL = ["mean_sq_logratio", "mean_k3"]
STATS_LEN = len(STATS_FIELDS) + ESPO_MAX_BUCKETS * len(STATS_ARRAYS) + len(STATS_TAIL)  # doubles


def stats_to_dict(t: torch.Tensor) -> dict:
    v = t.detach().to("cpu", torch.float64).tolist()
    d = {k: v[i] for i, k in enumerate(STATS_FIELDS)}
    o = len(STATS_FIELDS)
    for j, k in enumerate(STATS_ARRAYS):
        d[k] = v[o + j * ESPO_MAX_BUCKETS: o + (j + 1) * ESPO_MAX_BUCKETS]
    o += ESPO_MAX_BUCKETS * len(STATS_ARRAYS)
    for j, k in enumerate(STATS_TAIL):
        d[k] = v[o + j]
    return d


_lib = None


def load_library():
    """Loads libespo.so (after torch, so a world>1 context reuses torch's libnccl.so.2)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
    sig = {
        "espo_config_default": (None, [ctypes.POINTER(Config), I32]),
        "espo_get_unique_id": (I32, [P]),
        "espo_create": (I32, [ctypes.POINTER(Config), P, I32, I32, I32, ctypes.POINTER(P)]),
        "espo_destroy": (I32, [P]),
        "espo_prepare": (I32, [P, P, P, P, I32, I64, P, P, P]),
        "espo_loss_fwd": (I32, [P, P, I64, P, P, P, I64, I64, U32, P]),
        "espo_loss_finalize": (I32, [P, P, P, P]),
        "espo_loss_bwd": (I32, [P, P, I64, P, I64, P, I64, I64, P]),
        "espo_get_error": (I32, [P, P]),
        "espo_status_string": (ctypes.c_char_p, [I32]),
        "espo_export_token_stats": (I32, [P, I64, I64, P, P, P, P, P, P, P, P, P]),
        "espo_export_rollout_stats": (I32, [P, P, P, P, P, P, P, P]),
        "espo_launch_count": (ctypes.c_uint64, [P]),
        "espo_comm_size": (I32, [P]),
        "espo_set_option": (I32, [P, I32, I64]),
        "espo_set_entropies": (I32, [P, P, I64, I64, P]),
        "espo_loss_fwd_partial": (I32, [P, P, I64, P, P, P, I64, I64, P, P]),
        "espo_loss_fwd_combine": (I32, [P, P, I32, I64, I64, P]),
        "espo_attach_tp": (I32, [P, P, I32, I32]),
        "espo_lmhead_fwd": (I32, [P, P, I64, P, I64, I32, P, P, P, I64, I64, P]),
        "espo_set_mask": (I32, [P, P, P]),
        "espo_attach_cp": (I32, [P, P, I32, I32]),
        "espo_cp_gather_local": (I32, [P, P, I32, P]),
        "espo_tp_p2p_buffer": (I32, [P, I64, I32, P]),
        "espo_tp_p2p_open": (I32, [P, P, I32, I32]),
        "espo_tp_p2p_connect_local": (I32, [P, P, I32, I32]),
        "espo_tp_p2p_unmap": (I32, [P]),
        "espo_loss_fwd_p2p_send": (I32, [P, P, I64, P, P, P, I64, I64, P]),
        "espo_loss_fwd_p2p_recv": (I32, [P, I64, I64, P]),
        "espo_loss_fwd_bwd": (I32, [P, P, I64, P, P, P, I64, P, I64, I64, P]),
        "espo_loss_reduce_local": (I32, [P, P, P]),
        "espo_loss_finalize_reduced": (I32, [P, P, P, P, P]),
        "espo_loss_fwd_factored": (I32, [P, P, I64, P, P, P, P, I64, I64, I64, P]),
        "espo_loss_row_scale": (I32, [P, P, P, I64, I64, P]),
        "espo_lmhead_bwd": (I32, [P, P, I64, P, I64, I32, P, I64, I32, P, I64, P, I64, I64, P]),
        "espo_reward_shaping_default": (None, [ctypes.POINTER(RewardShaping), I32]),
        "espo_reshape_rewards": (I32, [P, ctypes.POINTER(RewardShaping), P, P, P, I32, I64, P,
                                       P, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _check(status, where):
    if status != 0:
        raise EspoError(status, where)


_DT = {torch.float32: F32, torch.bfloat16: BF16}


def check_tensor(t, name, dtype, device, rows=None, width=None, optional=False):
    """Argument check before a pointer crosses the C ABI (which only sees addresses and
    pitches): dtype, device, unit inner stride, and the row count / row width the call will
    touch. Raises TypeError (dtype) or ValueError (everything else); None passes only when
    `optional`. A 1-D tensor must be contiguous with ≥ rows elements; a 2-D tensor needs
    stride(-1) == 1, ≥ rows rows and ≥ width columns."""
    if t is None:
        if optional:
            return
        raise ValueError(f"{name} is required")
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor, got {type(t).__name__}")
    if t.dtype != dtype:
        raise TypeError(f"{name} dtype {t.dtype} != {dtype}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, the context on {device}")
    if t.dim() == 1:
        if t.numel() > 1 and t.stride(0) != 1:
            raise ValueError(f"{name} must be contiguous")
        if rows is not None and t.shape[0] < rows:
            raise ValueError(f"{name} has {t.shape[0]} elements < {rows}")
    elif t.dim() == 2:
        if t.shape[1] > 1 and t.stride(1) != 1:
            raise ValueError(f"{name} inner stride {t.stride(1)} != 1")
        if rows is not None and t.shape[0] < rows:
            raise ValueError(f"{name} has {t.shape[0]} rows < {rows}")
        if width is not None and t.shape[1] < width:
            raise ValueError(f"{name} has {t.shape[1]} columns < {width}")
    else:
        raise ValueError(f"{name} must be 1-D or 2-D, got {t.dim()}-D")


def new_unique_id() -> bytes:
    """A fresh NCCL unique id (espo_get_unique_id), e.g. for a one-rank communicator."""
    raw = ctypes.create_string_buffer(128)
    _check(load_library().espo_get_unique_id(raw), "espo_get_unique_id")
    return raw.raw


def bootstrap_unique_id(rank: int, process_group=None) -> bytes:
    """Rank 0 draws the NCCL unique id through libespo (espo_get_unique_id) and broadcasts
    its 128 bytes over the caller's torch.distributed process group (gloo or nccl)."""
    import torch.distributed as dist
    buf = [None]
    if rank == 0:
        raw = ctypes.create_string_buffer(128)
        _check(load_library().espo_get_unique_id(raw), "espo_get_unique_id")
        buf[0] = raw.raw
    if process_group is None:
        dist.broadcast_object_list(buf, src=0)
    else:   # `rank` is the rank inside `process_group`; its member 0 draws the id
        dist.broadcast_object_list(buf, group=process_group, group_src=0)
    return buf[0]


class Espo:
    """One ESPO loss context on one CUDA device (one rank). See include/espo.h."""

    def __init__(self, vocab: int, *, alpha=0.4, eps_min=0.01, n_buckets=2, split=(4, 5),
                 partition=PART_QUANTILE, ratio_mode=RATIO_GSPO_TOKEN, norm=NORM_SEQ,
                 std_unbiased=False, adv_eps=1e-6, zv_var_eps=0.0, logit_scale=1.0,
                 log_ratio_clamp=20.0, logits_dtype=torch.bfloat16, grad_dtype=None,
                 zero_fill_inactive_rows=True, zv_mode=ZV_MASK, zvp_beta=0.05,
                 zvp_threshold=0.5, vocab_shard=None, device=None, rank=0, world=1,
                 process_group=None, tp_rank=0, tp_world=1, tp_group=None, nccl_id=None):
        lib = load_library()
        self._lib = lib
        cfg = Config()
        lib.espo_config_default(ctypes.byref(cfg), int(vocab))
        cfg.alpha, cfg.eps_min = float(alpha), float(eps_min)
        cfg.n_buckets = int(n_buckets)
        cfg.split_num, cfg.split_den = int(split[0]), int(split[1])
        cfg.partition, cfg.ratio_mode, cfg.norm = int(partition), int(ratio_mode), int(norm)
        cfg.std_unbiased = int(bool(std_unbiased))
        cfg.adv_eps, cfg.zv_var_eps = float(adv_eps), float(zv_var_eps)
        cfg.logit_scale, cfg.log_ratio_clamp = float(logit_scale), float(log_ratio_clamp)
        self.logits_dtype = logits_dtype
        self.grad_dtype = grad_dtype if grad_dtype is not None else logits_dtype
        cfg.logits_dtype, cfg.grad_dtype = _DT[self.logits_dtype], _DT[self.grad_dtype]
        cfg.zero_fill_inactive_rows = int(bool(zero_fill_inactive_rows))
        cfg.zv_mode = int(zv_mode)
        cfg.zvp_beta, cfg.zvp_threshold = float(zvp_beta), float(zvp_threshold)
        if vocab_shard is not None:                  # (begin, width) of this rank's columns
            cfg.vocab_begin, cfg.vocab_local = int(vocab_shard[0]), int(vocab_shard[1])
        self.cfg = cfg
        self.vocab = int(vocab)
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.rank, self.world = int(rank), int(world)
        uid = None
        if nccl_id is not None:          # explicit id (any world, including a 1-rank group)
            uid = ctypes.create_string_buffer(bytes(nccl_id), 128)
        elif self.world > 1:
            uid = ctypes.create_string_buffer(
                bootstrap_unique_id(self.rank, process_group), 128)
        h = ctypes.c_void_p()
        _check(lib.espo_create(ctypes.byref(cfg), uid, self.rank, self.world,
                               self.device.index, ctypes.byref(h)), "espo_create")
        self._h = h
        self.n_tokens = 0
        self.n_rollouts = 0
        self.cp_rank, self.cp_world = 0, 1
        if tp_world > 1:
            tuid = ctypes.create_string_buffer(bootstrap_unique_id(tp_rank, tp_group), 128)
            _check(lib.espo_attach_tp(self._h, tuid, int(tp_rank), int(tp_world)),
                   "espo_attach_tp")

    # -- lifecycle ------------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.espo_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def set_option(self, option: int, value: int):
        _check(self._lib.espo_set_option(self._h, int(option), int(value)), "espo_set_option")

    @property
    def launch_count(self) -> int:
        return int(self._lib.espo_launch_count(self._h))

    @property
    def comm_size(self) -> int:
        """espo_comm_size: ranks of the DP communicator (ncclCommCount; 1 at world 1)."""
        return int(self._lib.espo_comm_size(self._h))

    @property
    def width(self) -> int:
        """Columns a logits chunk of this context holds (the shard width when sharded)."""
        return int(self.cfg.vocab_local) if self.cfg.vocab_local > 0 else self.vocab

    def _check_fwd(self, logits, tokens, old_logp, mask):
        check_tensor(logits, "logits", self.logits_dtype, self.device, width=self.width)
        if logits.dim() != 2:
            raise ValueError("logits must be 2-D [rows, >= vocab]")
        n = int(logits.shape[0])
        check_tensor(tokens, "tokens", torch.int32, self.device, n)
        check_tensor(old_logp, "old_logp", torch.float32, self.device, n)
        check_tensor(mask, "mask", torch.uint8, self.device, n, optional=True)
        return n

    def _check_grad(self, t, name, n, optional=False):
        check_tensor(t, name, self.grad_dtype, self.device, n, self.width, optional=optional)
        if t is not None and t.dim() != 2:
            raise ValueError(f"{name} must be 2-D [rows, >= vocab]")

    def _check_scalar(self, grad_loss):
        check_tensor(grad_loss, "grad_loss", torch.float32, self.device, 1, optional=True)

    # -- the pass ---------------------------------------------------------------------------
    def prepare(self, rewards, group_ids, seq_offsets, n_tokens=None, adv_out=None, zv_out=None):
        """espo_prepare: rewards f32[R], group_ids i32[R], seq_offsets i64[R+1] (device)."""
        R = int(rewards.shape[0])
        check_tensor(rewards, "rewards", torch.float32, self.device, R)
        check_tensor(group_ids, "group_ids", torch.int32, self.device, R)
        check_tensor(seq_offsets, "seq_offsets", torch.int64, self.device, R + 1)
        check_tensor(adv_out, "adv_out", torch.float32, self.device, R, optional=True)
        check_tensor(zv_out, "zv_out", torch.uint8, self.device, R, optional=True)
        if n_tokens is None:
            n_tokens = int(seq_offsets[-1].item())
        self.n_tokens, self.n_rollouts = int(n_tokens), R
        _check(self._lib.espo_prepare(self._h, _ptr(rewards), _ptr(group_ids), _ptr(seq_offsets),
                                      R, int(n_tokens), _ptr(adv_out), _ptr(zv_out),
                                      self._stream()), "espo_prepare")

    def loss_fwd(self, logits, tokens, old_logp, mask=None, row_begin=0):
        """espo_loss_fwd over rows [row_begin, row_begin + logits.shape[0])."""
        n = self._check_fwd(logits, tokens, old_logp, mask)
        _check(self._lib.espo_loss_fwd(self._h, _ptr(logits), int(logits.stride(0)),
                                       _ptr(tokens), _ptr(old_logp), _ptr(mask), int(row_begin),
                                       n, 0, self._stream()), "espo_loss_fwd")

    # -- context parallelism ------------------------------------------------------------------
    def attach_tp_id(self, nccl_id: bytes, tp_rank: int, tp_world: int):
        """espo_attach_tp with an explicit NCCL id (the TP group's id, already shared)."""
        _check(self._lib.espo_attach_tp(self._h, ctypes.create_string_buffer(bytes(nccl_id), 128),
                                        int(tp_rank), int(tp_world)), "espo_attach_tp")

    def attach_cp(self, cp_rank: int, cp_world: int, group=None, local=False, nccl_id=None):
        """espo_attach_cp: this context is CP rank cp_rank of cp_world (token blocks). With
        local=True (same-device emulation) no communicator is created; call cp_gather_local
        before loss_finalize. Otherwise the NCCL id is broadcast over `group`."""
        uid = None
        if nccl_id is not None:
            uid = ctypes.create_string_buffer(bytes(nccl_id), 128)
        elif cp_world > 1 and not local:
            uid = ctypes.create_string_buffer(bootstrap_unique_id(cp_rank, group), 128)
        _check(self._lib.espo_attach_cp(self._h, uid, int(cp_rank), int(cp_world)),
               "espo_attach_cp")
        self.cp_rank, self.cp_world = int(cp_rank), int(cp_world)

    def cp_block(self):
        """(first, end) token rows this CP rank owns for the prepared batch."""
        tb = -(-self.n_tokens // self.cp_world)
        return min(self.n_tokens, self.cp_rank * tb), min(self.n_tokens, (self.cp_rank + 1) * tb)

    def cp_gather_local(self, ranks):
        arr = (ctypes.c_void_p * len(ranks))(*[r._h.value for r in ranks])
        _check(self._lib.espo_cp_gather_local(self._h, arr, len(ranks), self._stream()),
               "espo_cp_gather_local")

    # -- vocabulary-parallel exchange over peer memory -----------------------------------
    def tp_p2p_buffer(self, max_rows: int, tp_world: int) -> bytes:
        """espo_tp_p2p_buffer: allocate this rank's exchange buffer; returns its IPC handle."""
        h = ctypes.create_string_buffer(64)
        _check(self._lib.espo_tp_p2p_buffer(self._h, int(max_rows), int(tp_world), h),
               "espo_tp_p2p_buffer")
        return h.raw

    def tp_p2p_open(self, handles: bytes, tp_rank: int, tp_world: int):
        """espo_tp_p2p_open: map the peers' buffers (handles concatenated in TP-rank order)."""
        buf = ctypes.create_string_buffer(bytes(handles), len(handles))
        _check(self._lib.espo_tp_p2p_open(self._h, buf, int(tp_rank), int(tp_world)),
               "espo_tp_p2p_open")

    def tp_p2p_connect_local(self, ranks, tp_rank: int):
        """espo_tp_p2p_connect_local: same-device TP group (tests / emulation)."""
        arr = (ctypes.c_void_p * len(ranks))(*[r._h.value for r in ranks])
        _check(self._lib.espo_tp_p2p_connect_local(self._h, arr, int(tp_rank), len(ranks)),
               "espo_tp_p2p_connect_local")

    def tp_p2p_unmap(self):
        _check(self._lib.espo_tp_p2p_unmap(self._h), "espo_tp_p2p_unmap")

    def loss_fwd_p2p_send(self, logits, tokens, old_logp, mask=None, row_begin=0):
        self._check_fwd(logits, tokens, old_logp, mask)
        _check(self._lib.espo_loss_fwd_p2p_send(self._h, _ptr(logits), int(logits.stride(0)),
                                                _ptr(tokens), _ptr(old_logp), _ptr(mask),
                                                int(row_begin), int(logits.shape[0]),
                                                self._stream()), "espo_loss_fwd_p2p_send")

    def loss_fwd_p2p_recv(self, row_begin, n_rows):
        _check(self._lib.espo_loss_fwd_p2p_recv(self._h, int(row_begin), int(n_rows),
                                                self._stream()), "espo_loss_fwd_p2p_recv")

    def set_mask(self, mask=None):
        """espo_set_mask: single-pass mode; D counted from the batch mask u8[T] (None = ones)."""
        check_tensor(mask, "mask", torch.uint8, self.device, self.n_tokens, optional=True)
        _check(self._lib.espo_set_mask(self._h, _ptr(mask), self._stream()), "espo_set_mask")

    def loss_fwd_bwd(self, logits, tokens, old_logp, dlogits=None, row_begin=0, grad_loss=None):
        """espo_loss_fwd_bwd: forward + backward of a chunk of complete rollouts."""
        n = self._check_fwd(logits, tokens, old_logp, None)
        self._check_scalar(grad_loss)
        if dlogits is None:
            dlogits = torch.empty(logits.shape, dtype=self.grad_dtype, device=logits.device)
        self._check_grad(dlogits, "dlogits", n)
        _check(self._lib.espo_loss_fwd_bwd(self._h, _ptr(logits), int(logits.stride(0)),
                                           _ptr(tokens), _ptr(old_logp), _ptr(dlogits),
                                           int(dlogits.stride(0)), _ptr(grad_loss),
                                           int(row_begin), int(logits.shape[0]), self._stream()),
               "espo_loss_fwd_bwd")
        return dlogits

    def loss_fwd_factored(self, logits, tokens, old_logp, mask=None, grad=None, row_begin=0):
        """espo_loss_fwd_factored: the forward of these rows plus G = onehot(y) − softmax(λz)
        written to `grad` (allocated if None; may be `logits` itself). Returns grad.
        In compact mode rows without gradient are left as they were, so an allocated grad
        is zero-initialised (a consumer's diag(scale)·G then never meets garbage)."""
        n = self._check_fwd(logits, tokens, old_logp, mask)
        if grad is None:
            alloc = torch.empty if self.cfg.zero_fill_inactive_rows else torch.zeros
            grad = alloc(logits.shape, dtype=self.grad_dtype, device=logits.device)
        self._check_grad(grad, "grad", n)
        _check(self._lib.espo_loss_fwd_factored(
            self._h, _ptr(logits), int(logits.stride(0)), _ptr(tokens), _ptr(old_logp), _ptr(mask),
            _ptr(grad), int(grad.stride(0)), int(row_begin), int(logits.shape[0]), self._stream()),
            "espo_loss_fwd_factored")
        return grad

    def loss_row_scale(self, row_begin=0, n_rows=None, grad_loss=None, out=None):
        """espo_loss_row_scale: per-row scale_t with dlogits_t = scale_t · G_t."""
        if n_rows is None:
            n_rows = self.n_tokens - row_begin
        if out is None:
            out = torch.empty(n_rows, dtype=torch.float32, device=self.device)
        check_tensor(out, "out", torch.float32, self.device, n_rows)
        self._check_scalar(grad_loss)
        _check(self._lib.espo_loss_row_scale(self._h, _ptr(grad_loss), _ptr(out), int(row_begin),
                                             int(n_rows), self._stream()), "espo_loss_row_scale")
        return out

    def loss_fwd_partial(self, logits, tokens, old_logp, mask=None, row_begin=0, partial=None):
        """espo_loss_fwd_partial: this vocabulary shard's per-row {R, S, W, u_y} (f32[n, 4])."""
        n = self._check_fwd(logits, tokens, old_logp, mask)
        if partial is None:
            partial = torch.empty((n, 4), dtype=torch.float32, device=logits.device)
        check_tensor(partial, "partial", torch.float32, self.device, n, 4)
        if partial.dim() != 2 or partial.stride(0) != 4:
            raise ValueError("partial must be a dense [n_rows, 4] tensor")
        _check(self._lib.espo_loss_fwd_partial(self._h, _ptr(logits), int(logits.stride(0)),
                                               _ptr(tokens), _ptr(old_logp), _ptr(mask),
                                               int(row_begin), n, _ptr(partial), self._stream()),
               "espo_loss_fwd_partial")
        return partial

    def loss_fwd_combine(self, partials, row_begin=0):
        """espo_loss_fwd_combine over partials [n_shards, n_rows, 4] (device)."""
        partials = partials.contiguous()
        if partials.dim() != 3 or partials.shape[2] != 4:
            raise ValueError("partials must be [n_shards, n_rows, 4]")
        if partials.dtype != torch.float32 or partials.device != self.device:
            raise TypeError("partials must be float32 on the context's device")
        _check(self._lib.espo_loss_fwd_combine(self._h, _ptr(partials), int(partials.shape[0]),
                                               int(row_begin), int(partials.shape[1]),
                                               self._stream()), "espo_loss_fwd_combine")

    def lmhead_fwd(self, hidden, weight, tokens, old_logp, mask=None, row_begin=0):
        """espo_lmhead_fwd: fused LM head (tcgen05) + forward statistics; logits never
        materialised. hidden bf16 [n, d], weight bf16 [vocab, d]."""
        check_tensor(hidden, "hidden", torch.bfloat16, self.device)
        n, d = int(hidden.shape[0]), int(hidden.shape[1])
        full = self.vocab if self.cfg.vocab_local == 0 else None   # sharded: UNSUPPORTED below
        check_tensor(weight, "weight", torch.bfloat16, self.device, full, d)
        check_tensor(tokens, "tokens", torch.int32, self.device, n)
        check_tensor(old_logp, "old_logp", torch.float32, self.device, n)
        check_tensor(mask, "mask", torch.uint8, self.device, n, optional=True)
        _check(self._lib.espo_lmhead_fwd(self._h, _ptr(hidden), int(hidden.stride(0)),
                                         _ptr(weight), int(weight.stride(0)), d, _ptr(tokens),
                                         _ptr(old_logp), _ptr(mask), int(row_begin), n,
                                         self._stream()), "espo_lmhead_fwd")

    def lmhead_bwd(self, hidden, weight, dhidden=None, dweight=None, row_begin=0, grad_loss=None,
                   dh_dtype=None):
        """espo_lmhead_bwd: dhidden (overwritten, [n, d]) and dweight (f32 [vocab, d],
        accumulated) for rows [row_begin, row_begin + n) of the fused LM head."""
        check_tensor(hidden, "hidden", torch.bfloat16, self.device)
        n, d = int(hidden.shape[0]), int(hidden.shape[1])
        full = self.vocab if self.cfg.vocab_local == 0 else None
        check_tensor(weight, "weight", torch.bfloat16, self.device, full, d)
        self._check_scalar(grad_loss)
        if dhidden is None:
            dhidden = torch.empty((n, d), dtype=dh_dtype or torch.float32, device=hidden.device)
        if dhidden is not False:
            if dhidden.dtype not in _DT:
                raise TypeError(f"dhidden dtype {dhidden.dtype} not float32/bfloat16")
            check_tensor(dhidden, "dhidden", dhidden.dtype, self.device, n, d)
        check_tensor(dweight, "dweight", torch.float32, self.device, full, d, optional=True)
        dt = _DT[dhidden.dtype] if dhidden is not False else F32
        dh = None if dhidden is False else dhidden
        _check(self._lib.espo_lmhead_bwd(self._h, _ptr(hidden), int(hidden.stride(0)),
                                         _ptr(weight), int(weight.stride(0)), d, _ptr(dh),
                                         int(dh.stride(0)) if dh is not None else 0, dt,
                                         _ptr(dweight),
                                         int(dweight.stride(0)) if dweight is not None else 0,
                                         _ptr(grad_loss), int(row_begin), n, self._stream()),
               "espo_lmhead_bwd")
        return dh, dweight

    def reshape_rewards(self, base_rewards, tokens, seq_offsets, n_tokens, max_len, buffer=0,
                        ngram=4, gamma_rep=1.0, rep_thresh=0.2):
        """espo_reshape_rewards (ZVE stage 2): returns (rewards, length_pen, rep_pen) f32[R]."""
        prm = RewardShaping()
        self._lib.espo_reward_shaping_default(ctypes.byref(prm), int(max_len))
        prm.buffer, prm.ngram = int(buffer), int(ngram)
        prm.gamma_rep, prm.rep_thresh = float(gamma_rep), float(rep_thresh)
        R = int(base_rewards.shape[0])
        out = [torch.empty(R, dtype=torch.float32, device=base_rewards.device) for _ in range(3)]
        _check(self._lib.espo_reshape_rewards(self._h, ctypes.byref(prm), _ptr(base_rewards),
                                              _ptr(tokens), _ptr(seq_offsets), R, int(n_tokens),
                                              *[_ptr(o) for o in out], self._stream()),
               "espo_reshape_rewards")
        return tuple(out)

    def loss_finalize(self, loss_out=None, stats_out=None):
        """espo_loss_finalize → (loss f32[1], stats f64[STATS_LEN]) device tensors."""
        loss_out, stats_out = self._outs(loss_out, stats_out)
        _check(self._lib.espo_loss_finalize(self._h, _ptr(loss_out), _ptr(stats_out),
                                            self._stream()), "espo_loss_finalize")
        return loss_out, stats_out

    def _outs(self, loss_out, stats_out):
        if loss_out is None:
            loss_out = torch.empty(1, dtype=torch.float32, device=self.device)
        if stats_out is None:
            stats_out = torch.empty(STATS_LEN, dtype=torch.float64, device=self.device)
        check_tensor(loss_out, "loss_out", torch.float32, self.device, 1)
        check_tensor(stats_out, "stats_out", torch.float64, self.device, STATS_LEN)
        return loss_out, stats_out

    def loss_reduce_local(self, partial_out=None):
        """espo_loss_reduce_local → this rank's REDUCE_LEN fp64 terms (device), to be summed
        over ranks by the caller's collective and passed to loss_finalize_reduced."""
        if partial_out is None:
            partial_out = torch.empty(REDUCE_LEN, dtype=torch.float64, device=self.device)
        check_tensor(partial_out, "partial_out", torch.float64, self.device, REDUCE_LEN)
        _check(self._lib.espo_loss_reduce_local(self._h, _ptr(partial_out), self._stream()),
               "espo_loss_reduce_local")
        return partial_out

    def loss_finalize_reduced(self, reduced, loss_out=None, stats_out=None):
        """espo_loss_finalize_reduced with the rank-summed terms → (loss, stats)."""
        check_tensor(reduced, "reduced", torch.float64, self.device, REDUCE_LEN)
        loss_out, stats_out = self._outs(loss_out, stats_out)
        _check(self._lib.espo_loss_finalize_reduced(self._h, _ptr(reduced), _ptr(loss_out),
                                                    _ptr(stats_out), self._stream()),
               "espo_loss_finalize_reduced")
        return loss_out, stats_out

    def loss_bwd(self, logits, dlogits=None, row_begin=0, grad_loss=None):
        """espo_loss_bwd: d(grad_loss·loss)/d logits for rows of this chunk."""
        check_tensor(logits, "logits", self.logits_dtype, self.device, width=self.width)
        if logits.dim() != 2:
            raise ValueError("logits must be 2-D [rows, >= vocab]")
        self._check_scalar(grad_loss)
        if dlogits is None:
            dlogits = torch.empty(logits.shape, dtype=self.grad_dtype, device=logits.device)
        self._check_grad(dlogits, "dlogits", int(logits.shape[0]))
        _check(self._lib.espo_loss_bwd(self._h, _ptr(logits), int(logits.stride(0)),
                                       _ptr(dlogits), int(dlogits.stride(0)), _ptr(grad_loss),
                                       int(row_begin), int(logits.shape[0]), self._stream()),
               "espo_loss_bwd")
        return dlogits

    def set_entropies(self, entropy, row_begin=0):
        """espo_set_entropies: caller-supplied selection entropies (f32 [n], nats) for rows
        [row_begin, row_begin + n): used for the entropy buckets, Eq. 3's ε and RL-ZVP
        instead of the sweep's own (reading Q4's alternative)."""
        check_tensor(entropy, "entropy", torch.float32, self.device)
        if entropy.dim() != 1:
            raise ValueError("entropy must be a 1-D float32 tensor")
        _check(self._lib.espo_set_entropies(self._h, _ptr(entropy), int(row_begin),
                                            int(entropy.shape[0]), self._stream()),
               "espo_set_entropies")

    def get_error(self):
        """espo_get_error: synchronises the current stream; raises on a device error."""
        _check(self._lib.espo_get_error(self._h, self._stream()), "espo_get_error")

    # -- introspection ------------------------------------------------------------------------
    def export_token_stats(self, row_begin=0, n_rows=None):
        if n_rows is None:
            n_rows = self.n_tokens - row_begin
        f = lambda: torch.empty(n_rows, dtype=torch.float32, device=self.device)
        u = lambda: torch.empty(n_rows, dtype=torch.uint8, device=self.device)
        out = dict(lse=f(), lp=f(), H=f(), q=f(), coef=f(), bucket=u(), clip=u(), valid=u())
        _check(self._lib.espo_export_token_stats(
            self._h, int(row_begin), int(n_rows), *[_ptr(out[k]) for k in
                                                    ("lse", "lp", "H", "q", "coef", "bucket",
                                                     "clip", "valid")],
            self._stream()), "espo_export_token_stats")
        return out

    def export_rollout_stats(self):
        R = self.n_rollouts
        d = self.device
        out = dict(adv=torch.empty(R, dtype=torch.float64, device=d),
                   zv=torch.empty(R, dtype=torch.uint8, device=d),
                   active=torch.empty(R, dtype=torch.uint8, device=d),
                   J=torch.empty(R, dtype=torch.float64, device=d),
                   nb=torch.empty(R, dtype=torch.int32, device=d),
                   theta=torch.empty(R * (ESPO_MAX_BUCKETS - 1), dtype=torch.float32, device=d))
        _check(self._lib.espo_export_rollout_stats(
            self._h, *[_ptr(out[k]) for k in ("adv", "zv", "active", "J", "nb", "theta")],
            self._stream()), "espo_export_rollout_stats")
        out["theta"] = out["theta"].view(R, ESPO_MAX_BUCKETS - 1)
        return out


def attach_tp_p2p(ctx: "Espo", max_rows: int, tp_rank: int, tp_world: int, group=None):
    """Connects a vocabulary-sharded context to its TP group over peer memory: allocate the
    exchange buffer, all-gather the IPC handles over `group` (torch.distributed), map them."""
    import torch.distributed as dist
    h = ctx.tp_p2p_buffer(max_rows, tp_world)
    handles = [None] * tp_world
    dist.all_gather_object(handles, h, group=group)
    ctx.tp_p2p_open(b"".join(handles), tp_rank, tp_world)


def espo_loss(ctx: Espo, logits, tokens, old_logp, rewards, group_ids, seq_offsets, mask=None,
              grad_loss=None, dlogits=None, with_grad=True):
    """Single-chunk convenience: prepare → fwd → finalize → bwd. Returns
    (loss f32[1], stats f64[...], dlogits or None), all on the device."""
    ctx.prepare(rewards, group_ids, seq_offsets, n_tokens=int(logits.shape[0]))
    ctx.loss_fwd(logits, tokens, old_logp, mask)
    loss, stats = ctx.loss_finalize()
    dz = ctx.loss_bwd(logits, dlogits, grad_loss=grad_loss) if with_grad else None
    return loss, stats, dz


class EspoLossFunction(torch.autograd.Function):
    """autograd wrapper (single chunk): loss = ESPO(logits); backward = espo_loss_bwd."""

    @staticmethod
    def forward(fctx, logits, ctx, tokens, old_logp, rewards, group_ids, seq_offsets, mask=None):
        ctx.prepare(rewards, group_ids, seq_offsets, n_tokens=int(logits.shape[0]))
        ctx.loss_fwd(logits, tokens, old_logp, mask)
        loss, _ = ctx.loss_finalize()
        fctx.espo = ctx
        fctx.save_for_backward(logits)
        return loss.reshape(())

    @staticmethod
    def backward(fctx, grad_out):
        (logits,) = fctx.saved_tensors
        g = grad_out.reshape(1).to(torch.float32).contiguous()
        dz = fctx.espo.loss_bwd(logits, grad_loss=g)
        return (dz.to(logits.dtype),) + (None,) * 7
