"""otk — B200-native hot path of OpenTinker's (arxiv 2601.07376) RL policy-gradient update.

Thin ctypes binding over ``libotk.so`` (C ABI, ``include/otk.h``). Functions carry the C names and
only marshal arguments: every step of the path runs in the library's sm_100a kernels. torch supplies
device memory and streams. There is no CPU fallback: importing this package without the built
library raises ImportError (build it with ``python paper_2601_07376_b200/build.py``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OTK_LIB") or os.path.join(HERE, "libotk.so")  # OTK_LIB: experiment builds only

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2601_07376_b200/build.py` "
                      "(the otk hot path has no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

OTK_F32, OTK_BF16 = 0, 1
OTK_KL_K1, OTK_KL_K2, OTK_KL_K3 = 1, 2, 3
OTK_ANY_AGENT = -1
OTK_ADV_STD_NORM, OTK_ADV_UNBIASED, OTK_ADV_SKIP_UNGROUPED = 0x1, 0x2, 0x4
CONTEXT, ACTION, OBSERVATION, PAD = 0, 1, 2, 3

STATUS = {0: "OTK_OK", 1: "OTK_ERR_INVALID_ARG", 2: "OTK_ERR_SHAPE", 3: "OTK_ERR_ALIGNMENT", 4: "OTK_ERR_DTYPE",
          5: "OTK_ERR_EMPTY_GROUP", 6: "OTK_ERR_UNTERMINATED", 7: "OTK_ERR_BAD_TRAJECTORY",
          8: "OTK_ERR_TARGET_RANGE", 9: "OTK_ERR_CUDA", 10: "OTK_ERR_GROUP_RANGE",
          11: "OTK_ERR_PEER_TIMEOUT", 12: "OTK_ERR_NCCL", 13: "OTK_ERR_NO_COMM"}


class OtkError(RuntimeError):
    def __init__(self, status: int, detail: str = ""):
        self.status = int(status)
        self.name = STATUS.get(self.status, "OTK_ERR_UNKNOWN")
        super().__init__(f"{self.name}: {detail}")


class otk_traj_batch(C.Structure):
    _fields_ = [("num_traj", C.c_int32), ("num_rows", C.c_int64), ("tok_offsets", C.c_void_p),
                ("seg_offsets", C.c_void_p), ("seg_source", C.c_void_p), ("seg_agent", C.c_void_p),
                ("seg_len", C.c_void_p), ("terminated", C.c_void_p), ("traj_agent", C.c_void_p)]


class otk_loss_cfg(C.Structure):
    _fields_ = [("clip_low", C.c_double), ("clip_high", C.c_double), ("kl_beta", C.c_double),
                ("log_ratio_clamp", C.c_double), ("logit_scale", C.c_double), ("kl_type", C.c_int32),
                ("zero_masked_rows", C.c_int32), ("accumulate_stats", C.c_int32), ("reserved", C.c_int32),
                ("ent_coef", C.c_double), ("dual_clip", C.c_double), ("reduction", C.c_int32), ("sft", C.c_int32),
                ("traj_loss_tokens", C.c_void_p), ("n_active_traj", C.c_void_p), ("adv_index", C.c_void_p),
                ("num_adv", C.c_int64), ("num_traj", C.c_int64)]


OTK_TOKEN_MEAN, OTK_SEQ_MEAN_TOKEN_MEAN, OTK_SEQ_MEAN_TOKEN_SUM = 0, 1, 2


class otk_vocab_shard(C.Structure):
    _fields_ = [("vocab_start", C.c_int64), ("vocab_total", C.c_int64)]


OTK_VPF_MAX_RANKS = 8
OTK_IPC_HANDLE_BYTES = 64


class otk_vpf_peers(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("rows_cap", C.c_int64),
                ("xchg", C.c_void_p * OTK_VPF_MAX_RANKS), ("max_ctas", C.c_int32)]


class otk_vpf_rank_call(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("vocab_local", C.c_int64), ("logits", C.c_void_p), ("shard", otk_vocab_shard),
                ("peers", C.POINTER(otk_vpf_peers)), ("dlogits", C.c_void_p), ("logp", C.c_void_p),
                ("entropy", C.c_void_p), ("stats", C.c_void_p)]


STATS_FIELDS = ("loss", "n_clipped", "kl_sum", "entropy_sum", "n_tokens")   # otk_loss_stats (5 doubles)

_P = C.c_void_p
_I64 = C.c_int64
_sig = {
    "otk_version": (C.c_int, []),
    "otk_last_error": (C.c_char_p, []),
    "otk_status_string": (C.c_char_p, [C.c_int]),
    "otk_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "otk_ctx_destroy": (C.c_int, [_P]),
    "otk_ctx_check": (C.c_int, [_P, _P]),
    "otk_ctx_launch_count": (_I64, [_P]),
    "otk_build_masks": (C.c_int, [_P, C.POINTER(otk_traj_batch), C.c_int16, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "otk_group_advantages": (C.c_int, [_P, C.c_int32, _P, C.c_int32, _P, _P, _P, C.c_uint32, C.c_double,
                                       _P, _P, _P, _P, _P, _P]),
    "otk_turn_returns": (C.c_int, [_P, C.POINTER(otk_traj_batch), C.c_int32, C.c_int16, _P, _P, _P, C.c_double,
                                   _P, _P, _P]),
    "otk_logprob_entropy_fwd": (C.c_int, [_P, _I64, _I64, _I64, C.c_int, _P, _P, _P, C.c_float, _P, _P, _P, _P]),
    "otk_policy_loss_fwd_bwd": (C.c_int, [_P, _I64, _I64, _I64, C.c_int, _P, _P, _P, _P, _P, _P, _P, _P,
                                          C.POINTER(otk_loss_cfg), _P, _P, _P, _P, _P]),
    "otk_policy_loss_fwd_bwd_host": (C.c_int, [_P, _I64, _I64, _I64, C.c_int, _P, _P, _P, _P, C.c_int32, _P, _P,
                                               _P, _I64, C.POINTER(otk_loss_cfg), _P, _P, _I64]),
    "otk_lmhead_workspace_bytes": (_I64, [_P, _I64, _I64]),
    "otk_lmhead_logprob_fwd": (C.c_int, [_P, _I64, _I64, _I64, _P, _P, _P, _P, C.c_float, _P, _I64, _P, _P, _P, _P]),
    "otk_lmhead_row_partials": (C.c_int, [_P, _I64, _I64, _I64, _P, _P, _P, _P, C.POINTER(otk_vocab_shard), C.c_float,
                                          _P, _I64, _P, _P]),
    "otk_lmhead_loss_workspace_bytes": (_I64, [_P, _I64, _I64, _I64]),
    "otk_lmhead_policy_loss_fwd_bwd": (C.c_int, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                                 C.POINTER(otk_loss_cfg), _P, _I64, _P, _P, _P, _P, _P, _P]),
    "otk_sample_tokens": (C.c_int, [_P, _I64, _I64, _I64, C.c_int, _P, _P, C.c_float, C.c_int32, _P, _P, _P]),
    "otk_row_partials": (C.c_int, [_P, _I64, _I64, _I64, C.c_int, _P, _P, _P, C.POINTER(otk_vocab_shard),
                                   C.c_float, _P, _P]),
    "otk_logprob_entropy_combine": (C.c_int, [_P, _I64, C.c_int32, _P, _P, _P, _P, _P, _P]),
    "otk_policy_loss_fwd_bwd_partials": (C.c_int, [_P, _I64, _I64, _I64, C.c_int, _P, _P, _P, _P, _P, _P, _P,
                                                   _P, C.POINTER(otk_loss_cfg), C.POINTER(otk_vocab_shard),
                                                   C.c_int32, _P, _P, _P, _P, _P, _P]),
    "otk_vpf_xchg_bytes": (_I64, [_I64, C.c_int32]),
    "otk_policy_loss_fwd_bwd_vpf": (C.c_int, [_P, _I64, _I64, _I64, C.c_int, _P, _P, _P, _P, _P, _P, _P, _P,
                                              C.POINTER(otk_loss_cfg), C.POINTER(otk_vocab_shard),
                                              C.POINTER(otk_vpf_peers), _P, _P, _P, _P, _P]),
    "otk_policy_loss_fwd_bwd_vpf_group": (C.c_int, [C.c_int32, C.POINTER(otk_vpf_rank_call), _I64, _I64, C.c_int,
                                                    _P, _P, _P, _P, _P, _P, _P, C.POINTER(otk_loss_cfg), _P]),
    "otk_xchg_alloc": (C.c_int, [_P, _I64, C.POINTER(C.c_void_p)]),
    "otk_xchg_free": (C.c_int, [_P, _P]),
    "otk_ipc_get_handle": (C.c_int, [_P, _P]),
    "otk_ipc_open": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "otk_ipc_close": (C.c_int, [_P]),
    "otk_comm_unique_id": (C.c_int, [_P]),
    "otk_comm_init": (C.c_int, [_P, _P, C.c_int32, C.c_int32]),
    "otk_comm_destroy": (C.c_int, [_P]),
    "otk_comm_size": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "otk_batch_allreduce_i64": (C.c_int, [_P, _P, _I64, _P]),
    "otk_batch_allreduce_f64": (C.c_int, [_P, _P, _I64, _P]),
    "otk_batch_group_advantages": (C.c_int, [_P, C.c_int32, _P, _P, _P, C.c_int32, C.c_uint32, C.c_double,
                                             _P, _P, _P, _P, _P, _P, _P]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sig)


def _check(st: int):
    if st != 0:
        raise OtkError(st, _lib.otk_last_error().decode())


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    return t.data_ptr()


def _dev(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _host(t: torch.Tensor, name: str, dtype, numel: Optional[int]):
    """Marshalling check of a HOST array of the host-buffer entry point (the C side reads numel elements)."""
    if t.is_cuda:
        raise ValueError(f"{name}: the host entry point takes CPU tensors")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} has {t.numel()} elements, expected {numel}")


def _arr(t: Optional[torch.Tensor], name: str, dtype, numel: Optional[int], device, optional: bool = False,
         at_least: bool = False):
    """Marshalling check of a per-row / per-trajectory array: device, contiguity, dtype and size (the kernels
    index these arrays by row, so a short array would be read out of bounds)."""
    if t is None:
        if optional:
            return
        raise ValueError(f"{name} is required")
    _dev(t, name)
    if t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if numel is not None and (t.numel() < numel if at_least else t.numel() != numel):
        raise ValueError(f"{name} has {t.numel()} elements, expected {'>= ' if at_least else ''}{numel}")


def _loss_args(logits, targets, loss_mask, row_traj, adv, old_logp, ref_logp, n_loss, cfg, dlogits, stats):
    _side_args(logits.shape[0], logits.device, targets, loss_mask, row_traj, adv, old_logp, ref_logp, n_loss, cfg,
               stats)
    _dev(dlogits, "dlogits")
    if dlogits.shape != logits.shape or dlogits.dtype != logits.dtype:
        raise ValueError("dlogits must have the logits' shape and dtype")


def _side_args(N, dev, targets, loss_mask, row_traj, adv, old_logp, ref_logp, n_loss, cfg, stats):
    _arr(targets, "targets", torch.int32, N, dev)
    _arr(loss_mask, "loss_mask", torch.uint8, N, dev)
    _arr(row_traj, "row_traj", torch.int32, N, dev)
    _arr(adv, "adv", torch.float64, 1, dev, at_least=True)
    _arr(old_logp, "old_logp", torch.float32, N, dev)
    _arr(ref_logp, "ref_logp", torch.float32, N, dev, optional=True)   # required-ness: the C ABI checks it
    _arr(n_loss, "n_loss", torch.int64, 1, dev)
    _arr(stats, "stats", torch.float64, len(STATS_FIELDS), dev)
    _arr(cfg.adv_index, "cfg.adv_index", torch.int32, N, dev, optional=True)
    _arr(cfg.traj_loss_tokens, "cfg.traj_loss_tokens", torch.int64, None, dev, optional=True)
    _arr(cfg.n_active_traj, "cfg.n_active_traj", torch.int64, 1, dev, optional=True)


def _stream(stream) -> Optional[int]:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return OTK_BF16
    if t.dtype == torch.float32:
        return OTK_F32
    raise ValueError("logits must be bfloat16 or float32")


@dataclass
class LossCfg:
    clip_low: float = 0.2
    clip_high: float = 0.2
    kl_beta: float = 0.04
    kl_type: int = OTK_KL_K3
    log_ratio_clamp: float = 20.0
    logit_scale: float = 1.0
    zero_masked_rows: bool = True
    accumulate_stats: bool = False
    ent_coef: float = 0.0                  # entropy bonus (NEXT-4)
    dual_clip: float = 0.0                 # dual-clip c > 1 (0 = off)
    reduction: int = 0                     # OTK_TOKEN_MEAN | OTK_SEQ_MEAN_TOKEN_MEAN | OTK_SEQ_MEAN_TOKEN_SUM
    sft: bool = False                      # supervised mode
    traj_loss_tokens: Optional[torch.Tensor] = None   # device i64 [B] (sequence-mean reductions)
    n_active_traj: Optional[torch.Tensor] = None      # device i64 [1] (sequence-mean reductions, global)
    adv_index: Optional[torch.Tensor] = None          # device i32 [num_rows]: A_j = adv[adv_index[j]] (turn level)

    def c(self, accumulate: Optional[bool] = None, adv: Optional[torch.Tensor] = None) -> otk_loss_cfg:
        """The C struct; `adv` (the advantage array of the call) gives num_adv, the kernels' index bound."""
        acc = self.accumulate_stats if accumulate is None else accumulate
        return otk_loss_cfg(self.clip_low, self.clip_high, self.kl_beta, self.log_ratio_clamp, self.logit_scale,
                            int(self.kl_type), int(bool(self.zero_masked_rows)), int(bool(acc)), 0,
                            float(self.ent_coef), float(self.dual_clip), int(self.reduction), int(bool(self.sft)),
                            _ptr(self.traj_loss_tokens), _ptr(self.n_active_traj), _ptr(self.adv_index),
                            int(adv.numel()) if adv is not None else 0,
                            int(self.traj_loss_tokens.numel()) if self.traj_loss_tokens is not None else 0)


class Context:
    """Owns an otk_ctx (sticky error word, reduction scratch, staging) on one CUDA device."""

    def __init__(self, device: Optional[int] = None):
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        h = C.c_void_p()
        _check(_lib.otk_ctx_create(self.device, C.byref(h)))
        self.handle = h

    def check(self, stream=None):
        """Synchronise `stream` and raise OtkError for a device-side data error since the last check."""
        _check(_lib.otk_ctx_check(self.handle, _stream(stream)))

    @property
    def launches(self) -> int:
        return int(_lib.otk_ctx_launch_count(self.handle))

    def close(self):
        if self.handle:
            _lib.otk_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------------------------------------
# trajectories on the device
# ------------------------------------------------------------------------------------------------
@dataclass
class DeviceTrajBatch:
    tok_offsets: torch.Tensor
    seg_offsets: torch.Tensor
    seg_source: torch.Tensor
    seg_agent: torch.Tensor
    seg_len: torch.Tensor
    terminated: Optional[torch.Tensor]
    traj_agent: Optional[torch.Tensor]
    num_traj: int
    num_rows: int

    def c(self) -> otk_traj_batch:
        return otk_traj_batch(self.num_traj, self.num_rows, _ptr(self.tok_offsets), _ptr(self.seg_offsets),
                              _ptr(self.seg_source), _ptr(self.seg_agent), _ptr(self.seg_len),
                              _ptr(self.terminated), _ptr(self.traj_agent))


def traj_batch_to_device(tb, device="cuda", non_blocking=False) -> DeviceTrajBatch:
    """Copy a host segment CSR (any object with the otk_traj_batch fields as numpy arrays) to `device`."""
    def t(a, dt):
        if a is None:
            return None
        x = torch.as_tensor(a).to(dt)
        return x.to(device, non_blocking=non_blocking)
    return DeviceTrajBatch(
        tok_offsets=t(tb.tok_offsets, torch.int64), seg_offsets=t(tb.seg_offsets, torch.int32),
        seg_source=t(tb.seg_source, torch.uint8), seg_agent=t(tb.seg_agent, torch.int16),
        seg_len=t(tb.seg_len, torch.int32), terminated=t(tb.terminated, torch.uint8),
        traj_agent=t(getattr(tb, "traj_agent", None), torch.int16),
        num_traj=int(len(tb.tok_offsets) - 1), num_rows=int(tb.tok_offsets[-1]))


# ------------------------------------------------------------------------------------------------
# (1) masks
# ------------------------------------------------------------------------------------------------
def otk_build_masks(ctx: Context, batch: DeviceTrajBatch, train_agent: int = OTK_ANY_AGENT, *,
                    response_mask: bool = True, source_counts: bool = True, row_seg: bool = False,
                    out: Optional[dict] = None, stream=None) -> dict:
    dev = batch.tok_offsets.device
    N, B = batch.num_rows, batch.num_traj
    o = out if out is not None else {}
    o.setdefault("loss_mask", torch.empty(N, dtype=torch.uint8, device=dev))
    if response_mask:
        o.setdefault("response_mask", torch.empty(N, dtype=torch.uint8, device=dev))
    o.setdefault("row_traj", torch.empty(N, dtype=torch.int32, device=dev))
    o.setdefault("traj_loss_tokens", torch.empty(B, dtype=torch.int64, device=dev))
    if source_counts:
        o.setdefault("traj_source_counts", torch.empty((B, 4), dtype=torch.int64, device=dev))
    o.setdefault("n_loss", torch.empty(1, dtype=torch.int64, device=dev))
    o.setdefault("n_active_traj", torch.empty(1, dtype=torch.int64, device=dev))
    if row_seg:
        o.setdefault("row_seg", torch.empty(N, dtype=torch.int32, device=dev))
    cb = batch.c()
    _check(_lib.otk_build_masks(ctx.handle, C.byref(cb), train_agent, _ptr(o["loss_mask"]),
                                _ptr(o.get("response_mask")), _ptr(o["row_traj"]), _ptr(o["traj_loss_tokens"]),
                                _ptr(o.get("traj_source_counts")), _ptr(o["n_loss"]), _ptr(o["n_active_traj"]),
                                _ptr(o.get("row_seg")), _stream(stream)))
    return o


# ------------------------------------------------------------------------------------------------
# (2) advantages
# ------------------------------------------------------------------------------------------------
def otk_group_advantages(ctx: Context, group_id: torch.Tensor, num_groups: int, *,
                         returns: Optional[torch.Tensor] = None, turn_offsets: Optional[torch.Tensor] = None,
                         turn_rewards: Optional[torch.Tensor] = None, std_norm: bool = True,
                         unbiased: bool = False, std_floor: float = 1e-8, skip_ungrouped: bool = False,
                         out: Optional[dict] = None, stream=None) -> dict:
    _dev(group_id, "group_id")
    B = int(group_id.numel())
    dev = group_id.device
    _arr(group_id, "group_id", torch.int32, B, dev)
    _arr(returns, "returns", torch.float64, B, dev, optional=True)
    _arr(turn_offsets, "turn_offsets", torch.int32, B + 1, dev, optional=True)
    _arr(turn_rewards, "turn_rewards", torch.float64, None, dev, optional=True)
    o = out if out is not None else {}
    o.setdefault("adv", torch.empty(B, dtype=torch.float64, device=dev))
    o.setdefault("returns", torch.empty(B, dtype=torch.float64, device=dev))
    o.setdefault("group_mean", torch.empty(num_groups, dtype=torch.float64, device=dev))
    o.setdefault("group_std", torch.empty(num_groups, dtype=torch.float64, device=dev))
    o.setdefault("group_size", torch.empty(num_groups, dtype=torch.int32, device=dev))
    flags = ((OTK_ADV_STD_NORM if std_norm else 0) | (OTK_ADV_UNBIASED if unbiased else 0)
             | (OTK_ADV_SKIP_UNGROUPED if skip_ungrouped else 0))
    _check(_lib.otk_group_advantages(ctx.handle, B, _ptr(group_id), int(num_groups), _ptr(returns),
                                     _ptr(turn_offsets), _ptr(turn_rewards), flags, float(std_floor),
                                     _ptr(o["adv"]), _ptr(o["returns"]), _ptr(o["group_mean"]),
                                     _ptr(o["group_std"]), _ptr(o["group_size"]), _stream(stream)))
    return o


# ------------------------------------------------------------------------------------------------
# batch sharding over NCCL (otk.h "Batch sharding"; SURVEY.md §8(e) BATCH)
# ------------------------------------------------------------------------------------------------
def otk_comm_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) on one rank; the caller hands it to every rank."""
    buf = (C.c_ubyte * 128)()
    _check(_lib.otk_comm_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def otk_comm_init(ctx: Context, uid: bytes, nranks: int, rank: int) -> None:
    if len(uid) != 128:
        raise ValueError("uid must be the 128 bytes of otk_comm_unique_id")
    buf = (C.c_ubyte * 128).from_buffer_copy(uid)
    _check(_lib.otk_comm_init(ctx.handle, C.cast(buf, C.c_void_p), int(nranks), int(rank)))


def otk_comm_destroy(ctx: Context) -> None:
    _check(_lib.otk_comm_destroy(ctx.handle))


def otk_comm_size(ctx: Context) -> Tuple[int, int]:
    n, r = C.c_int32(), C.c_int32()
    _check(_lib.otk_comm_size(ctx.handle, C.byref(n), C.byref(r)))
    return n.value, r.value


def otk_batch_allreduce_i64(ctx: Context, buf: torch.Tensor, stream=None) -> torch.Tensor:
    _arr(buf, "buf", torch.int64, None, buf.device)
    _check(_lib.otk_batch_allreduce_i64(ctx.handle, _ptr(buf), int(buf.numel()), _stream(stream)))
    return buf


def otk_batch_allreduce_f64(ctx: Context, buf: torch.Tensor, stream=None) -> torch.Tensor:
    _arr(buf, "buf", torch.float64, None, buf.device)
    _check(_lib.otk_batch_allreduce_f64(ctx.handle, _ptr(buf), int(buf.numel()), _stream(stream)))
    return buf


def otk_batch_group_advantages(ctx: Context, group_id: torch.Tensor, returns: torch.Tensor, counts: Sequence[int],
                               num_groups: int, *, std_norm: bool = True, unbiased: bool = False,
                               std_floor: float = 1e-8, skip_ungrouped: bool = False, out: Optional[dict] = None,
                               stream=None) -> dict:
    """Step (2) over the global batch of a batch-sharded step: every rank's (group_id, return) gathered in rank
    order over NCCL, then the group statistics on the whole batch (identical on every rank). `counts` = host list
    of trajectories per rank. Returns gid_all, ret_all, adv_all (global), adv (this rank's slice) and the stats."""
    dev = group_id.device
    B = int(group_id.numel())
    counts = [int(c) for c in counts]
    total = sum(counts)
    _arr(group_id, "group_id", torch.int32, B, dev)
    _arr(returns, "returns", torch.float64, B, dev)
    o = out if out is not None else {}
    o.setdefault("gid_all", torch.empty(total, dtype=torch.int32, device=dev))
    o.setdefault("ret_all", torch.empty(total, dtype=torch.float64, device=dev))
    o.setdefault("adv_all", torch.empty(total, dtype=torch.float64, device=dev))
    o.setdefault("group_mean", torch.empty(num_groups, dtype=torch.float64, device=dev))
    o.setdefault("group_std", torch.empty(num_groups, dtype=torch.float64, device=dev))
    o.setdefault("group_size", torch.empty(num_groups, dtype=torch.int32, device=dev))
    for k in ("gid_all", "ret_all", "adv_all"):
        _arr(o[k], k, o[k].dtype, total, dev)
    flags = ((OTK_ADV_STD_NORM if std_norm else 0) | (OTK_ADV_UNBIASED if unbiased else 0)
             | (OTK_ADV_SKIP_UNGROUPED if skip_ungrouped else 0))
    cnt = (C.c_int32 * len(counts))(*counts)
    _check(_lib.otk_batch_group_advantages(ctx.handle, B, _ptr(group_id), _ptr(returns), C.cast(cnt, C.c_void_p),
                                           int(num_groups), flags, float(std_floor), _ptr(o["gid_all"]),
                                           _ptr(o["ret_all"]), _ptr(o["adv_all"]), _ptr(o["group_mean"]),
                                           _ptr(o["group_std"]), _ptr(o["group_size"]), _stream(stream)))
    _, rank = otk_comm_size(ctx)
    b0 = sum(counts[:rank])
    o["adv"] = o["adv_all"][b0:b0 + B]
    return o


def otk_turn_returns(ctx: Context, batch: DeviceTrajBatch, num_segments: int, group_id: torch.Tensor,
                     turn_offsets: torch.Tensor, turn_rewards: torch.Tensor, gamma: float = 1.0,
                     train_agent: int = OTK_ANY_AGENT, *, out: Optional[dict] = None, stream=None) -> dict:
    """(2') turn-level credit: per-segment reward-to-go of the trainable ACTION turns (otk.h otk_turn_returns)."""
    dev = batch.seg_offsets.device
    _arr(group_id, "group_id", torch.int32, batch.num_traj, dev)
    _arr(turn_offsets, "turn_offsets", torch.int32, batch.num_traj + 1, dev)
    _arr(turn_rewards, "turn_rewards", torch.float64, None, dev)
    o = out if out is not None else {}
    o.setdefault("seg_return", torch.empty(num_segments, dtype=torch.float64, device=dev))
    o.setdefault("seg_group", torch.empty(num_segments, dtype=torch.int32, device=dev))
    cb = batch.c()
    _check(_lib.otk_turn_returns(ctx.handle, C.byref(cb), int(num_segments), int(train_agent), _ptr(group_id),
                                 _ptr(turn_offsets), _ptr(turn_rewards), float(gamma), _ptr(o["seg_return"]),
                                 _ptr(o["seg_group"]), _stream(stream)))
    return o


# ------------------------------------------------------------------------------------------------
# LM head fused with (3) (NEXT-1, forward)
# ------------------------------------------------------------------------------------------------
def otk_lmhead_logprob_fwd(ctx: Context, hidden: torch.Tensor, weight: torch.Tensor, targets: torch.Tensor, *,
                           row_mask: Optional[torch.Tensor] = None, logit_scale: float = 1.0,
                           workspace: Optional[torch.Tensor] = None, want_lse: bool = False,
                           out: Optional[dict] = None, stream=None) -> dict:
    """logp / entropy of z = logit_scale * hidden @ weight.T without materialising z (otk.h)."""
    for t, n in ((hidden, "hidden"), (weight, "weight"), (targets, "targets")):
        _dev(t, n)
    if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise ValueError("hidden and weight must be bfloat16")
    N, d = hidden.shape
    V, d2 = weight.shape
    if d != d2:
        raise ValueError("hidden / weight inner dimensions differ")
    _arr(targets, "targets", torch.int32, N, hidden.device)
    _arr(row_mask, "row_mask", torch.uint8, N, hidden.device, optional=True)
    nbytes = int(_lib.otk_lmhead_workspace_bytes(ctx.handle, N, V))
    if workspace is None or workspace.numel() * workspace.element_size() < nbytes:
        workspace = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=hidden.device)
    o = out if out is not None else {}
    o.setdefault("logp", torch.empty(N, dtype=torch.float32, device=hidden.device))
    o.setdefault("entropy", torch.empty(N, dtype=torch.float32, device=hidden.device))
    if want_lse:
        o.setdefault("lse", torch.empty(N, dtype=torch.float32, device=hidden.device))
    _check(_lib.otk_lmhead_logprob_fwd(ctx.handle, N, d, V, _ptr(hidden), _ptr(weight), _ptr(targets),
                                       _ptr(row_mask), float(logit_scale), _ptr(workspace),
                                       workspace.numel() * workspace.element_size(), _ptr(o["logp"]),
                                       _ptr(o["entropy"]), _ptr(o.get("lse")), _stream(stream)))
    o["workspace"] = workspace
    return o


def otk_lmhead_policy_loss_fwd_bwd(ctx: Context, hidden: torch.Tensor, weight: torch.Tensor, targets: torch.Tensor,
                                   loss_mask: torch.Tensor, row_traj: torch.Tensor, adv: torch.Tensor,
                                   old_logp: torch.Tensor, ref_logp: Optional[torch.Tensor], n_loss: torch.Tensor,
                                   cfg: LossCfg = LossCfg(), *, workspace: Optional[torch.Tensor] = None,
                                   dhidden: Optional[torch.Tensor] = None, dweight: Optional[torch.Tensor] = None,
                                   want_logp: bool = True, stats: Optional[torch.Tensor] = None,
                                   accumulate: Optional[bool] = None, stream=None) -> dict:
    """Loss, dh and dW through the LM head, x = hidden @ weight.T (otk.h NEXT-1 fwd + bwd). workspace / dhidden /
    dweight are reused when passed; lmhead_x_from_workspace() reads the bf16 x the call left in the workspace."""
    for t, n in ((hidden, "hidden"), (weight, "weight")):
        _dev(t, n)
    if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise ValueError("hidden and weight must be bfloat16")
    N, d = hidden.shape
    V, d2 = weight.shape
    if d != d2:
        raise ValueError("hidden / weight inner dimensions differ")
    dev = hidden.device
    if dhidden is None:
        dhidden = torch.empty_like(hidden)
    if dweight is None:
        dweight = torch.empty_like(weight)
    for t, n, shp in ((dhidden, "dhidden", (N, d)), (dweight, "dweight", (V, d))):
        _dev(t, n)
        if tuple(t.shape) != shp or t.dtype != torch.bfloat16:
            raise ValueError(f"{n} must be bfloat16 {shp}")
    if stats is None:
        stats = torch.zeros(len(STATS_FIELDS), dtype=torch.float64, device=dev)
    logp = torch.empty(N, dtype=torch.float32, device=dev) if want_logp else None
    entropy = torch.empty(N, dtype=torch.float32, device=dev) if want_logp else None
    _side_args(N, dev, targets, loss_mask, row_traj, adv, old_logp, ref_logp, n_loss, cfg, stats)
    nbytes = max(int(_lib.otk_lmhead_loss_workspace_bytes(ctx.handle, N, d, V)), 16)  # -1: the call reports why
    if workspace is None or workspace.numel() * workspace.element_size() < nbytes:
        workspace = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
    c = cfg.c(accumulate, adv)
    _check(_lib.otk_lmhead_policy_loss_fwd_bwd(ctx.handle, N, d, V, _ptr(hidden), _ptr(weight), _ptr(targets),
                                               _ptr(loss_mask), _ptr(row_traj), _ptr(adv), _ptr(old_logp),
                                               _ptr(ref_logp), _ptr(n_loss), C.byref(c), _ptr(workspace),
                                               workspace.numel() * workspace.element_size(), _ptr(dhidden),
                                               _ptr(dweight), _ptr(logp), _ptr(entropy), _ptr(stats),
                                               _stream(stream)))
    return dict(workspace=workspace, dh=dhidden, dW=dweight, logp=logp, entropy=entropy, stats=stats,
                shape=(N, V))


def lmhead_x_from_workspace(out: dict) -> torch.Tensor:
    """The bf16 x = h W^T that otk_lmhead_policy_loss_fwd_bwd left at the start of its workspace, un-tiled to
    [N, V] (a copy; otk.h: 64 x 64 tiles [rows_pad/64][cols_pad/64][64][64])."""
    N, V = out["shape"]
    rp, cp = (N + 255) // 256 * 256, (V + 255) // 256 * 256
    t = out["workspace"][: rp * cp * 2].view(torch.bfloat16).view(rp // 64, cp // 64, 64, 64)
    return t.permute(0, 2, 1, 3).reshape(rp, cp)[:N, :V].contiguous()


def otk_lmhead_row_partials(ctx: Context, hidden: torch.Tensor, weight_shard: torch.Tensor, targets: torch.Tensor,
                            vocab_start: int, vocab_total: int, *, row_mask: Optional[torch.Tensor] = None,
                            logit_scale: float = 1.0, workspace: Optional[torch.Tensor] = None,
                            partials: Optional[torch.Tensor] = None, stream=None):
    """This rank's [N, 4] partials of a vocab-sharded LM head (otk.h otk_lmhead_row_partials); returns
    (partials, workspace)."""
    for t, n in ((hidden, "hidden"), (weight_shard, "weight_shard"), (targets, "targets")):
        _dev(t, n)
    N, d = hidden.shape
    Vl = weight_shard.shape[0]
    if weight_shard.shape[1] != d or hidden.dtype != torch.bfloat16 or weight_shard.dtype != torch.bfloat16:
        raise ValueError("hidden [N, d] and weight_shard [V_local, d] must be bfloat16 with the same d")
    _arr(targets, "targets", torch.int32, N, hidden.device)
    _arr(row_mask, "row_mask", torch.uint8, N, hidden.device, optional=True)
    nbytes = int(_lib.otk_lmhead_workspace_bytes(ctx.handle, N, Vl))
    if workspace is None or workspace.numel() * workspace.element_size() < nbytes:
        workspace = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=hidden.device)
    if partials is None:
        partials = torch.empty((N, 4), dtype=torch.float32, device=hidden.device)
    sh = otk_vocab_shard(int(vocab_start), int(vocab_total))
    _check(_lib.otk_lmhead_row_partials(ctx.handle, N, d, Vl, _ptr(hidden), _ptr(weight_shard), _ptr(targets),
                                        _ptr(row_mask), C.byref(sh), float(logit_scale), _ptr(workspace),
                                        workspace.numel() * workspace.element_size(), _ptr(partials),
                                        _stream(stream)))
    return partials, workspace


# ------------------------------------------------------------------------------------------------
# rollout sampling (NEXT-3)
# ------------------------------------------------------------------------------------------------
def otk_sample_tokens(ctx: Context, logits: torch.Tensor, uniforms: Optional[torch.Tensor] = None, *,
                      logit_scale: float = 1.0, greedy: bool = False, vocab: Optional[int] = None,
                      temperature: Optional[float] = None, want_logp: bool = True, out: Optional[dict] = None,
                      stream=None) -> dict:
    """One token per row: inverse-transform draw from softmax(logit_scale * x) with the caller's uniforms,
    or the greedy argmax (otk.h otk_sample_tokens). temperature (optional) sets logit_scale = 1/temperature;
    below 1e-6 it means greedy."""
    if temperature is not None:
        if temperature < 1e-6:
            greedy = True
        else:
            logit_scale = 1.0 / float(temperature)
    _dev(logits, "logits")
    N, ld = logits.shape
    V = ld if vocab is None else int(vocab)
    if not greedy:
        if uniforms is None:
            raise ValueError("uniforms are required unless greedy")
        _dev(uniforms, "uniforms")
        _arr(uniforms, "uniforms", torch.float32, N, logits.device)
    o = out if out is not None else {}
    o.setdefault("tokens", torch.empty(N, dtype=torch.int32, device=logits.device))
    if want_logp:
        o.setdefault("logp", torch.empty(N, dtype=torch.float32, device=logits.device))
    _check(_lib.otk_sample_tokens(ctx.handle, N, V, ld, _dtype_code(logits), _ptr(logits),
                                  _ptr(uniforms) if not greedy else None, float(logit_scale), int(bool(greedy)),
                                  _ptr(o["tokens"]), _ptr(o.get("logp")), _stream(stream)))
    return o


# ------------------------------------------------------------------------------------------------
# (3) forward
# ------------------------------------------------------------------------------------------------
def otk_logprob_entropy_fwd(ctx: Context, logits: torch.Tensor, targets: torch.Tensor, *,
                            vocab: Optional[int] = None, row_mask: Optional[torch.Tensor] = None,
                            logit_scale: float = 1.0, want_lse: bool = False, out: Optional[dict] = None,
                            stream=None) -> dict:
    _dev(logits, "logits")
    N, ld = logits.shape
    V = ld if vocab is None else int(vocab)
    dev = logits.device
    _arr(targets, "targets", torch.int32, N, dev)
    _arr(row_mask, "row_mask", torch.uint8, N, dev, optional=True)
    o = out if out is not None else {}
    o.setdefault("logp", torch.empty(N, dtype=torch.float32, device=dev))
    o.setdefault("entropy", torch.empty(N, dtype=torch.float32, device=dev))
    if want_lse:
        o.setdefault("lse", torch.empty(N, dtype=torch.float32, device=dev))
    _check(_lib.otk_logprob_entropy_fwd(ctx.handle, N, V, ld, _dtype_code(logits), _ptr(logits), _ptr(targets),
                                        _ptr(row_mask), float(logit_scale), _ptr(o["logp"]), _ptr(o.get("entropy")),
                                        _ptr(o.get("lse")), _stream(stream)))
    return o


# ------------------------------------------------------------------------------------------------
# (4) loss forward + fused backward
# ------------------------------------------------------------------------------------------------
def otk_policy_loss_fwd_bwd(ctx: Context, logits: torch.Tensor, targets: torch.Tensor, loss_mask: torch.Tensor,
                            row_traj: torch.Tensor, adv: torch.Tensor, old_logp: torch.Tensor,
                            ref_logp: Optional[torch.Tensor], n_loss: torch.Tensor, cfg: LossCfg = LossCfg(), *,
                            vocab: Optional[int] = None, dlogits: Optional[torch.Tensor] = None,
                            logp: Optional[torch.Tensor] = None, entropy: Optional[torch.Tensor] = None,
                            stats: Optional[torch.Tensor] = None, accumulate: Optional[bool] = None,
                            want_logp: bool = True, stream=None) -> dict:
    _dev(logits, "logits")
    N, ld = logits.shape
    V = ld if vocab is None else int(vocab)
    dev = logits.device
    if dlogits is None:
        dlogits = torch.empty_like(logits)
    if want_logp and logp is None:
        logp = torch.empty(N, dtype=torch.float32, device=dev)
    if want_logp and entropy is None:
        entropy = torch.empty(N, dtype=torch.float32, device=dev)
    if stats is None:
        stats = torch.zeros(len(STATS_FIELDS), dtype=torch.float64, device=dev)
    _loss_args(logits, targets, loss_mask, row_traj, adv, old_logp, ref_logp, n_loss, cfg, dlogits, stats)
    c = cfg.c(accumulate, adv)
    _check(_lib.otk_policy_loss_fwd_bwd(ctx.handle, N, V, ld, _dtype_code(logits), _ptr(logits), _ptr(targets),
                                        _ptr(loss_mask), _ptr(row_traj), _ptr(adv), _ptr(old_logp),
                                        _ptr(ref_logp), _ptr(n_loss), C.byref(c), _ptr(dlogits), _ptr(logp),
                                        _ptr(entropy), _ptr(stats), _stream(stream)))
    return dict(dlogits=dlogits, logp=logp, entropy=entropy, stats=stats)


def otk_policy_loss_fwd_bwd_host(ctx: Context, logits: torch.Tensor, targets, loss_mask, row_traj, adv, old_logp,
                                 ref_logp, n_loss: int, cfg: LossCfg = LossCfg(), *, vocab: Optional[int] = None,
                                 dlogits: Optional[torch.Tensor] = None, rows_per_chunk: int = 4096):
    """Host-buffer entry point: every tensor is a CPU (ideally pinned) tensor; returns the stats dict.
    dlogits (CPU, same shape / dtype as logits) receives the gradient (trainable rows only when
    cfg.zero_masked_rows is False)."""
    N, ld = logits.shape
    V = ld if vocab is None else int(vocab)
    _host(logits, "logits", logits.dtype, N * ld)
    if logits.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("logits must be float32 or bfloat16")
    _host(targets, "targets", torch.int32, N)
    _host(loss_mask, "loss_mask", torch.uint8, N)
    _host(row_traj, "row_traj", torch.int32, N)
    _host(adv, "adv", torch.float64, None)
    if adv.numel() < 1:
        raise ValueError("adv must hold >= 1 trajectory")
    _host(old_logp, "old_logp", torch.float32, N)
    if ref_logp is not None:
        _host(ref_logp, "ref_logp", torch.float32, N)
    if dlogits is not None:
        _host(dlogits, "dlogits", logits.dtype, N * ld)
    stats = (C.c_double * len(STATS_FIELDS))()
    c = cfg.c(False, adv)
    _check(_lib.otk_policy_loss_fwd_bwd_host(ctx.handle, N, V, ld, _dtype_code(logits), _ptr(logits), _ptr(targets),
                                             _ptr(loss_mask), _ptr(row_traj), int(adv.numel()), _ptr(adv),
                                             _ptr(old_logp), _ptr(ref_logp), int(n_loss), C.byref(c),
                                             _ptr(dlogits), C.cast(stats, C.c_void_p), int(rows_per_chunk)))
    return dict(zip(STATS_FIELDS, list(stats)))


def stats_dict(stats: torch.Tensor) -> dict:
    return dict(zip(STATS_FIELDS, stats.detach().cpu().tolist()))


# ------------------------------------------------------------------------------------------------
# vocab sharding
# ------------------------------------------------------------------------------------------------
def otk_row_partials(ctx: Context, logits: torch.Tensor, targets: torch.Tensor, vocab_start: int, vocab_total: int,
                     *, vocab_local: Optional[int] = None, row_mask: Optional[torch.Tensor] = None,
                     logit_scale: float = 1.0, partials: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    _dev(logits, "logits")
    N, ld = logits.shape
    V = ld if vocab_local is None else int(vocab_local)
    _arr(targets, "targets", torch.int32, N, logits.device)
    _arr(row_mask, "row_mask", torch.uint8, N, logits.device, optional=True)
    if partials is None:
        partials = torch.empty((N, 4), dtype=torch.float32, device=logits.device)
    _arr(partials, "partials", torch.float32, 4 * N, logits.device)
    sh = otk_vocab_shard(int(vocab_start), int(vocab_total))
    _check(_lib.otk_row_partials(ctx.handle, N, V, ld, _dtype_code(logits), _ptr(logits), _ptr(targets),
                                 _ptr(row_mask), C.byref(sh), float(logit_scale), _ptr(partials), _stream(stream)))
    return partials


def otk_logprob_entropy_combine(ctx: Context, partials: torch.Tensor, *, row_mask: Optional[torch.Tensor] = None,
                                want_lse: bool = False, stream=None) -> dict:
    """partials: [nshards, N, 4] float32 (rank order)."""
    _dev(partials, "partials")
    if partials.dim() != 3 or partials.shape[2] != 4 or partials.dtype != torch.float32:
        raise ValueError("partials must be float32 [nshards, N, 4]")
    P, N, _ = partials.shape
    dev = partials.device
    _arr(row_mask, "row_mask", torch.uint8, N, dev, optional=True)
    o = dict(logp=torch.empty(N, dtype=torch.float32, device=dev),
             entropy=torch.empty(N, dtype=torch.float32, device=dev))
    if want_lse:
        o["lse"] = torch.empty(N, dtype=torch.float32, device=dev)
    _check(_lib.otk_logprob_entropy_combine(ctx.handle, N, P, _ptr(partials), _ptr(row_mask), _ptr(o["logp"]),
                                            _ptr(o["entropy"]), _ptr(o.get("lse")), _stream(stream)))
    return o


def otk_policy_loss_fwd_bwd_partials(ctx: Context, logits: torch.Tensor, targets, loss_mask, row_traj, adv,
                                     old_logp, ref_logp, n_loss, cfg: LossCfg, vocab_start: int, vocab_total: int,
                                     partials: torch.Tensor, *, vocab_local: Optional[int] = None,
                                     dlogits: Optional[torch.Tensor] = None, logp=None, entropy=None, stats=None,
                                     accumulate: Optional[bool] = None, stream=None) -> dict:
    _dev(logits, "logits")
    N, ld = logits.shape
    V = ld if vocab_local is None else int(vocab_local)
    dev = logits.device
    if dlogits is None:
        dlogits = torch.empty_like(logits)
    if logp is None:
        logp = torch.empty(N, dtype=torch.float32, device=dev)
    if entropy is None:
        entropy = torch.empty(N, dtype=torch.float32, device=dev)
    if stats is None:
        stats = torch.zeros(len(STATS_FIELDS), dtype=torch.float64, device=dev)
    _loss_args(logits, targets, loss_mask, row_traj, adv, old_logp, ref_logp, n_loss, cfg, dlogits, stats)
    if partials.dim() != 3 or partials.shape[1:] != (N, 4) or partials.dtype != torch.float32:
        raise ValueError("partials must be float32 [nshards, N, 4]")
    sh = otk_vocab_shard(int(vocab_start), int(vocab_total))
    c = cfg.c(accumulate, adv)
    _check(_lib.otk_policy_loss_fwd_bwd_partials(
        ctx.handle, N, V, ld, _dtype_code(logits), _ptr(logits), _ptr(targets), _ptr(loss_mask), _ptr(row_traj),
        _ptr(adv), _ptr(old_logp), _ptr(ref_logp), _ptr(n_loss), C.byref(c), C.byref(sh), int(partials.shape[0]),
        _ptr(partials), _ptr(dlogits), _ptr(logp), _ptr(entropy), _ptr(stats), _stream(stream)))
    return dict(dlogits=dlogits, logp=logp, entropy=entropy, stats=stats)


# ---- K4-VPF: vocab-sharded (4) with the row-partial exchange inside the kernel (otk.h otk_policy_loss_fwd_bwd_vpf)
def otk_vpf_xchg_bytes(rows_cap: int, nranks: int) -> int:
    n = int(_lib.otk_vpf_xchg_bytes(int(rows_cap), int(nranks)))
    if n < 0:
        raise ValueError("otk_vpf_xchg_bytes: bad rows_cap / nranks")
    return n


def otk_xchg_alloc(ctx: "Context", nbytes: int) -> int:
    out = C.c_void_p()
    _check(_lib.otk_xchg_alloc(ctx.handle, int(nbytes), C.byref(out)))
    return int(out.value)


def otk_xchg_free(ctx: "Context", ptr: int):
    _check(_lib.otk_xchg_free(ctx.handle, C.c_void_p(int(ptr))))


def otk_ipc_get_handle(ptr: int) -> bytes:
    h = C.create_string_buffer(OTK_IPC_HANDLE_BYTES)
    _check(_lib.otk_ipc_get_handle(C.c_void_p(int(ptr)), h))
    return h.raw


def otk_ipc_open(handle: bytes) -> int:
    if len(handle) != OTK_IPC_HANDLE_BYTES:
        raise ValueError("IPC handle must be OTK_IPC_HANDLE_BYTES bytes")
    out = C.c_void_p()
    _check(_lib.otk_ipc_open(C.create_string_buffer(bytes(handle), OTK_IPC_HANDLE_BYTES), C.byref(out)))
    return int(out.value)


def otk_ipc_close(ptr: int):
    _check(_lib.otk_ipc_close(C.c_void_p(int(ptr))))


class VpfExchange:
    """One rank's view of the K4-VPF exchange buffers: the device address of every rank's buffer as seen from
    this process (ptrs[rank] = own buffer from otk_xchg_alloc; peers' mapped with otk_ipc_open, or — ranks sharing
    one GPU — the peers' own buffers). The per-call epoch lives on the device (own buffer tail, bumped by the kernel),
    so calls are CUDA-graph capturable; all ranks must make the same sequence of calls.
    close() unmaps the opened peers and frees the owned buffer."""

    def __init__(self, rank: int, nranks: int, rows_cap: int, ptrs, *, max_ctas: int = 0, opened=(),
                 owner: Optional["Context"] = None):
        if not (0 <= rank < nranks <= OTK_VPF_MAX_RANKS) or len(ptrs) != nranks:
            raise ValueError("need 0 <= rank < nranks <= OTK_VPF_MAX_RANKS and one pointer per rank")
        self.rank, self.nranks, self.rows_cap = rank, nranks, int(rows_cap)
        self.ptrs, self.max_ctas, self.opened = [int(x) for x in ptrs], int(max_ctas), list(opened)
        self.owner = owner

    @staticmethod
    def local_group(ctxs, rows_cap: int, max_ctas: int = 0):
        """Exchanges of len(ctxs) ranks that share ONE process (e.g. ranks co-scheduled on one GPU, each with
        its own ctx and stream): plain device buffers, no IPC."""
        P = len(ctxs)
        ptrs = [otk_xchg_alloc(c, otk_vpf_xchg_bytes(rows_cap, P)) for c in ctxs]
        return [VpfExchange(r, P, rows_cap, ptrs, max_ctas=max_ctas, owner=ctxs[r]) for r in range(P)]

    def peers(self) -> otk_vpf_peers:
        pp = otk_vpf_peers(self.rank, self.nranks, self.rows_cap)
        for q, a in enumerate(self.ptrs):
            pp.xchg[q] = a
        pp.max_ctas = self.max_ctas
        return pp

    def close(self):
        for a in self.opened:
            otk_ipc_close(a)
        self.opened = []
        if self.owner is not None:
            otk_xchg_free(self.owner, self.ptrs[self.rank])
            self.owner = None


def _row_view(t: torch.Tensor, name: str):
    """(rows, ld) of a 2-D row-major tensor whose rows may be a column slice of a wider buffer (stride(1) == 1)."""
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dim() != 2 or t.stride(1) != 1 or (t.shape[0] > 1 and t.stride(0) < t.shape[1]):
        raise ValueError(f"{name} must be 2-D with unit column stride")
    return t.shape[0], (t.stride(0) if t.shape[0] > 1 else t.shape[1])


def otk_policy_loss_fwd_bwd_vpf(ctx: Context, logits: torch.Tensor, targets, loss_mask, row_traj, adv, old_logp,
                                ref_logp, n_loss, cfg: LossCfg, vocab_start: int, vocab_total: int,
                                xchg: VpfExchange, *, dlogits: Optional[torch.Tensor] = None, logp=None,
                                entropy=None, stats=None, accumulate: Optional[bool] = None, stream=None) -> dict:
    """logits: this rank's shard [N, vocab_local] (may be a column slice of a wider row buffer); dlogits the
    same shape (default: a new contiguous tensor)."""
    N, ld = _row_view(logits, "logits")
    V = logits.shape[1]
    dev = logits.device
    # default outputs are allocated (and zeroed) on the stream the call runs on: ranks run on their own streams
    import contextlib
    on = torch.cuda.stream(stream) if isinstance(stream, torch.cuda.Stream) else contextlib.nullcontext()
    with on:
        if dlogits is None:   # same row stride as the logits (the C ABI takes one ld for both)
            dlogits = torch.empty((N, max(ld, V)), dtype=logits.dtype, device=dev)[:, :V]
        if logp is None:
            logp = torch.empty(N, dtype=torch.float32, device=dev)
        if entropy is None:
            entropy = torch.empty(N, dtype=torch.float32, device=dev)
        if stats is None:
            stats = torch.zeros(len(STATS_FIELDS), dtype=torch.float64, device=dev)
    Nd, ldd = _row_view(dlogits, "dlogits")
    if dlogits.shape != logits.shape or dlogits.dtype != logits.dtype or ldd != ld:
        raise ValueError("dlogits must have the logits' shape, dtype and row stride")
    _arr(targets, "targets", torch.int32, N, dev)
    _arr(loss_mask, "loss_mask", torch.uint8, N, dev)
    _arr(row_traj, "row_traj", torch.int32, N, dev)
    _arr(adv, "adv", torch.float64, 1, dev, at_least=True)
    _arr(old_logp, "old_logp", torch.float32, N, dev)
    _arr(ref_logp, "ref_logp", torch.float32, N, dev, optional=True)
    _arr(n_loss, "n_loss", torch.int64, 1, dev)
    _arr(stats, "stats", torch.float64, len(STATS_FIELDS), dev)
    _arr(logp, "logp", torch.float32, N, dev)
    _arr(entropy, "entropy", torch.float32, N, dev)
    _arr(cfg.adv_index, "cfg.adv_index", torch.int32, N, dev, optional=True)
    _arr(cfg.traj_loss_tokens, "cfg.traj_loss_tokens", torch.int64, None, dev, optional=True)
    _arr(cfg.n_active_traj, "cfg.n_active_traj", torch.int64, 1, dev, optional=True)
    sh = otk_vocab_shard(int(vocab_start), int(vocab_total))
    c = cfg.c(accumulate, adv)
    peers = xchg.peers()
    st = _lib.otk_policy_loss_fwd_bwd_vpf(
        ctx.handle, N, V, ld, _dtype_code(logits), _ptr(logits), _ptr(targets), _ptr(loss_mask), _ptr(row_traj),
        _ptr(adv), _ptr(old_logp), _ptr(ref_logp), _ptr(n_loss), C.byref(c), C.byref(sh), C.byref(peers),
        _ptr(dlogits), _ptr(logp), _ptr(entropy), _ptr(stats), _stream(stream))
    _check(st)
    return dict(dlogits=dlogits, logp=logp, entropy=entropy, stats=stats)


def otk_policy_loss_fwd_bwd_vpf_group(ctxs, logits_shards, targets, loss_mask, row_traj, adv, old_logp, ref_logp,
                                      n_loss, cfg: LossCfg, vocab_starts, vocab_total: int, xchgs, *,
                                      dlogits=None, outs=None, accumulate: Optional[bool] = None,
                                      stream=None) -> list:
    """K4-VPF with P ranks EMULATED on this GPU in ONE cooperative launch (otk.h otk_policy_loss_fwd_bwd_vpf_group):
    rank k = (ctxs[k], logits_shards[k] = column slice [vocab_starts[k], +width) of the rows, xchgs[k]). Every
    rank's CTAs are resident together, so nothing depends on separate launches being co-scheduled. Returns one
    dict per rank (dlogits, logp, entropy, stats), bitwise the per-rank calls' results."""
    P = len(ctxs)
    if not (len(logits_shards) == len(vocab_starts) == len(xchgs) == P):
        raise ValueError("one logits shard, vocab start and exchange per rank")
    N, ld = _row_view(logits_shards[0], "logits")
    dev = logits_shards[0].device
    res = []
    for k in range(P):
        lg = logits_shards[k]
        n_k, ld_k = _row_view(lg, "logits")
        if n_k != N or ld_k != ld or lg.dtype != logits_shards[0].dtype:
            raise ValueError("every shard needs the same rows, row stride and dtype")
        dl = dlogits[k] if dlogits is not None else torch.empty((N, max(ld, lg.shape[1])), dtype=lg.dtype,
                                                                 device=dev)[:, :lg.shape[1]]
        Nd, ldd = _row_view(dl, "dlogits")
        if dl.shape != lg.shape or dl.dtype != lg.dtype or ldd != ld:
            raise ValueError("dlogits must have the logits' shape, dtype and row stride")
        o = dict(outs[k]) if outs is not None else dict(
            logp=torch.empty(N, dtype=torch.float32, device=dev),
            entropy=torch.empty(N, dtype=torch.float32, device=dev),
            stats=torch.zeros(len(STATS_FIELDS), dtype=torch.float64, device=dev))
        _arr(o["logp"], "logp", torch.float32, N, dev)
        _arr(o["entropy"], "entropy", torch.float32, N, dev)
        _arr(o["stats"], "stats", torch.float64, len(STATS_FIELDS), dev)
        o["dlogits"] = dl
        res.append(o)
    _arr(targets, "targets", torch.int32, N, dev)
    _arr(loss_mask, "loss_mask", torch.uint8, N, dev)
    _arr(row_traj, "row_traj", torch.int32, N, dev)
    _arr(adv, "adv", torch.float64, 1, dev, at_least=True)
    _arr(old_logp, "old_logp", torch.float32, N, dev)
    _arr(ref_logp, "ref_logp", torch.float32, N, dev, optional=True)
    _arr(n_loss, "n_loss", torch.int64, 1, dev)
    _arr(cfg.adv_index, "cfg.adv_index", torch.int32, N, dev, optional=True)
    _arr(cfg.traj_loss_tokens, "cfg.traj_loss_tokens", torch.int64, None, dev, optional=True)
    _arr(cfg.n_active_traj, "cfg.n_active_traj", torch.int64, 1, dev, optional=True)
    peers = [x.peers() for x in xchgs]
    calls = (otk_vpf_rank_call * P)()
    for k in range(P):
        o = res[k]
        calls[k] = otk_vpf_rank_call(ctxs[k].handle.value, logits_shards[k].shape[1], _ptr(logits_shards[k]),
                                     otk_vocab_shard(int(vocab_starts[k]), int(vocab_total)), C.pointer(peers[k]),
                                     _ptr(o["dlogits"]), _ptr(o["logp"]), _ptr(o["entropy"]), _ptr(o["stats"]))
    c = cfg.c(accumulate, adv)
    _check(_lib.otk_policy_loss_fwd_bwd_vpf_group(P, calls, N, ld, _dtype_code(logits_shards[0]), _ptr(targets),
                                                  _ptr(loss_mask), _ptr(row_traj), _ptr(adv), _ptr(old_logp),
                                                  _ptr(ref_logp), _ptr(n_loss), C.byref(c), _stream(stream)))
    return res


__all__ = [n for n in list(globals()) if n.startswith("otk_") or n in (
    "Context", "LossCfg", "OtkError", "DeviceTrajBatch", "traj_batch_to_device", "stats_dict", "EXPORTED",
    "VpfExchange")]
