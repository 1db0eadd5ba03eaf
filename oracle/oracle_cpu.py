"""ctypes front end of oracle_cpu.c (float64 C oracle, OpenMP over rows) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__ (build + smoke) and bench.py's cpu_baseline / --impl reference legs use it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle_cpu.c")
LIB = os.path.join(HERE, "liboracle_cpu.so")


class orc_cfg(C.Structure):
    _fields_ = [("clip_low", C.c_double), ("clip_high", C.c_double), ("kl_beta", C.c_double),
                ("log_ratio_clamp", C.c_double), ("logit_scale", C.c_double),
                ("kl_type", C.c_int32), ("zero_masked_rows", C.c_int32)]


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", LIB, SRC, "-lm"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _dtype_code(arr):
    if arr.dtype == np.float32:
        return 0
    if arr.dtype == np.uint16:   # bf16 bit patterns
        return 1
    raise TypeError("logits must be float32 or uint16 (bf16 bits)")


def logprob_entropy(logits: np.ndarray, targets, row_mask=None, V=None, logit_scale=1.0):
    logits = np.ascontiguousarray(logits)
    n, ld = logits.shape
    V = ld if V is None else V
    targets = np.ascontiguousarray(targets, np.int32)
    rm = None if row_mask is None else np.ascontiguousarray(row_mask, np.uint8)
    out = [np.zeros(n) for _ in range(3)]
    bad = lib().orc_logprob_entropy(C.c_int64(n), C.c_int64(V), C.c_int64(ld), C.c_int32(_dtype_code(logits)),
                                    _p(logits), _p(targets), _p(rm), C.c_double(logit_scale),
                                    _p(out[0]), _p(out[1]), _p(out[2]))
    if bad:
        raise ValueError("target out of range")
    return dict(logp=out[0], entropy=out[1], lse=out[2])


def policy_loss(logits: np.ndarray, targets, loss_mask, row_traj, adv, old_logp, ref_logp, n_loss, cfg,
                V=None, want_dlogits=True, zero_masked_rows=True):
    """cfg: any object with clip_low, clip_high, kl_beta, kl_type, log_ratio_clamp, logit_scale."""
    logits = np.ascontiguousarray(logits)
    n, ld = logits.shape
    V = ld if V is None else V
    c = orc_cfg(cfg.clip_low, cfg.clip_high, cfg.kl_beta, cfg.log_ratio_clamp, cfg.logit_scale,
                int(cfg.kl_type), int(zero_masked_rows))
    targets = np.ascontiguousarray(targets, np.int32)
    mask = np.ascontiguousarray(loss_mask, np.uint8)
    rt = np.ascontiguousarray(row_traj, np.int32)
    adv = np.ascontiguousarray(adv, np.float64)
    old = np.ascontiguousarray(old_logp, np.float32)
    ref = None if ref_logp is None else np.ascontiguousarray(ref_logp, np.float32)
    dl = np.zeros((n, V)) if want_dlogits else None
    logp, H, L, kl, lse, coef = (np.zeros(n) for _ in range(6))
    clipped = np.zeros(n, np.uint8)
    bad = lib().orc_policy_loss(C.c_int64(n), C.c_int64(V), C.c_int64(ld), C.c_int32(_dtype_code(logits)),
                                _p(logits), _p(targets), _p(mask), _p(rt), _p(adv), _p(old), _p(ref),
                                C.c_int64(int(n_loss)), C.byref(c), _p(dl), _p(logp), _p(H), _p(L),
                                _p(clipped), _p(kl), _p(lse), _p(coef))
    if bad:
        raise ValueError("target out of range")
    return dict(dlogits=dl, logp=logp, entropy=H, row_L=L, row_clipped=clipped, row_kl=kl, row_lse=lse,
                row_coef=coef)


def dlogits_compare(logits: np.ndarray, targets, sel, logit_scale, lse, coef, dcoef, logp_err, rel, abs_floor, got,
                    V=None):
    """Element-by-element comparison of a CUDA-path dlogits block (`got`: float32 or bf16 bits, [n, >= V])
    with the O4 gradient re-formed in float64 from the oracle's per-row lse / coef (orc_dlogits_compare;
    the tolerance terms come from oracle/parity.py)."""
    logits = np.ascontiguousarray(logits)
    got = np.ascontiguousarray(got)
    n, ld = logits.shape
    V = ld if V is None else V
    targets = np.ascontiguousarray(targets, np.int32)
    sel = None if sel is None else np.ascontiguousarray(sel, np.uint8)
    lse = np.ascontiguousarray(lse, np.float64)
    coef = np.ascontiguousarray(coef, np.float64)
    dcoef = np.ascontiguousarray(dcoef, np.float64)
    out = [np.zeros(n) for _ in range(5)]
    lib().orc_dlogits_compare(C.c_int64(n), C.c_int64(V), C.c_int64(ld), C.c_int32(_dtype_code(logits)),
                              _p(logits), _p(targets), _p(sel), C.c_double(logit_scale), _p(lse), _p(coef), _p(dcoef),
                              C.c_double(logp_err), C.c_double(rel), C.c_double(abs_floor), _p(got),
                              C.c_int64(got.shape[1]), C.c_int32(_dtype_code(got)), _p(out[0]), _p(out[1]),
                              _p(out[2]), _p(out[3]), _p(out[4]))
    return dict(max_ratio=out[0], l1_err=out[1], l1_ref=out[2], l2_ref=out[3], l1_floor=out[4])


def build_masks(tb, train_agent=-1):
    B = tb.num_traj
    N = tb.num_rows
    lm, rm = np.zeros(N, np.uint8), np.zeros(N, np.uint8)
    rt = np.zeros(N, np.int32)
    tl = np.zeros(B, np.int64)
    nl = np.zeros(1, np.int64)
    ta = None if tb.traj_agent is None else np.ascontiguousarray(tb.traj_agent, np.int16)
    rc = lib().orc_build_masks(C.c_int32(B), _p(tb.tok_offsets), _p(tb.seg_offsets), _p(tb.seg_source),
                               _p(tb.seg_agent), _p(tb.seg_len), _p(tb.terminated), C.c_int16(train_agent),
                               _p(ta), _p(lm), _p(rm), _p(rt), _p(tl), _p(nl))
    if rc:
        raise ValueError(f"build_masks error {rc}")
    return dict(loss_mask=lm, response_mask=rm, row_traj=rt, traj_loss_tokens=tl, n_loss=int(nl[0]))


def bf16_bits(t) -> np.ndarray:
    """torch bf16 tensor -> numpy uint16 bit patterns (exact)."""
    import torch
    return t.detach().to("cpu").contiguous().view(torch.int16).numpy().view(np.uint16)
