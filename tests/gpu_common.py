"""Shared helpers for the -m gpu parity tests: problem setup and the tolerance checks of DESIGN.md §3/§6."""
import math

import numpy as np
import torch

from oracle import oracle_ref as O
from synth import make_logits, make_noise

BF16_REL = 2.0 ** -7      # dlogits per-element relative tolerance (bf16 output)
F32_REL = 1e-5            # dlogits per-element relative tolerance (fp32 output)
COEF_ABS = 1e-5           # dlogits absolute floor, in units of |coef_j|
LOGP_TOL = {"bf16": 2e-3, "f32": 1e-5}   # north_star: log-probs within 2e-3 abs (bf16 logits)


def oracle_cfg(cfg):
    return O.LossCfg(clip_low=cfg.clip_low, clip_high=cfg.clip_high, kl_beta=cfg.kl_beta, kl_type=cfg.kl_type,
                     log_ratio_clamp=cfg.log_ratio_clamp, logit_scale=cfg.logit_scale)


def row_problem(n, V, *, dtype="bf16", ld=None, seed=0, mask_p=0.7, B=6, old_sd=0.05, ref_sd=0.1,
                force_clip=0, uniform_rows=(), logit_scale=1.0, device="cuda"):
    """Rows + side data. old/ref = ORACLE logp + synth noise (no input derives from the CUDA path)."""
    logits, targets = make_logits(n, V, ld=ld, dtype=dtype, seed=seed, device="cpu", uniform_rows=uniform_rows)
    wide = logits.to(torch.float64).numpy()[:, :V]
    rng = np.random.default_rng(seed + 1000)
    mask = (rng.random(n) < mask_p).astype(np.uint8)
    row_traj = np.sort(rng.integers(0, B, n)).astype(np.int32)
    adv = rng.normal(size=B)
    y = targets.numpy()
    logp0 = np.array([O.row_forward(wide[j], int(y[j]), logit_scale)[0] for j in range(n)])
    old = logp0 + make_noise(n, old_sd, seed + 1).double().numpy()
    ref = logp0 + make_noise(n, ref_sd, seed + 2).double().numpy()
    for j in np.flatnonzero(mask)[:force_clip]:
        A = adv[row_traj[j]]
        old[j] = logp0[j] - (math.log(1.6) if A > 0 else math.log(0.5))   # r = 1.6 / 0.5: clipped
    old32 = old.astype(np.float32)
    ref32 = ref.astype(np.float32)
    d = dict(logits=logits.to(device), targets=targets.to(device), mask=torch.from_numpy(mask).to(device),
             row_traj=torch.from_numpy(row_traj).to(device), adv=torch.from_numpy(adv).to(device),
             old=torch.from_numpy(old32).to(device), ref=torch.from_numpy(ref32).to(device))
    h = dict(wide=wide, targets=y, mask=mask, row_traj=row_traj, adv=adv, old=old32.astype(np.float64),
             ref=ref32.astype(np.float64), V=V)
    return d, h


def near_kink(logp, old, ref, A, cfg, eps=1e-4):
    """Rows whose clip / clamp decision is within eps of a boundary: either branch is correct."""
    r = math.exp(max(min(logp - old, cfg.log_ratio_clamp), -cfg.log_ratio_clamp))
    return (abs(r - (1 + cfg.clip_high)) < eps or abs(r - (1 - cfg.clip_low)) < eps
            or abs(abs(logp - old) - cfg.log_ratio_clamp) < eps
            or (ref is not None and abs(abs(ref - logp) - cfg.log_ratio_clamp) < eps))


def coef_sensitivity(logp, old, ref, A, N, cfg):
    """|d coef_j / d logp_j| from oracle quantities: coef = -s (m/N) G(logp) with dG/dlogp = -A r
    (unclipped) + beta * (k3: e^d, k1: 0, k2: 1). The kernel's fp32 logp carries ~1e-6 absolute error,
    so coef inherits |dcoef/dlogp| * dlogp of ABSOLUTE error even when coef itself is tiny (G can cancel)."""
    C = cfg.log_ratio_clamp
    r = math.exp(max(min(logp - old, C), -C))
    s = cfg.logit_scale
    dg = abs(A) * r
    if cfg.kl_beta:
        if cfg.kl_type == 3:
            dg += cfg.kl_beta * math.exp(max(min(ref - logp, C), -C))
        elif cfg.kl_type == 2:
            dg += cfg.kl_beta
    return s * dg / max(N, 1)


def check_dlogits_rows(got, want, coef, rows, dtype, V, dcoef=None, logp_err=1e-5):
    """|d| <= rel*|ref| + 1e-5*|coef_j| + logp_err*|dcoef_j/dlogp_j| per element."""
    rel = BF16_REL if dtype == "bf16" else F32_REL
    worst = 0.0
    for j in rows:
        g = got[j, :V].double().cpu().numpy() if isinstance(got, torch.Tensor) else got[j]
        w = want[j]
        floor = COEF_ABS * abs(coef[j]) + (logp_err * dcoef[j] if dcoef is not None else 0.0)
        tol = rel * np.abs(w) + floor + 1e-30
        ratio = float(np.max(np.abs(g - w) / tol))
        worst = max(worst, ratio)
    return worst


def dcoef_rows(h, want_logp, cfg, N, beta):
    return {j: coef_sensitivity(want_logp[j], h["old"][j], h["ref"][j] if beta else 0.0,
                                h["adv"][h["row_traj"][j]], N, cfg)
            for j in range(len(h["mask"])) if h["mask"][j]}
