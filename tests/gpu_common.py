"""Shared helpers for the -m gpu parity tests: problem setup and the tolerance checks of DESIGN.md §6
(the tolerance model itself lives in oracle/parity.py, shared with bench.py's parity block)."""
import math

import numpy as np
import torch

from oracle import oracle_ref as O
from oracle import parity as P
from oracle.parity import KINK_EPS, LOGP_TOL  # noqa: F401  (north_star: log-probs within 2e-3 abs, bf16 logits)
from synth import make_logits, make_noise


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


def near_kink(logp, old, ref, A, cfg, eps=KINK_EPS):
    """Rows whose clip / clamp decision is within eps of a boundary: either branch is correct (both are
    checked, see check_dlogits_rows)."""
    return P.near_kink(logp, old, ref, A, cfg, eps)


def coef_sensitivity(logp, old, ref, A, N, cfg):
    """|d coef_j / d logp_j| per unit weight 1/N: coef = -s w G(logp) with dG/dlogp = -A r (unclipped) +
    beta * (k3: e^d, k1: 0, k2: 1)."""
    return abs(cfg.logit_scale) * float(P.g_sensitivity(logp, old, ref, A, cfg)) / max(N, 1)


def dcoef_rows(h, want_logp, cfg, N, beta, W=None):
    """Per trainable row: |d coef_j / d logp_j| (row weight W[j], default the token-mean 1/N)."""
    out = {}
    for j in range(len(h["mask"])):
        if h["mask"][j]:
            w = (1.0 / max(N, 1)) if W is None else float(W[j])
            out[j] = abs(cfg.logit_scale) * w * float(P.g_sensitivity(want_logp[j], h["old"][j],
                                                                       h["ref"][j] if beta else 0.0,
                                                                       h["adv"][h["row_traj"][j]], cfg))
    return out


def check_dlogits_rows(got, want, coef, rows, dtype, V, dcoef=None, logp_err=P.LOGP_ERR, *, wide, targets,
                       scale=1.0, h=None, cfg=None, W=None, ent=None):
    """Worst max(elementwise, L1) error / tolerance ratio over `rows` (oracle/parity.py):
    |d_v| <= rel |want_v| + (1e-5 |coef_j| + logp_err |dcoef_j/dlogp_j|) |p_v - [v=y_j]| + [v=y_j] |coef_j| p_y logp_err,
    and sum_v |d_v| <= L1_REL sum_v |want_v| + sum_v floor_v. `wide[j]` (array or callable) is the row's
    logits in float64, from which the oracle's p is formed. With h / cfg given, a row near a clip / clamp kink
    passes if either branch's coefficient passes. ent = (c_H, H dict): entropy-bonus rows (want includes the
    bonus term; its magnitude w c_H s p (|ln p| + H) gets the relative tolerance too)."""
    worst = 0.0
    for j in rows:
        g = got[j, :V].double().cpu().numpy() if isinstance(got, torch.Tensor) else np.asarray(got[j])
        x = wide(j) if callable(wide) else wide[j]
        y = int(targets[j])
        lpj, H, _, p = O.row_forward(x[:V], y, scale)
        q = p.copy()
        q[y] -= 1.0
        w = np.asarray(want[j], np.float64)
        c = float(coef[j])
        dslope = dcoef[j] if dcoef is not None else 0.0
        ent_mag = None
        if ent is not None:
            c_h, wj = ent
            with np.errstate(divide="ignore"):
                lnp = np.where(p > 0, np.log(np.where(p > 0, p, 1.0)), 0.0)
            ent_mag = abs(wj[j] * c_h * scale) * p * (np.abs(lnp) + H)
        cands = [(c, w)]
        if h is not None and cfg is not None:
            A = h["adv"][h["row_traj"][j]]
            refj = h["ref"][j] if cfg.kl_beta else None
            if P.near_kink(lpj, h["old"][j], refj, A, cfg):
                wj = (1.0 / max(int(h["mask"].sum()), 1)) if W is None else float(W[j])
                cands += [(a, w + (a - c) * q) for a in P.branch_coefs(lpj, h["old"][j], refj, A, wj, cfg)]
        dets = [dict() for _ in cands]
        rs = [P.row_ratio(g, wc, q, y, cc, P.COEF_REL * abs(cc) + logp_err * dslope, dtype, ent_mag, dets[i])
              for i, (cc, wc) in enumerate(cands)]
        best = min(rs)
        if best > 1.0:   # diagnostics of a failing row (pytest shows captured stdout on failure)
            print(f"dlogits row {j}: ratio {best:.4g}", dets[int(np.argmin(rs))])
        worst = max(worst, best)
    return worst
