"""Comparison of CUDA-path outputs with the float64 oracle — TEST INFRASTRUCTURE.

Only tests/ and bench.py's cpu_baseline / parity leg use this module. It imports the oracle (oracle_ref,
oracle_cpu) and nothing from the CUDA path: the CUDA path's outputs come in as plain tensors / arrays.

Tolerances (BASELINE.json north_star; DESIGN.md §6 "Error budget"):
  masks, row_traj, token counts, group sizes ........ bit-exact
  advantages ........................................ 1e-6 abs
  logp, entropy ..................................... 2e-3 abs for bf16 logits, 1e-5 for fp32
  loss .............................................. 1e-4 x max(|loss|, sum_j w_j |L_j|)   (R22)
  dlogits, per element (row j, column v; q_v = p_v - [v = y_j], the oracle's coef_j and p_v):
      |got - want| <= rel |want| + dcoef_j |q_v| + [v = y_j] |coef_j| p_y LOGP_ERR + ABS_FLOOR
      rel = 2^-7 (1 + 2^-6) for bf16 output: e and the product are each rounded once to 8 significant bits
      (<= 2^-8 relative each), plus the 16-bit split of the fp32 scale (3 x 2^-16); 1e-5 for fp32 output.
      dcoef_j = COEF_REL |coef_j| + LOGP_ERR s w_j |dG/dlogp| is the absolute error coef_j inherits from the
      fp32 logp (coef = -s w G(logp), and G's PPO / KL parts can cancel); the target column carries
      coef * p_y * dlogp from expm1(logp). Both floors scale with the element's own |p_v - onehot|, so a
      tiny-probability element is checked relative to itself, never against a row-wide floor. ABS_FLOOR =
      2^-126 (the smallest normal of fp32 and bf16): values below it may flush to 0 (fp32 math is
      flush-to-zero, and bf16 subnormals end at 2^-133) — e.g. p ~ e^-90 behind a dominant logit.
  dlogits, per row (L1, over the non-target columns v != y_j; the target column is one element, formed
      separately as coef expm1(logp), and carries half of the row's |want| mass, so it stays with the
      per-element check): sum_v |got - want| <= L1_REL sum_v |want| + 3 rel sqrt(sum_v want_v^2) + sum_v floor_v.
      The element errors are independent roundings with mean < L1_REL |want_v| (2^-8; two RNE roundings
      average ~2^-9) and range <= rel |want_v|, so by Hoeffding the sum exceeds its mean by more than
      3 rel sqrt(sum want^2) with probability < e^-18 per row. Where the mass is spread over many elements the
      second term vanishes and the check is 2^-8, half the per-element bound; a row dominated by one or two
      elements is left to the per-element check.
  Rows within KINK_EPS of a clip / ratio-clamp / KL-clamp / dual-clip boundary accept either branch's
  coefficient (the fp32 and the float64 logp can fall on different sides); both are checked in full.
"""
from __future__ import annotations

import math

import numpy as np

from oracle import oracle_ref as O

LOGP_TOL = {"bf16": 2e-3, "f32": 1e-5}
ADV_TOL = 1e-6
LOSS_REL = 1e-4
DL_REL = {"bf16": 2.0 ** -7 * (1 + 2.0 ** -6), "f32": 1e-5}
DL_L1_REL = {"bf16": 2.0 ** -8, "f32": 1e-5}
L1_DEV = 3.0          # Hoeffding deviation, in units of rel * sqrt(sum want^2)
ABS_FLOOR = 2.0 ** -126
COEF_REL = 1e-5
LOGP_ERR = 1e-5
KINK_EPS = 1e-4


def _arr(x):
    return np.asarray(x, np.float64)


def g_sensitivity(logp, old, ref, A, cfg):
    """|dG/dlogp| (vectorised): G = dL/dlogp = -A r (unclipped PPO part) + beta * Gk; dG/dlogp = -A r +
    beta * (k3: e^d, k2: 1, k1: 0). Bounded from above on both branches (used for an error bound only)."""
    logp, old, A = _arr(logp), _arr(old), _arr(A)
    C = cfg.log_ratio_clamp
    out = np.zeros_like(logp)
    if not getattr(cfg, "sft", False):
        out += np.abs(A) * np.exp(np.clip(logp - old, -C, C))
    if cfg.kl_beta:
        if cfg.kl_type == O.KL_K3:
            out += cfg.kl_beta * np.exp(np.clip(_arr(ref) - logp, -C, C))
        elif cfg.kl_type == O.KL_K2:
            out += cfg.kl_beta
    return out


def coef_error(coef, logp, old, ref, A, w, cfg):
    """Absolute error bound of coef_j = -s w_j G_j(logp_j) given a LOGP_ERR error in the fp32 logp."""
    return COEF_REL * np.abs(_arr(coef)) + LOGP_ERR * abs(cfg.logit_scale) * np.abs(_arr(w)) * \
        g_sensitivity(logp, old, ref, A, cfg)


def near_kink(logp, old, ref, A, cfg, eps=KINK_EPS):
    """Scalar: is the row's clip / clamp decision within eps of a boundary (either branch correct)?"""
    C = cfg.log_ratio_clamp
    r = math.exp(max(min(logp - old, C), -C))
    k = (abs(abs(logp - old) - C) < eps
         or (not getattr(cfg, "sft", False) and (abs(r - (1 + cfg.clip_high)) < eps or abs(r - (1 - cfg.clip_low)) < eps)))
    if cfg.kl_beta and ref is not None and cfg.kl_type == O.KL_K3:
        k = k or abs(abs(ref - logp) - C) < eps
    dual = getattr(cfg, "dual_clip", 0.0)
    if dual and A < 0:
        rbar = min(max(r, 1 - cfg.clip_low), 1 + cfg.clip_high)
        k = k or abs(max(-A * r, -A * rbar) + dual * A) < eps * abs(A)
    return bool(k)


def branch_coefs(logp, old, ref, A, w, cfg):
    """Every coefficient a near-kink row may correctly carry: G_pg in {-A r, 0} x G_kl in {k3 slope, 0}."""
    C = cfg.log_ratio_clamp
    s = cfg.logit_scale
    if getattr(cfg, "sft", False):
        pgs = [-1.0]
    else:
        pgs = [-A * math.exp(max(min(logp - old, C), -C)), 0.0]
    kls = [0.0]
    if cfg.kl_beta:
        if cfg.kl_type == O.KL_K3:
            kls = [1.0 - math.exp(max(min(ref - logp, C), -C)), 0.0]
        elif cfg.kl_type == O.KL_K1:
            kls = [1.0]
        else:
            kls = [logp - ref]
    return [-s * w * (gp + cfg.kl_beta * gk) for gp in pgs for gk in kls]


def l1_ratio(err, ref, ref_sq, floor, dtype):
    """Row L1 check (module docstring): sum|d| / (L1_REL sum|want| + L1_DEV rel sqrt(sum want^2) + sum floor)."""
    err = _arr(err)
    den = DL_L1_REL[dtype] * _arr(ref) + L1_DEV * DL_REL[dtype] * np.sqrt(_arr(ref_sq)) + _arr(floor) + 1e-300
    return np.where(err == 0, 0.0, err / den)


def row_ratio(got, want, q, y, coef, dcoef, dtype, ent_mag=None, detail=None):
    """max(elementwise ratio, L1 ratio) of one row; `want` = coef q (+ entropy term), q = p - onehot.
    detail (a dict) receives the worst element (index, got, want, tol) and the L1 ratio, for diagnostics."""
    rel = DL_REL[dtype]
    aq = np.abs(q)
    floor = dcoef * aq + ABS_FLOOR
    floor[y] += abs(coef) * (q[y] + 1.0) * LOGP_ERR
    if ent_mag is not None:
        floor = floor + rel * ent_mag
    d = np.abs(_arr(got) - want)
    tol = rel * np.abs(want) + floor
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(d == 0, 0.0, d / tol)
    r = np.where(np.isnan(r), np.inf, r)
    nt = np.ones(len(d), bool)
    nt[y] = False
    l1 = float(l1_ratio(math.fsum(d[nt]), math.fsum(np.abs(want[nt])), math.fsum(want[nt] * want[nt]),
                        math.fsum(floor[nt]), dtype))
    if detail is not None and r.size:
        v = int(np.argmax(r))
        detail.update(elem=v, got=float(_arr(got)[v]), want=float(want[v]), tol=float(tol[v]),
                      elem_ratio=float(r[v]), l1_ratio=l1, target=int(y), coef=float(coef))
    return max(float(np.max(r)) if r.size else 0.0, l1)


# ------------------------------------------------------------------------------------------------
# all-row comparison of a full micro-batch (C oracle, chunked host copies) — tests/test_gpu_fullsize.py,
# bench.py parity block
# ------------------------------------------------------------------------------------------------
def _host_rows(t, r0, r1, dtype):
    from oracle import oracle_cpu as OC
    if dtype == "bf16":
        return OC.bf16_bits(t[r0:r1])
    return t[r0:r1].detach().cpu().contiguous().numpy()


def oracle_logp(logits, targets, V, dtype, chunk=4096, logit_scale=1.0):
    """Oracle O3 (C, float64) over every row of a device tensor, chunked through host memory."""
    from oracle import oracle_cpu as OC
    n = logits.shape[0]
    out = {k: np.zeros(n) for k in ("logp", "entropy", "lse")}
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        f = OC.logprob_entropy(_host_rows(logits, r0, r1, dtype), targets[r0:r1].cpu().numpy(), V=V,
                               logit_scale=logit_scale)
        for k in out:
            out[k][r0:r1] = f[k]
    return out


def microbatch_parity(logits, targets, loss_mask, row_traj, adv, old, ref, n_loss, cfg, dtype, V,
                      got_logp, got_entropy, got_dlogits, got_stats, chunk=4096):
    """Every row of one micro-batch: the C oracle (O3 + O4, float64) against the CUDA path's outputs.

    logits / targets / got_* may be device tensors; loss_mask, row_traj, adv, old, ref are host arrays (old and
    ref float32, as the kernel read them). cfg: oracle_ref.LossCfg (token-mean). got_stats: dict with loss,
    n_clipped, n_tokens. Returns the max error / tolerance ratios (<= 1 passes) and the raw maxima."""
    from oracle import oracle_cpu as OC
    n = logits.shape[0]
    mask = np.asarray(loss_mask, np.uint8)
    rt = np.asarray(row_traj)
    adv = _arr(adv)
    s = cfg.logit_scale
    w_tok = 1.0 / n_loss if n_loss > 0 else 0.0
    glp = got_logp.double().cpu().numpy() if hasattr(got_logp, "cpu") else _arr(got_logp)
    gH = got_entropy.double().cpu().numpy() if hasattr(got_entropy, "cpu") else _arr(got_entropy)
    row_L = np.zeros(n)
    clipped = 0
    n_kink = 0
    worst_el, worst_l1, worst_lp, worst_H = 0.0, 0.0, 0.0, 0.0
    masked_nonzero = 0
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        bits = _host_rows(logits, r0, r1, dtype)
        tg = targets[r0:r1].cpu().numpy()
        m = mask[r0:r1]
        o = OC.policy_loss(bits, tg, m, rt[r0:r1], adv, old[r0:r1], None if ref is None else ref[r0:r1], n_loss,
                           cfg, V=V, want_dlogits=False)
        row_L[r0:r1] = o["row_L"]
        clipped += int(o["row_clipped"].sum())
        tr = m != 0
        if tr.any():
            worst_lp = max(worst_lp, float(np.max(np.abs(glp[r0:r1][tr] - o["logp"][tr]))))
            worst_H = max(worst_H, float(np.max(np.abs(gH[r0:r1][tr] - o["entropy"][tr]))))
        A = adv[rt[r0:r1]]
        refc = None if ref is None else ref[r0:r1]
        dc = coef_error(o["row_coef"], o["logp"], old[r0:r1], refc if refc is not None else 0.0, A, w_tok, cfg)
        got = _host_rows(got_dlogits, r0, r1, dtype)
        cmp = OC.dlogits_compare(bits, tg, m, s, o["row_lse"], o["row_coef"], dc, LOGP_ERR, DL_REL[dtype],
                                 ABS_FLOOR, got, V=V)
        el = cmp["max_ratio"]
        l1 = l1_ratio(cmp["l1_err"], cmp["l1_ref"], cmp["l2_ref"], cmp["l1_floor"], dtype)
        bad = np.flatnonzero(tr & ((el > 1.0) | (l1 > 1.0)))
        for i in bad:   # a row on a clip / clamp boundary may carry the other branch's coefficient
            j = r0 + i
            refj = None if ref is None else float(ref[j])
            if not near_kink(o["logp"][i], float(old[j]), refj, float(A[i]), cfg):
                continue
            n_kink += 1
            best = (el[i], l1[i])
            for c in branch_coefs(o["logp"][i], float(old[j]), refj, float(A[i]), w_tok, cfg):
                one = np.zeros(r1 - r0, np.uint8)
                one[i] = 1
                cc = OC.dlogits_compare(bits, tg, one, s, o["row_lse"], np.full(r1 - r0, c),
                                        np.full(r1 - r0, dc[i]), LOGP_ERR, DL_REL[dtype], ABS_FLOOR, got, V=V)
                li = float(l1_ratio(cc["l1_err"][i], cc["l1_ref"][i], cc["l2_ref"][i], cc["l1_floor"][i], dtype))
                if max(cc["max_ratio"][i], li) < max(best):
                    best = (cc["max_ratio"][i], li)
            el[i], l1[i] = best
        if tr.any():
            worst_el = max(worst_el, float(np.max(el[tr])))
            worst_l1 = max(worst_l1, float(np.max(l1[tr])))
        if (~tr).any():
            masked_nonzero += int(np.count_nonzero(got[~tr][:, :V]))
    loss = math.fsum(row_L[mask != 0] * w_tok)
    scale = max(abs(loss), math.fsum(np.abs(row_L[mask != 0])) * w_tok)
    loss_err = abs(got_stats["loss"] - loss)
    return {
        "rows": int(n), "trainable": int(mask.sum()),
        "logp_max_abs_err": worst_lp, "logp_ratio": worst_lp / LOGP_TOL[dtype],
        "entropy_max_abs_err": worst_H, "entropy_ratio": worst_H / LOGP_TOL[dtype],
        "dlogits_elem_ratio": worst_el, "dlogits_l1_ratio": worst_l1,
        "masked_rows_nonzero": masked_nonzero,
        "loss": got_stats["loss"], "loss_oracle": loss, "loss_abs_err": loss_err,
        "loss_ratio": loss_err / (LOSS_REL * scale) if scale > 0 else (0.0 if loss_err == 0 else math.inf),
        "n_clipped": int(got_stats["n_clipped"]), "n_clipped_oracle": clipped, "kink_rows": n_kink,
        "n_tokens_exact": int(got_stats["n_tokens"]) == int(mask.sum()),
    }


def parity_ok(p):
    return (p["logp_ratio"] <= 1 and p["entropy_ratio"] <= 1 and p["dlogits_elem_ratio"] <= 1
            and p["dlogits_l1_ratio"] <= 1 and p["loss_ratio"] <= 1 and p["masked_rows_nonzero"] == 0
            and p["n_tokens_exact"] and abs(p["n_clipped"] - p["n_clipped_oracle"]) <= p["kink_rows"])


# ------------------------------------------------------------------------------------------------
# LM head (NEXT-1): dh / dW tolerance from ambiguous bf16 roundings of the logits (R34)
# ------------------------------------------------------------------------------------------------
def bf16_ulp(x):
    """Spacing of bf16 numbers at |x| (8 significant bits): 2^(floor(log2|x|) - 7); the smallest normal's below."""
    ax = np.maximum(np.abs(_arr(x)), 2.0 ** -126)
    return np.exp2(np.floor(np.log2(ax)) - 7.0)


def lmhead_flip_tolerance(h, W, x64, xb, y, coef, logp, old, ref, A, w_row, cfg, mask, acc_terms=None):
    """Extra absolute tolerance of dh = dx W and dW = dx^T h where the device's bf16 logits may differ from the
    oracle's by one bf16 rounding (R34).

    The oracle rounds x64 = h W^T (float64) to bf16 (xb); the device rounds an fp32 accumulation of the same bf16
    products, whose error is at most d 2^-24 sum_k |h_jk W_vk| (recursive fp32 summation, round to nearest). Where
    x64 lies that close to a bf16 rounding midpoint either neighbour is a correct logit (as either branch of a clip
    kink is a correct coefficient), and dx moves by first-order amounts that the rounding spread of the element-wise
    check does not cover — one flipped element can dominate a column of dW. Bound, per ambiguous (j, v) with
    Delta = the other neighbour - xb:
      dx_jv itself:       |coef_j| p_jv |expm1(s Delta)|                    (delta_jv)
      the row's lse:      |coef_j| p_jv' rho_j for every v',  rho_j = sum_v p_jv |expm1(s Delta_jv)|
      the coefficient:    |dcoef_j / dlogp_j| s sum_v |Delta_jv| (p_jv + [v = y_j]) |p_jv' - [v' = y_j]|
    each pushed through |W| (dh) or |h| (dW), the sum scaled by 1.5 for second-order terms. Returns
    (tol_dh [N, d], tol_dW [V, d], number of ambiguous logits, the ambiguity mask). acc_terms overrides d in the
    accumulation bound (tests widen it to exercise many flips)."""
    h, W, x64, xb = _arr(h), _arr(W), _arr(x64), _arr(xb)
    N, d = h.shape
    s = cfg.logit_scale
    eps = (d if acc_terms is None else acc_terms) * 2.0 ** -24 * (np.abs(h) @ np.abs(W).T)
    u = bf16_ulp(xb)
    side = np.where(x64 >= xb, 1.0, -1.0)
    mid = xb + side * u / 2
    amb = np.abs(x64 - mid) <= eps
    delta = np.where(amb, side * u, 0.0)
    z = s * xb
    z = z - z.max(axis=1, keepdims=True)
    P = np.exp(z)
    P /= P.sum(axis=1, keepdims=True)
    em = np.abs(np.expm1(s * delta))
    ac = np.abs(_arr(coef))[:, None]
    prim = ac * P * em
    rho = (P * em).sum(axis=1)
    onehot = np.zeros_like(P)
    onehot[np.arange(N), np.asarray(y)] = 1.0
    dlp = s * (np.abs(delta) * (P + onehot)).sum(axis=1)
    sens = abs(s) * np.abs(_arr(w_row)) * g_sensitivity(logp, old, ref if cfg.kl_beta else 0.0, A, cfg)
    dco = sens * dlp
    ent = getattr(cfg, "ent_coef", 0.0)
    if ent:   # the entropy-bonus part w c_H s p (ln p + H) of dx moves with p as well
        with np.errstate(divide="ignore"):
            lnP = np.where(P > 0, np.log(np.where(P > 0, P, 1.0)), 0.0)
        Hrow = -(P * lnP).sum(axis=1, keepdims=True)
        prim = prim + np.abs(_arr(w_row) * ent * s)[:, None] * P * (np.abs(lnP) + Hrow + 1.0) * em
    m = (_arr(mask) != 0)[:, None]
    E = m * (prim + (ac[:, 0] * rho)[:, None] * P + dco[:, None] * np.abs(P - onehot))
    tol_dh = 1.5 * (E @ np.abs(W))
    tol_dW = 1.5 * (E.T @ np.abs(h))
    return tol_dh, tol_dW, int(amb.sum()), amb
