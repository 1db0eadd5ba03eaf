"""The comparison itself (oracle/parity.py, orc_dlogits_compare) is pinned before it judges the CUDA path:
the oracle's own gradient rounded to the kernel's output precision passes, and plausible kernel mistakes
fail — a zeroed small-probability tail, one wrong element, a systematic row bias below the per-element
bound, a wrong-branch coefficient away from a kink. CPU only (-m "not gpu")."""
import math

import numpy as np
import torch

from oracle import oracle_cpu as OC
from oracle import oracle_ref as O
from oracle import parity as P
from synth import make_logits, make_noise


def _problem(n=12, V=4096, seed=5, dtype="bf16"):
    lg, tg = make_logits(n, V, dtype=dtype, seed=seed, uniform_rows=(1,))
    wide = lg.double().numpy()
    y = tg.numpy()
    f = O.logprob_entropy_fwd(wide, y)
    rng = np.random.default_rng(seed)
    mask = np.ones(n, np.uint8)
    mask[[3, 7]] = 0
    rt = (np.arange(n) * 3 // n).astype(np.int32)
    adv = rng.normal(size=3)
    old = (f["logp"] + make_noise(n, 0.05, 1).double().numpy()).astype(np.float32)
    ref = (f["logp"] + make_noise(n, 0.1, 2).double().numpy()).astype(np.float32)
    N = int(mask.sum())
    cfg = O.LossCfg()
    want = O.policy_loss_fwd_bwd(wide, y, mask, rt, adv, old.astype(np.float64), ref.astype(np.float64), N, cfg)
    return lg, tg, wide, y, mask, rt, adv, old, ref, N, cfg, want


def _bf16(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16)


def _ratios(got, wide, y, want, rows, adv, rt, old, ref, N, cfg, dtype="bf16"):
    worst = 0.0
    for j in rows:
        lp, H, _, p = O.row_forward(wide[j], int(y[j]))
        q = p.copy()
        q[y[j]] -= 1.0
        dc = float(P.coef_error(want["coef"][j], lp, old[j], ref[j], adv[rt[j]], 1.0 / N, cfg))
        worst = max(worst, P.row_ratio(got[j].double().numpy(), want["dlogits"][j], q, int(y[j]), want["coef"][j],
                                       dc, dtype))
    return worst


def test_rounded_oracle_passes_and_c_agrees():
    lg, tg, wide, y, mask, rt, adv, old, ref, N, cfg, want = _problem()
    got = _bf16(want["dlogits"])
    rows = np.flatnonzero(mask)
    assert _ratios(got, wide, y, want, rows, adv, rt, old, ref, N, cfg) <= 0.51   # one RNE rounding: <= 2^-8
    o = OC.policy_loss(OC.bf16_bits(lg), y, mask, rt, adv, old, ref, N, cfg, want_dlogits=False)
    assert np.max(np.abs(o["row_coef"] - want["coef"])) <= 1e-13 * np.max(np.abs(want["coef"]))
    assert np.max(np.abs(o["row_lse"][mask == 1] - O.logprob_entropy_fwd(wide, y)["lse"][mask == 1])) < 1e-12
    dc = P.coef_error(o["row_coef"], o["logp"], old, ref, adv[rt], 1.0 / N, cfg)
    c = OC.dlogits_compare(OC.bf16_bits(lg), y, mask, 1.0, o["row_lse"], o["row_coef"], dc, P.LOGP_ERR,
                           P.DL_REL["bf16"], P.ABS_FLOOR, OC.bf16_bits(got))
    assert np.max(c["max_ratio"][mask == 1]) <= 0.51
    # the C helper's per-row ratio equals the Python one (same formula, independent loops)
    for j in rows:
        lp, H, _, p = O.row_forward(wide[j], int(y[j]))
        q = p.copy()
        q[y[j]] -= 1.0
        rp = P.row_ratio(got[j].double().numpy(), want["dlogits"][j], q, int(y[j]), want["coef"][j], dc[j], "bf16")
        l1 = float(P.l1_ratio(c["l1_err"][j], c["l1_ref"][j], c["l2_ref"][j], c["l1_floor"][j], "bf16"))
        assert abs(max(c["max_ratio"][j], l1) - rp) <= 1e-9 * max(1.0, rp)


def test_zeroed_small_probability_tail_fails():
    """VERDICT r1 'What's weak' 1: a kernel writing 0 for every p < 1e-5 element must fail."""
    lg, tg, wide, y, mask, rt, adv, old, ref, N, cfg, want = _problem()
    j = int(np.flatnonzero(mask)[0])
    _, _, _, p = O.row_forward(wide[j], int(y[j]))
    assert (p < 1e-5).mean() > 0.2
    bad = want["dlogits"].copy()
    bad[j, p < 1e-5] = 0.0
    assert _ratios(_bf16(bad), wide, y, want, [j], adv, rt, old, ref, N, cfg) > 1.0


def test_single_wrong_element_fails():
    lg, tg, wide, y, mask, rt, adv, old, ref, N, cfg, want = _problem()
    j = int(np.flatnonzero(mask)[2])
    _, _, _, p = O.row_forward(wide[j], int(y[j]))
    v = int(np.argmin(p))                        # the smallest-probability element of the row
    bad = want["dlogits"].copy()
    bad[j, v] *= 1.03
    assert _ratios(_bf16(bad), wide, y, want, [j], adv, rt, old, ref, N, cfg) > 1.0


def test_systematic_row_bias_fails_l1_only():
    """A 0.6 % bias of a whole row passes every element (< 2^-7) but fails the row L1 check (> 2^-8), on a row
    whose gradient mass is spread (the uniform row: the Hoeffding term of the L1 bound is small there)."""
    lg, tg, wide, y, mask, rt, adv, old, ref, N, cfg, want = _problem()
    j = 1                                         # the uniform row (make_logits uniform_rows=(1,))
    assert mask[j]
    bad = want["dlogits"].astype(np.float32).copy()
    bad[j] *= 1.0 + 2.0 ** -7.4                  # below the per-element 2^-7, above the L1 2^-8
    got = torch.from_numpy(bad)
    lp, H, _, p = O.row_forward(wide[j], int(y[j]))
    q = p.copy()
    q[y[j]] -= 1.0
    dc = float(P.coef_error(want["coef"][j], lp, old[j], ref[j], adv[rt[j]], 1.0 / N, cfg))
    d = np.abs(bad[j].astype(np.float64) - want["dlogits"][j])
    assert np.max(d / (P.DL_REL["bf16"] * np.abs(want["dlogits"][j]) + dc * np.abs(q) + P.ABS_FLOOR)) <= 1.0
    assert P.row_ratio(got[j].double().numpy(), want["dlogits"][j], q, int(y[j]), want["coef"][j], dc, "bf16") > 1.0


def test_wrong_branch_fails_unless_on_a_kink():
    lg, tg, wide, y, mask, rt, adv, old, ref, N, cfg, want = _problem()
    j = int(np.flatnonzero(mask)[1])
    lp = want["logp"][j]
    A = adv[rt[j]]
    cands = P.branch_coefs(lp, float(old[j]), float(ref[j]), A, 1.0 / N, cfg)
    assert any(abs(c - want["coef"][j]) <= 1e-15 * abs(want["coef"][j]) for c in cands)
    assert not P.near_kink(lp, float(old[j]), float(ref[j]), A, cfg)
    other = max(cands, key=lambda c: abs(c - want["coef"][j]))     # the PPO branch switched
    _, _, _, p = O.row_forward(wide[j], int(y[j]))
    q = p.copy()
    q[y[j]] -= 1.0
    dc = float(P.coef_error(want["coef"][j], lp, old[j], ref[j], A, 1.0 / N, cfg))
    g = _bf16(other * q).double().numpy()
    assert P.row_ratio(g, want["dlogits"][j], q, int(y[j]), want["coef"][j], dc, "bf16") > 1.0
    # a row placed on the clip boundary r = 1 + eps is a kink: both branches are offered
    old_k = lp - math.log(1.2)
    assert P.near_kink(lp, old_k, float(ref[j]), abs(A), cfg)


def test_microbatch_parity_flow_on_cpu():
    """The all-row flow used by tests/test_gpu_fullsize.py and bench.py, on CPU tensors."""
    lg, tg, wide, y, mask, rt, adv, old, ref, N, cfg, want = _problem(n=40, V=2048, seed=9)
    got = _bf16(want["dlogits"])
    st = dict(loss=want["loss"], n_clipped=want["stats"]["n_clipped"], n_tokens=int(mask.sum()))
    lp = torch.from_numpy(want["logp"]).float()
    H = torch.from_numpy(want["entropy"]).float()
    par = P.microbatch_parity(lg, tg, mask, rt, adv, old, ref, N, cfg, "bf16", 2048, lp, H, got, st, chunk=16)
    assert P.parity_ok(par), par
    bad = got.clone()
    bad[np.flatnonzero(mask)[5], :100] = 0
    par = P.microbatch_parity(lg, tg, mask, rt, adv, old, ref, N, cfg, "bf16", 2048, lp, H, bad, st, chunk=16)
    assert not P.parity_ok(par)
    bad = got.clone()
    bad[3, 0] = 1e-20                             # a masked row not exactly zero
    par = P.microbatch_parity(lg, tg, mask, rt, adv, old, ref, N, cfg, "bf16", 2048, lp, H, bad, st, chunk=16)
    assert par["masked_rows_nonzero"] == 1 and not P.parity_ok(par)


def test_underflow_below_smallest_normal_is_tolerated():
    """A logit 90 above the rest: the other elements' gradient (~1e-45) is below fp32 / bf16 normals and may flush to
    0 (oracle/parity.py ABS_FLOOR); an element above that range set to 0 still fails."""
    V = 1024
    x = np.zeros(V)
    x[5] = 90.0
    lp, H, lse, p = O.row_forward(x, 7)
    coef = -1e-5
    q = p.copy()
    q[7] -= 1.0
    want = coef * q
    got = want.copy()
    got[np.abs(want) < 2.0 ** -126] = 0.0
    assert (got == 0).sum() > 1000
    assert P.row_ratio(got, want, q, 7, coef, 1e-10, "f32") <= 1.0
    got[5] = 0.0
    assert P.row_ratio(got, want, q, 7, coef, 1e-10, "f32") > 1.0


def test_lmhead_flip_tolerance_covers_flipped_roundings():
    """The LM-head dh / dW flip allowance (oracle/parity.py lmhead_flip_tolerance, R34): flipping EVERY
    ambiguous logit to its other bf16 neighbour moves the float64 oracle's dh and dW by no more than the allowance;
    a flipped NON-ambiguous logit (a wrong rounding, not an accumulation-order effect) is not covered."""
    from synth import make_lmhead
    N, V, d = 96, 1024, 128
    h, w, y = make_lmhead(N, V, d, seed=4)
    H, Wm, yy = h.double().numpy(), w.double().numpy(), y.numpy()
    x64 = H @ Wm.T
    xb = torch.from_numpy(x64).to(torch.bfloat16).double().numpy()
    rng = np.random.default_rng(1)
    mask = (rng.random(N) < 0.8).astype(np.uint8)
    rt = np.zeros(N, np.int32)
    adv = np.array([0.9])
    lp0 = np.array([O.row_forward(xb[j], int(yy[j]))[0] for j in range(N)])
    old, ref = lp0 + 0.05, lp0 - 0.1
    cfg = O.LossCfg(kl_beta=0.04)
    n = int(mask.sum())
    want = O.policy_loss_fwd_bwd(xb, yy, mask, rt, adv, old, ref, n, cfg)
    args = (H, Wm, x64, xb, yy, want["coef"], want["logp"], old, ref, adv[rt], np.full(N, 1.0 / n), cfg, mask)
    # a widened accumulation bound (as if d were 2^16) makes hundreds of logits ambiguous
    tdh, tdW, n_amb, amb = P.lmhead_flip_tolerance(*args, acc_terms=2 ** 16)
    assert n_amb > 100
    u = P.bf16_ulp(xb)
    side = np.where(x64 >= xb, 1.0, -1.0)
    alt = O.policy_loss_fwd_bwd(np.where(amb, xb + side * u, xb), yy, mask, rt, adv, old, ref, n, cfg)
    ddx = alt["dlogits"] - want["dlogits"]
    assert np.all(np.abs(ddx @ Wm) <= tdh) and np.all(np.abs(ddx.T @ H) <= tdW)
    assert np.max(np.abs(ddx @ Wm) / np.maximum(tdh, 1e-300)) > 0.05   # the allowance is not vacuous
    # a flip outside the (real-d) ambiguous set is not covered: the largest trainable dx element, rounded the other way
    t_dh, _, _, amb_d = P.lmhead_flip_tolerance(*args)
    dx0 = want["dlogits"]
    j, v = np.unravel_index(np.argmax(np.where(amb_d | (mask[:, None] == 0), 0, np.abs(dx0))), dx0.shape)
    xw = xb.copy()
    xw[j, v] += side[j, v] * u[j, v]
    bad = O.policy_loss_fwd_bwd(xw, yy, mask, rt, adv, old, ref, n, cfg)["dlogits"]
    assert np.max(np.abs((bad - dx0) @ Wm) - 2.0 ** -8 * np.abs(dx0 @ Wm) - t_dh) > 0
