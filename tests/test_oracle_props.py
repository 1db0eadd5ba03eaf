"""Randomised invariants of the float64 oracle (-m "not gpu"; hypothesis, SURVEY.md §4 "property tests"). Each
property follows from the definitions, not from the oracle's code: softmax - onehot sums to zero over the
vocabulary (so does the entropy-bonus term p(ln p + H)); logp <= 0 and 0 <= H <= ln V; a constant shift of a
row's logits changes nothing; on-policy with beta = 0 the token-mean loss is -sum(m_j A_j)/N; the gradient
matches central finite differences of the loss."""
import math

import numpy as np
from hypothesis import given, settings, strategies as st

from oracle import oracle_ref as O


def _problem(seed, n, V, scale):
    rng = np.random.default_rng(seed)
    x = rng.normal(scale=scale, size=(n, V))
    y = rng.integers(0, V, n)
    mask = (rng.random(n) < 0.7).astype(np.uint8)
    if mask.sum() == 0:
        mask[0] = 1
    rt = np.sort(rng.integers(0, 3, n)).astype(np.int32)
    adv = rng.normal(size=3)
    return rng, x, y, mask, rt, adv


@settings(max_examples=40, deadline=None, derandomize=True)
@given(seed=st.integers(0, 2**31 - 1), n=st.integers(1, 12), V=st.integers(2, 300),
       scale=st.floats(0.1, 8.0), s=st.floats(0.25, 2.0), ent=st.sampled_from([0.0, 0.01]),
       beta=st.sampled_from([0.0, 0.04]))
def test_gradient_rows_sum_to_zero_and_ranges(seed, n, V, scale, s, ent, beta):
    rng, x, y, mask, rt, adv = _problem(seed, n, V, scale)
    lp = np.array([O.row_forward(x[j], int(y[j]), s)[0] for j in range(n)])
    old = lp + rng.normal(scale=0.05, size=n)
    ref = lp + rng.normal(scale=0.1, size=n)
    cfg = O.LossCfg(kl_beta=beta, logit_scale=s, ent_coef=ent)
    out = O.policy_loss_fwd_bwd(x, y, mask, rt, adv, old, ref if beta else None, int(mask.sum()), cfg)
    for j in range(n):
        assert abs(math.fsum(out["dlogits"][j])) <= 1e-12 * max(1.0, float(np.abs(out["dlogits"][j]).sum()))
        if mask[j]:
            assert out["logp"][j] <= 1e-15
            assert -1e-12 <= out["entropy"][j] <= math.log(V) + 1e-12
        else:
            assert not np.any(out["dlogits"][j])


@settings(max_examples=40, deadline=None, derandomize=True)
@given(seed=st.integers(0, 2**31 - 1), n=st.integers(1, 8), V=st.integers(2, 200), c=st.floats(-50.0, 50.0))
def test_shift_invariance(seed, n, V, c):
    rng, x, y, mask, rt, adv = _problem(seed, n, V, 2.0)
    a = O.logprob_entropy_fwd(x, y)
    b = O.logprob_entropy_fwd(x + c, y)
    assert np.allclose(a["logp"], b["logp"], atol=1e-10) and np.allclose(a["entropy"], b["entropy"], atol=1e-10)


@settings(max_examples=40, deadline=None, derandomize=True)
@given(seed=st.integers(0, 2**31 - 1), n=st.integers(1, 10), V=st.integers(2, 100))
def test_on_policy_loss_is_minus_mean_advantage(seed, n, V):
    rng, x, y, mask, rt, adv = _problem(seed, n, V, 1.5)
    lp = np.array([O.row_forward(x[j], int(y[j]))[0] for j in range(n)])
    N = int(mask.sum())
    out = O.policy_loss_fwd_bwd(x, y, mask, rt, adv, lp, None, N, O.LossCfg(kl_beta=0.0))
    want = -math.fsum(float(adv[rt[j]]) for j in range(n) if mask[j]) / N
    assert abs(out["loss"] - want) <= 1e-12 * max(1.0, abs(want))


@settings(max_examples=15, deadline=None, derandomize=True)
@given(seed=st.integers(0, 2**31 - 1), V=st.integers(2, 12), s=st.floats(0.5, 1.5),
       beta=st.sampled_from([0.0, 0.04]), ent=st.sampled_from([0.0, 0.02]))
def test_gradient_matches_finite_differences(seed, V, s, beta, ent):
    n = 3
    rng, x, y, mask, rt, adv = _problem(seed, n, V, 1.0)
    lp = np.array([O.row_forward(x[j], int(y[j]), s)[0] for j in range(n)])
    old = lp + rng.normal(scale=0.02, size=n)      # near on-policy: away from the clip kinks
    ref = lp + rng.normal(scale=0.05, size=n)
    N = int(mask.sum())
    cfg = O.LossCfg(kl_beta=beta, logit_scale=s, ent_coef=ent)
    base = O.policy_loss_fwd_bwd(x, y, mask, rt, adv, old, ref if beta else None, N, cfg)
    h = 1e-6
    for j in range(n):
        r_ = math.exp(base["logp"][j] - old[j]) if mask[j] else 1.0
        if abs(r_ - 1.2) < 1e-3 or abs(r_ - 0.8) < 1e-3:
            continue                                  # at a clip kink the loss is not differentiable
        for v in range(V):
            xp, xm = x.copy(), x.copy()
            xp[j, v] += h
            xm[j, v] -= h
            lp_ = O.policy_loss_fwd_bwd(xp, y, mask, rt, adv, old, ref if beta else None, N, cfg)["loss"]
            lm_ = O.policy_loss_fwd_bwd(xm, y, mask, rt, adv, old, ref if beta else None, N, cfg)["loss"]
            fd = (lp_ - lm_) / (2 * h)
            g = base["dlogits"][j][v]
            assert abs(fd - g) <= 1e-6 + 1e-4 * abs(g), (j, v, fd, g)
