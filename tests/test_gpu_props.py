"""Randomised parity of the fused kernels against the float64 oracle (-m gpu; hypothesis, SURVEY.md §4 "unit …
hypothesis-generated small cases"): random vocabulary sizes (ragged tails, odd V, 16-byte padded rows), row
counts, logit scales, masks, KL forms and dtypes, through the C ABI. Tolerances as tests/test_gpu_parity.py."""
import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings, strategies as st

from oracle import oracle_ref as O
from tests.gpu_common import LOGP_TOL, check_dlogits_rows, dcoef_rows, near_kink, oracle_cfg, row_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def otk():
    import paper_2601_07376_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(otk):
    c = otk.Context(0)
    yield c
    c.close()


@settings(max_examples=30, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(V=st.integers(2, 5000), n=st.integers(1, 40), dtype=st.sampled_from(["bf16", "f32"]),
       scale=st.floats(0.5, 2.0), beta=st.sampled_from([0.0, 0.04]), kl=st.sampled_from([1, 2, 3]),
       seed=st.integers(0, 10**6))
def test_random_loss_vs_oracle(otk, ctx, V, n, dtype, scale, beta, kl, seed):
    align = 8 if dtype == "bf16" else 4
    ld = -(-V // align) * align
    d, h = row_problem(n, V, dtype=dtype, ld=ld, seed=seed, logit_scale=scale)
    cfg = otk.LossCfg(kl_beta=beta, kl_type=kl, logit_scale=scale)
    N = int(h["mask"].sum())
    nl = torch.tensor([N], dtype=torch.int64, device="cuda")
    got = otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"], d["old"],
                                      d["ref"] if beta else None, nl, cfg, vocab=V)
    f = otk.otk_logprob_entropy_fwd(ctx, d["logits"], d["targets"], vocab=V, logit_scale=scale)
    ctx.check()
    ocfg = oracle_cfg(cfg)
    want = O.policy_loss_fwd_bwd(h["wide"], h["targets"], h["mask"], h["row_traj"], h["adv"], h["old"],
                                 h["ref"] if beta else None, N, ocfg)
    fw = O.logprob_entropy_fwd(h["wide"], h["targets"], logit_scale=scale)
    tol = LOGP_TOL[dtype]
    assert np.max(np.abs(f["logp"].cpu().numpy() - fw["logp"])) < tol
    assert np.max(np.abs(f["entropy"].cpu().numpy() - fw["entropy"])) < tol
    m = h["mask"].astype(bool)
    assert np.all(f["logp"].cpu().numpy()[m] == got["logp"].cpu().numpy()[m])   # (3) and (4): bitwise equal logp
    kinks = {j for j in range(n) if m[j] and near_kink(want["logp"][j], h["old"][j], h["ref"][j] if beta else None,
                                                       h["adv"][h["row_traj"][j]], ocfg)}
    rows = [j for j in range(n) if m[j]]
    dc = dcoef_rows(h, want["logp"], ocfg, N, beta)
    assert check_dlogits_rows(got["dlogits"], want["dlogits"], want["coef"], rows, dtype, V, dc, wide=h["wide"],
                              targets=h["targets"], scale=scale, h=h, cfg=ocfg) <= 1.0
    if N:
        st_ = otk.stats_dict(got["stats"])
        scale_ = max(abs(want["loss"]), sum(abs(O.row_loss_terms(want["logp"][j], h["old"][j],
                                                                 h["ref"][j] if beta else None,
                                                                 h["adv"][h["row_traj"][j]], ocfg)[0])
                                            for j in range(n) if m[j]) / N)
        assert abs(st_["loss"] - want["loss"]) <= 1e-4 * scale_           # L is continuous across the kinks
        assert abs(st_["n_clipped"] - want["stats"]["n_clipped"]) <= len(kinks)
