"""The C oracle (oracle/oracle_cpu.c) against the pinned Python oracle and the closed forms."""
import math

import numpy as np
import pytest
import torch

from oracle import oracle_cpu as OC
from oracle import oracle_ref as O
from synth import make_batch, make_logits
from tests.conftest import load_golden

CF = {k: float(v) for k, v in load_golden("closed_forms.txt").items()}


def test_closed_forms_c():
    V = 151936
    x = np.zeros((2, V), np.float32)
    x[1, 3] = 10.0
    out = OC.logprob_entropy(x, [7, 3])
    assert abs(out["logp"][0] - CF["uniform_logp_V151936"]) < 1e-12
    assert abs(out["entropy"][0] + CF["uniform_logp_V151936"]) < 1e-12
    assert abs(out["logp"][1] - CF["twolevel_V151936_L10_logp"]) < 1e-11
    assert abs(out["entropy"][1] - CF["twolevel_V151936_L10_H"]) < 1e-11


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_c_matches_python_oracle(dtype):
    n, V = 24, 1000
    lg, tg = make_logits(n, V, ld=1008, dtype=dtype, seed=3)
    arr = lg.numpy() if dtype == "f32" else OC.bf16_bits(lg)
    wide = lg.to(torch.float64).numpy()[:, :V]
    rng = np.random.default_rng(0)
    mask = (rng.random(n) < 0.6).astype(np.uint8)
    rt = np.arange(n, dtype=np.int32) // 6
    adv = rng.normal(size=4)
    ref_py = O.logprob_entropy_fwd(wide, tg.numpy(), logit_scale=1 / 0.7)
    old = (ref_py["logp"] + rng.normal(scale=0.1, size=n)).astype(np.float32)
    ref = (ref_py["logp"] + rng.normal(scale=0.1, size=n)).astype(np.float32)
    c = OC.logprob_entropy(arr, tg.numpy(), V=V, logit_scale=1 / 0.7)
    assert np.max(np.abs(c["logp"] - ref_py["logp"])) < 1e-12
    assert np.max(np.abs(c["entropy"] - ref_py["entropy"])) < 1e-12
    for kl_type in (1, 2, 3):
        cfg = O.LossCfg(kl_type=kl_type, logit_scale=1 / 0.7)
        N = int(mask.sum())
        py = O.policy_loss_fwd_bwd(wide, tg.numpy(), mask, rt, adv, old.astype(np.float64),
                                   ref.astype(np.float64), N, cfg)
        cc = OC.policy_loss(arr, tg.numpy(), mask, rt, adv, old, ref, N, cfg, V=V)
        assert np.max(np.abs(cc["dlogits"] - py["dlogits"])) < 1e-15
        assert abs(math.fsum(cc["row_L"]) / N - py["loss"]) < 1e-13
        assert int(cc["row_clipped"].sum()) == py["stats"]["n_clipped"]


@pytest.mark.parametrize("name", ["tiny", "marl"])
def test_c_masks_match_python(name):
    tb = make_batch(name)
    a = OC.build_masks(tb)
    b = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len,
                      tb.terminated, traj_agent=tb.traj_agent)
    for k in ("loss_mask", "response_mask", "row_traj", "traj_loss_tokens"):
        assert np.array_equal(a[k], b[k])
    assert a["n_loss"] == b["n_loss"]
