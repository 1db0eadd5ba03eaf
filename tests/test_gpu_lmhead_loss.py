"""Policy loss through the LM head (step.LMHeadPolicyLoss: cuBLAS GEMMs around otk_policy_loss_fwd_bwd) vs the
float64 oracle on the same bf16 h and W (-m gpu): loss within 1e-3 relative (the logits are rounded to bf16 before
the loss, as in any bf16 head), dh and dW within 2e-2 in relative Frobenius norm (bf16 logits, bf16 dx, fp32
accumulation over V = 4096 / N = 512 terms)."""
import numpy as np
import pytest
import torch

from oracle import oracle_ref as O
from synth import make_lmhead, make_noise

pytestmark = pytest.mark.gpu


def test_lmhead_policy_loss_vs_oracle():
    import paper_2601_07376_b200 as otk
    from paper_2601_07376_b200.step import LMHeadPolicyLoss
    ctx = otk.Context(0)
    N, V, d, s = 512, 4096, 256, 1.0
    h, w, y = make_lmhead(N, V, d, seed=11)
    rng = np.random.default_rng(5)
    mask = (rng.random(N) < 0.7).astype(np.uint8)
    rt = np.sort(rng.integers(0, 8, N)).astype(np.int32)
    adv = rng.normal(size=8)
    # the oracle's logits: the same bf16 operands in float64, rounded to bf16 like the head's output
    x64 = h.double().numpy() @ w.double().numpy().T
    xb = torch.from_numpy(x64).to(torch.bfloat16).double().numpy()
    lp0 = np.array([O.row_forward(xb[j], int(y[j]), s)[0] for j in range(N)])
    old = (lp0 + make_noise(N, 0.05, 1).double().numpy()).astype(np.float32)
    ref = (lp0 + make_noise(N, 0.1, 2).double().numpy()).astype(np.float32)
    cfg = otk.LossCfg(kl_beta=0.04, logit_scale=s)
    n_loss = int(mask.sum())
    want = O.policy_loss_fwd_bwd(xb, y.numpy(), mask, rt, adv, old.astype(np.float64), ref.astype(np.float64), n_loss,
                                 O.LossCfg(kl_beta=0.04, logit_scale=s))
    dx = np.array([want["dlogits"][j] for j in range(N)])
    dh_ref = dx @ w.double().numpy()
    dW_ref = dx.T @ h.double().numpy()
    dev = "cuda"
    step = LMHeadPolicyLoss(ctx)
    out = step(h.to(dev), w.to(dev), y.to(dev), torch.from_numpy(mask).to(dev), torch.from_numpy(rt).to(dev),
               torch.from_numpy(adv).to(dev), torch.from_numpy(old).to(dev), torch.from_numpy(ref).to(dev),
               torch.tensor([n_loss], dtype=torch.int64, device=dev), cfg, timings=True)
    ctx.check()
    loss = otk.stats_dict(out["stats"])["loss"]
    assert abs(loss - want["loss"]) <= 1e-3 * max(abs(want["loss"]), 1e-3), (loss, want["loss"])
    for got, ref_ in ((out["dh"], dh_ref), (out["dW"], dW_ref)):
        g = got.double().cpu().numpy()
        assert np.linalg.norm(g - ref_) <= 2e-2 * np.linalg.norm(ref_)
    assert set(out["ms"]) == {"logits_gemm", "loss_kernel", "grad_gemms"}
    ctx.close()
