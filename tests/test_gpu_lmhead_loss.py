"""Policy loss through the LM head (step.LMHeadPolicyLoss: cuBLAS GEMMs around otk_policy_loss_fwd_bwd) vs the
float64 oracle on the same bf16 h and W (-m gpu): loss within 1e-3 relative (the logits are rounded to bf16 before
the loss, as in any bf16 head), and dh, dW ELEMENT-WISE:
    |d - ref| <= 2^-8 |ref| + 6 * 2^-8 * sqrt(sum_v (dx_jv W_vi)^2)      (dW: the same with h)
dx carries independent per-element rounding errors (<= 2^-7 relative, mean ~2^-9) and a bf16 logit
may round to the neighbouring value (fp32 vs float64 accumulation), so the error of a sum over V terms has a spread
of ~2^-9 sqrt(sum (dx W)^2); the output is rounded once more to bf16 (2^-8 |ref|). 6 x 2^-8 is ~12 of those
spreads; a CPU emulation of the roundings reached 0.40 of this bound."""
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
    W, H = w.double().numpy(), h.double().numpy()
    for got, ref_, spread in ((out["dh"], dh_ref, np.sqrt((dx ** 2) @ (W ** 2))),
                              (out["dW"], dW_ref, np.sqrt((dx.T ** 2) @ (H ** 2)))):
        g = got.double().cpu().numpy()
        d_ = np.abs(g - ref_)
        tol = 2.0 ** -8 * np.abs(ref_) + 6 * 2.0 ** -8 * spread
        ratio = np.where(d_ == 0, 0.0, d_ / np.maximum(tol, 1e-300))
        assert float(ratio.max()) <= 1.0, float(ratio.max())
    # rows with loss mask 0 contribute nothing: their dh rows are exactly 0
    assert bool((out["dh"][torch.from_numpy(mask == 0).to(dev)] == 0).all())
    assert set(out["ms"]) == {"logits_gemm", "loss_kernel", "grad_gemms"}
    ctx.close()
