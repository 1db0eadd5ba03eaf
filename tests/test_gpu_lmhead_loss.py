"""Policy loss through the LM head — step.LMHeadPolicyLoss (cuBLAS GEMMs around otk_policy_loss_fwd_bwd) and
step.LMHeadPolicyLossFused (otk_lmhead_policy_loss_fwd_bwd: tcgen05 fwd + bwd, dx formed on chip) — vs the
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
from oracle import parity as P
from synth import make_lmhead, make_noise

pytestmark = pytest.mark.gpu


def _run_case(impl, N, V, d, seed=11, s=1.0, mask_p=0.7, **cfg_kw):
    import paper_2601_07376_b200 as otk
    from paper_2601_07376_b200.step import LMHeadPolicyLoss, LMHeadPolicyLossFused
    ctx = otk.Context(0)
    h, w, y = make_lmhead(N, V, d, seed=seed)
    rng = np.random.default_rng(seed + 5)
    mask = (rng.random(N) < mask_p).astype(np.uint8)
    rt = np.sort(rng.integers(0, 8, N)).astype(np.int32)
    adv = rng.normal(size=8)
    # the oracle's logits: the same bf16 operands in float64, rounded to bf16 like the head's output
    x64 = h.double().numpy() @ w.double().numpy().T
    xb = torch.from_numpy(x64).to(torch.bfloat16).double().numpy()
    lp0 = np.array([O.row_forward(xb[j], int(y[j]), s)[0] for j in range(N)])
    old = (lp0 + make_noise(N, 0.05, 1).double().numpy()).astype(np.float32)
    ref = (lp0 + make_noise(N, 0.1, 2).double().numpy()).astype(np.float32)
    cfg = otk.LossCfg(kl_beta=0.04, logit_scale=s, **cfg_kw)
    n_loss = int(mask.sum())
    want = O.policy_loss_fwd_bwd(xb, y.numpy(), mask, rt, adv, old.astype(np.float64), ref.astype(np.float64), n_loss,
                                 O.LossCfg(kl_beta=0.04, logit_scale=s, **cfg_kw))
    dx = np.array([want["dlogits"][j] for j in range(N)])
    dh_ref = dx @ w.double().numpy()
    dW_ref = dx.T @ h.double().numpy()
    dev = "cuda"
    step = (LMHeadPolicyLoss if impl == "cublas" else LMHeadPolicyLossFused)(ctx)
    out = step(h.to(dev), w.to(dev), y.to(dev), torch.from_numpy(mask).to(dev), torch.from_numpy(rt).to(dev),
               torch.from_numpy(adv).to(dev), torch.from_numpy(old).to(dev), torch.from_numpy(ref).to(dev),
               torch.tensor([n_loss], dtype=torch.int64, device=dev), cfg, timings=True)
    ctx.check()
    loss = otk.stats_dict(out["stats"])["loss"]
    assert abs(loss - want["loss"]) <= 1e-3 * max(abs(want["loss"]), 1e-3), (loss, want["loss"])
    W, H = w.double().numpy(), h.double().numpy()
    ocfg = O.LossCfg(kl_beta=0.04, logit_scale=s, **cfg_kw)
    flip_dh, flip_dW, n_amb, _ = P.lmhead_flip_tolerance(
        H, W, x64, xb, y.numpy(), want["coef"], want["logp"], old.astype(np.float64), ref.astype(np.float64),
        adv[rt], np.full(N, 1.0 / max(n_loss, 1)), ocfg, mask)
    worst = {}
    for name, got, ref_, spread, flip in (("dh", out["dh"], dh_ref, np.sqrt((dx ** 2) @ (W ** 2)), flip_dh),
                                          ("dW", out["dW"], dW_ref, np.sqrt((dx.T ** 2) @ (H ** 2)), flip_dW)):
        g = got.double().cpu().numpy()
        assert g.shape == ref_.shape
        d_ = np.abs(g - ref_)
        tol = 2.0 ** -8 * np.abs(ref_) + 6 * 2.0 ** -8 * spread + flip
        ratio = np.where(d_ == 0, 0.0, d_ / np.maximum(tol, 1e-300))
        worst[name] = float(ratio.max())
    assert max(worst.values()) <= 1.0, (worst, n_amb)
    # rows with loss mask 0 contribute nothing: their dh rows are exactly 0
    assert bool((out["dh"][torch.from_numpy(mask == 0).to(dev)] == 0).all())
    if impl == "fused":
        # logp / entropy of the trainable rows: the float64 oracle on the bf16 logits, 2e-3 (north_star)
        m = mask != 0
        assert np.max(np.abs(out["logp"].cpu().numpy()[m] - want["logp"][m])) < 2e-3
        # the x the call wrote is a bf16 rounding of h W^T: within the fp32 accumulation bound (d 2^-24 sum|h W|)
        # of the float64 product, then one rounding (half a bf16 ulp of the result)
        xg = otk.lmhead_x_from_workspace(out).double().cpu().numpy()
        eps = d * 2.0 ** -24 * (np.abs(H) @ np.abs(W).T)
        assert np.all(np.abs(xg - x64) <= eps + 0.5 * P.bf16_ulp(np.abs(x64) + eps) * (1 + 2.0 ** -8))
    ctx.close()
    return out


@pytest.mark.parametrize("impl", ["cublas", "fused"])
def test_lmhead_policy_loss_vs_oracle(impl):
    out = _run_case(impl, 512, 4096, 256)
    if impl == "cublas":
        assert set(out["ms"]) == {"logits_gemm", "loss_kernel", "grad_gemms"}


@pytest.mark.parametrize("impl", ["cublas", "fused"])
@pytest.mark.parametrize("N,V,d", [(600, 4104, 320),     # ragged rows, vocab not a multiple of 64, d < 512
                                   (257, 2056, 576),      # one row past a tile; d spans two 512-column tiles
                                   (1100, 8192, 1024)])   # several row tiles, split-K dh
def test_lmhead_shapes(impl, N, V, d):
    _run_case(impl, N, V, d, seed=N)


@pytest.mark.parametrize("kw", [dict(ent_coef=0.05), dict(dual_clip=3.0), dict(sft=True)])
def test_lmhead_fused_variants(kw):
    _run_case("fused", 384, 3072, 256, seed=3, **kw)


def test_lmhead_fused_scale_and_masked_rows():
    _run_case("fused", 320, 2048, 192, seed=7, s=0.7, mask_p=0.3)


def test_lmhead_fused_timed_vocab_and_hidden():
    """The timed shape's vocabulary and hidden size (V = 151936: 2374 vocab stages split across dh units; d = 3584: 7
    hidden tiles, the dx store of tile 0 read back by dW) on a ragged 257-row batch (one full 256-row tile + 1)."""
    _run_case("fused", 257, 151936, 3584, seed=17)


def test_lmhead_fused_errors_and_empty():
    """Host-checked errors of otk_lmhead_policy_loss_fwd_bwd return before any launch (otk.h): vocab not a multiple
    of 8, hidden_dim not a multiple of 64, a 16- but not 32-byte-aligned gradient buffer; 0 rows is a no-op."""
    import paper_2601_07376_b200 as otk
    ctx = otk.Context(0)
    dev = "cuda"

    def args(N, V, d):
        h, w, y = make_lmhead(N, V, d, seed=1, device=dev)
        return (h, w, y, torch.ones(N, dtype=torch.uint8, device=dev), torch.zeros(N, dtype=torch.int32, device=dev),
                torch.ones(1, dtype=torch.float64, device=dev), torch.zeros(N, device=dev), torch.zeros(N, device=dev),
                torch.tensor([max(N, 1)], dtype=torch.int64, device=dev))
    with pytest.raises(otk.OtkError) as e:
        otk.otk_lmhead_policy_loss_fwd_bwd(ctx, *args(64, 1028, 128))
    assert e.value.status == 2                                    # OTK_ERR_SHAPE
    with pytest.raises(otk.OtkError) as e:
        otk.otk_lmhead_policy_loss_fwd_bwd(ctx, *args(64, 1024, 96))
    assert e.value.status == 2
    a = args(64, 1024, 128)
    buf = torch.empty(64 * 128 + 8, dtype=torch.bfloat16, device=dev)
    with pytest.raises(otk.OtkError) as e:                        # dhidden at a 16-byte (not 32) offset
        otk.otk_lmhead_policy_loss_fwd_bwd(ctx, *a, dhidden=buf[8:].view(64, 128))
    assert e.value.status == 3                                    # OTK_ERR_ALIGNMENT
    out = otk.otk_lmhead_policy_loss_fwd_bwd(ctx, *args(0, 1024, 128),
                                             stats=torch.full((5,), 7.0, dtype=torch.float64, device=dev))
    ctx.check()
    assert out["dh"].shape == (0, 128)
    assert bool((out["dW"] == 0).all()) and bool((out["stats"] == 0).all())   # empty batch: no gradient, zero stats
    ctx.close()
