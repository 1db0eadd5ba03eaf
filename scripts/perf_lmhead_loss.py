"""Policy loss through the LM head, two implementations on the same inputs (DESIGN.md §6 "LM head, backward"):
  cublas: step.LMHeadPolicyLoss — logits GEMM (cuBLAS), the fused loss kernel (4), dh / dW GEMMs (cuBLAS), with the
          time split;
  fused:  step.LMHeadPolicyLossFused — otk_lmhead_policy_loss_fwd_bwd (tcgen05 x GEMM + loss rows + tcgen05 dh / dW
          with dx formed in shared memory), timed as one call.
Usage: python scripts/perf_lmhead_loss.py [--rows 8192] [--d 3584] [--impl both|cublas|fused]"""
import argparse, json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2601_07376_b200 as otk
from paper_2601_07376_b200.step import LMHeadPolicyLoss, LMHeadPolicyLossFused
from synth import make_lmhead, make_noise
ap = argparse.ArgumentParser(); ap.add_argument("--rows", type=int, default=8192); ap.add_argument("--d", type=int, default=3584)
ap.add_argument("--vocab", type=int, default=151936); ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--impl", default="both")
a = ap.parse_args()
torch.cuda.set_device(0)
ctx = otk.Context(0)
N, V, d = a.rows, a.vocab, a.d
h, w, y = make_lmhead(N, V, d, seed=1, device="cuda")
mask = (torch.rand(N, device="cuda") < 0.5).to(torch.uint8)
rt = torch.arange(N, device="cuda", dtype=torch.int32) // 512
adv = torch.randn(N // 512 + 1, device="cuda", dtype=torch.float64)
lp = otk.otk_lmhead_logprob_fwd(ctx, h, w, y)["logp"]
old = (lp + make_noise(N, 0.05, 1, device="cuda")).contiguous()
ref = (lp + make_noise(N, 0.1, 2, device="cuda")).contiguous()
nl = mask.sum().to(torch.int64).reshape(1)
cfg = otk.LossCfg(kl_beta=0.04)


CLOCKS = {}


def back_to_back(step, name=None):
    """ms per call of `iters` calls enqueued back to back (no host sync in between, so host-side argument
    marshalling overlaps the previous call's kernels — the device time, as bench.py measures a step); the SM clock
    is sampled meanwhile (bench.py's NVML sampler) into CLOCKS[name]."""
    from bench import ClockSampler
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with ClockSampler(0) as cs:
        e0.record()
        for _ in range(a.iters):
            step(h, w, y, mask, rt, adv, old, ref, nl, cfg)
        e1.record()
        torch.cuda.synchronize()
    if name:
        CLOCKS[name] = cs.summary()
    return e0.elapsed_time(e1) / a.iters


flops_gemm = 2.0 * N * V * d
res = dict(rows=N, vocab=V, hidden_dim=d)
if a.impl in ("both", "cublas"):
    step = LMHeadPolicyLoss(ctx)
    for _ in range(2):
        step(h, w, y, mask, rt, adv, old, ref, nl, cfg)
    acc = {}
    for _ in range(a.iters):
        o = step(h, w, y, mask, rt, adv, old, ref, nl, cfg, timings=True)
        for k, v in o["ms"].items():
            acc[k] = acc.get(k, 0.0) + v / a.iters
    ctx.check()
    tot = back_to_back(step, "cublas")
    res["cublas"] = dict(ms={k: round(v, 4) for k, v in acc.items()}, total_ms=round(tot, 4),
                         loss_kernel_share=round(acc["loss_kernel"] / tot, 4),
                         gemm_TFLOPs=round(3 * flops_gemm / (acc["logits_gemm"] + acc["grad_gemms"]) / 1e9, 1),
                         step_TFLOPs=round(3 * flops_gemm / tot / 1e9, 1))
    ref_out = o
    del step
if a.impl in ("both", "fused"):
    step = LMHeadPolicyLossFused(ctx)
    for _ in range(2):
        step(h, w, y, mask, rt, adv, old, ref, nl, cfg)
    t = back_to_back(step, "fused")
    o = step(h, w, y, mask, rt, adv, old, ref, nl, cfg)
    torch.cuda.synchronize()
    ctx.check()
    res["fused"] = dict(total_ms=round(t, 4), step_TFLOPs=round(3 * flops_gemm / t / 1e9, 1))
    if a.impl == "both":
        # the two implementations on the same inputs: loss and gradients agree within the bf16 budget
        lc = otk.stats_dict(ref_out["stats"])["loss"]
        lf = otk.stats_dict(o["stats"])["loss"]
        res["agree"] = dict(loss_rel=abs(lc - lf) / max(abs(lc), 1e-12),
                            dh_rel_fro=float((o["dh"].float() - ref_out["dh"].float()).norm() / ref_out["dh"].float().norm()),
                            dW_rel_fro=float((o["dW"].float() - ref_out["dW"].float()).norm() / ref_out["dW"].float().norm()))
        res["speedup_fused_vs_cublas"] = round(res["cublas"]["total_ms"] / t, 4)
res["clocks"] = CLOCKS
print(json.dumps(res))
