"""Time split of the policy loss through the LM head (step.LMHeadPolicyLoss): logits GEMM (cuBLAS), the fused
loss kernel (4), and the dh / dW GEMMs (cuBLAS) — the evidence behind DESIGN.md §10 (why the backward half of
NEXT-1 is not fused). Usage: python scripts/perf_lmhead_loss.py [--rows 8192] [--d 3584]"""
import argparse, json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2601_07376_b200 as otk
from paper_2601_07376_b200.step import LMHeadPolicyLoss
from synth import make_lmhead, make_noise
ap = argparse.ArgumentParser(); ap.add_argument("--rows", type=int, default=8192); ap.add_argument("--d", type=int, default=3584)
ap.add_argument("--vocab", type=int, default=151936); ap.add_argument("--iters", type=int, default=5)
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
step = LMHeadPolicyLoss(ctx)
cfg = otk.LossCfg(kl_beta=0.04)
for _ in range(2):
    step(h, w, y, mask, rt, adv, old, ref, nl, cfg)
acc = {}
for _ in range(a.iters):
    o = step(h, w, y, mask, rt, adv, old, ref, nl, cfg, timings=True)
    for k, v in o["ms"].items():
        acc[k] = acc.get(k, 0.0) + v / a.iters
ctx.check()
flops_gemm = 2.0 * N * V * d
tot = sum(acc.values())
print(json.dumps(dict(rows=N, vocab=V, hidden_dim=d, ms={k: round(v, 4) for k, v in acc.items()}, total_ms=round(tot, 4),
                      loss_kernel_share=round(acc["loss_kernel"] / tot, 4),
                      gemm_TFLOPs=round(3 * flops_gemm / (acc["logits_gemm"] + acc["grad_gemms"]) / 1e9, 1),
                      recompute_gemm_ms_est=round(acc["logits_gemm"], 4),
                      logits_traffic_ms_est=round(8 * N * V / 6.454e12 * 1e3, 4))))
