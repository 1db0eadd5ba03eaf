"""Calls of the fused LM-head policy loss (otk_lmhead_policy_loss_fwd_bwd) for ncu:
python scripts/prof_lmhead_loss.py [rows] [d] [calls]"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2601_07376_b200 as otk
from paper_2601_07376_b200.step import LMHeadPolicyLossFused
from synth import make_lmhead, make_noise
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
d = int(sys.argv[2]) if len(sys.argv) > 2 else 3584
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 2
V = 151936
ctx = otk.Context(0)
h, w, y = make_lmhead(n, V, d, seed=1, device="cuda")
mask = (torch.rand(n, device="cuda") < 0.5).to(torch.uint8)
rt = torch.arange(n, device="cuda", dtype=torch.int32) // 512
adv = torch.randn(n // 512 + 1, device="cuda", dtype=torch.float64)
lp = otk.otk_lmhead_logprob_fwd(ctx, h, w, y)["logp"]
old = (lp + make_noise(n, 0.05, 1, device="cuda")).contiguous()
ref = (lp + make_noise(n, 0.1, 2, device="cuda")).contiguous()
nl = mask.sum().to(torch.int64).reshape(1)
step = LMHeadPolicyLossFused(ctx)
for _ in range(calls):
    step(h, w, y, mask, rt, adv, old, ref, nl, otk.LossCfg(kl_beta=0.04))
torch.cuda.synchronize()
ctx.check()
