"""Experiment: where the fused LM-head backward's time goes (build with -DOTK_BW_TIMING, run with OTK_LIB=that .so).
Prints per kernel: the MMA thread's cycles waiting for B, for the transformed A, for the accumulators, and its
total; a transform warp's cycles waiting for A, transforming, and in the epilogue (per CTA averages)."""
import ctypes, json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2601_07376_b200 as otk
from paper_2601_07376_b200.step import LMHeadPolicyLossFused
from synth import make_lmhead, make_noise
n, d, V = int(sys.argv[1]), int(sys.argv[2]), 151936
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
fn = otk._lib.otk_debug_bw
buf = (ctypes.c_ulonglong * 32)()
step(h, w, y, mask, rt, adv, old, ref, nl, otk.LossCfg(kl_beta=0.04))
torch.cuda.synchronize()
fn(buf)   # reset
# time the two backward kernels separately: run the whole call but read the counters after it (both kernels add up)
step(h, w, y, mask, rt, adv, old, ref, nl, otk.LossCfg(kl_beta=0.04))
torch.cuda.synchronize()
fn(buf)
pairs, ctas = 74, 148
res = dict(rows=n, d=d)
for kname, base in (("dh", 0), ("dW", 16)):
    m = [buf[base + k] / pairs for k in range(8)]
    t = [buf[base + 8 + k] / ctas for k in range(8)]
    res[kname] = dict(mma=dict(wait_B=m[0], wait_readyA=m[1], wait_tempty=m[2], total=m[3], stages=m[7]),
                      xform=dict(wait_A=t[4], transform=t[5], epilogue=t[6]))
print(json.dumps(res))
