"""Time the fused LM-head forward (otk_lmhead_logprob_fwd) against the unfused baseline (cuBLAS bf16 GEMM
materialising the logits + otk_logprob_entropy_fwd) on N x d -> V.
Usage: python scripts/perf_lmhead.py [--rows 8192] [--d 3584] [--vocab 151936] [--iters 5]"""
import os, sys, json, argparse
sys.path.insert(0, os.getcwd())
import torch
import paper_2601_07376_b200 as otk
from synth import make_lmhead
ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=8192); ap.add_argument("--d", type=int, default=3584)
ap.add_argument("--vocab", type=int, default=151936); ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--no-baseline", action="store_true")
a = ap.parse_args()
torch.cuda.set_device(0)
ctx = otk.Context(0)
h, w, y = make_lmhead(a.rows, a.vocab, a.d, seed=1, device="cuda")
flops = 2.0 * a.rows * a.vocab * a.d
ws = None
def fused():
    global ws
    o = otk.otk_lmhead_logprob_fwd(ctx, h, w, y, workspace=ws)
    ws = o["workspace"]
def unfused():
    z = h @ w.T
    otk.otk_logprob_entropy_fwd(ctx, z, y)
def timeit(fn):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(a.iters): fn()
    ev[1].record(); torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / a.iters
res = dict(rows=a.rows, d=a.d, vocab=a.vocab)
ms = timeit(fused)
res["fused"] = dict(ms=round(ms, 3), tflops=round(flops / ms / 1e9, 1), frac=round(flops / ms / 1e9 / 1657.7, 4),
                    tokens_per_s=round(a.rows / ms * 1e3))
if not a.no_baseline:
    ms2 = timeit(unfused)
    res["unfused_cublas_plus_k3"] = dict(ms=round(ms2, 3), tflops=round(flops / ms2 / 1e9, 1))
    res["speedup"] = round(ms2 / ms, 3)
ctx.check()
print(json.dumps(res))
