"""Experiment: globaltimer stamps of CTA 0 of the decode sampler (build with -DOTK_SDEC_TIMING, OTK_LIB=that .so)."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2601_07376_b200 as otk
from synth import make_logits
ctx = otk.Context(0)
for n in (1, 16, 64):
    lg, _ = make_logits(n, 151936, dtype="bf16", seed=3, device="cuda")
    u = torch.rand(n, device="cuda")
    buf = (ctypes.c_ulonglong * 8)()
    for it in range(4):
        otk.otk_sample_tokens(ctx, lg, u)
        torch.cuda.synchronize()
        otk._lib.otk_debug_sdec(buf)
        t = [buf[i] - buf[0] for i in range(6)]
        print(n, it, t)
