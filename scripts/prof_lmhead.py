"""One fused LM-head forward launch for ncu: python scripts/prof_lmhead.py [rows] [d]"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2601_07376_b200 as otk
from synth import make_lmhead
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d = int(sys.argv[2]) if len(sys.argv) > 2 else 3584
ctx = otk.Context(0)
h, w, y = make_lmhead(n, 151936, d, seed=1, device="cuda")
ws = None
for _ in range(3):
    ws = otk.otk_lmhead_logprob_fwd(ctx, h, w, y, workspace=ws)["workspace"]
torch.cuda.synchronize()
ctx.check()
