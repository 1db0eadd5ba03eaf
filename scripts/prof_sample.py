"""One otk_sample_tokens launch on a decode batch (for ncu): python scripts/prof_sample.py [rows] [greedy]"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2601_07376_b200 as otk
from synth import make_logits
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
greedy = len(sys.argv) > 2 and sys.argv[2] == "greedy"
ctx = otk.Context(0)
lg, _ = make_logits(n, 151936, dtype="bf16", seed=7, device="cuda", rows_per_chunk=4096)
u = torch.rand(n, device="cuda")
for _ in range(3):
    otk.otk_sample_tokens(ctx, lg, u, greedy=greedy)
torch.cuda.synchronize()
ctx.check()
