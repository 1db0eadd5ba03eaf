"""Decode-batch sampler launches for ncu (k_sample_dec): python scripts/prof_sample_dec.py rows"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2601_07376_b200 as otk
from synth import make_logits
n = int(sys.argv[1])
ctx = otk.Context(0)
lg, _ = make_logits(n, 151936, dtype="bf16", seed=3, device="cuda")
u = torch.rand(n, device="cuda")
for _ in range(3):
    otk.otk_sample_tokens(ctx, lg, u)
    otk.otk_sample_tokens(ctx, lg, greedy=True)
torch.cuda.synchronize()
