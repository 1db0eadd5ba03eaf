"""Tiny invocation of every entry point, for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python scripts/sanitize.py"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2601_07376_b200 as otk
from paper_2601_07376_b200.step import MicroBatch, PolicyLossStep
from synth import make_batch, make_logits, make_noise
from synth.trajectories import random_small_batch
ctx = otk.Context(0)
tb = random_small_batch(np.random.default_rng(0), 6, max_segs=5, max_len=20)
db = otk.traj_batch_to_device(tb)
N = tb.num_rows
for V, dtype in ((151936, "bf16"), (1000, "f32")):
    lg, tg = make_logits(N, V, dtype=dtype, seed=1, device="cuda")
    f = otk.otk_logprob_entropy_fwd(ctx, lg, tg)
    old = (f["logp"] + make_noise(N, 0.05, 1, device="cuda")).contiguous()
    ref = (f["logp"] + make_noise(N, 0.1, 2, device="cuda")).contiguous()
    for credit in ("trajectory", "turn"):
        st = PolicyLossStep(ctx, db, torch.from_numpy(tb.group_id).cuda(), tb.num_groups,
                            torch.from_numpy(tb.turn_offsets).cuda(), torch.from_numpy(tb.turn_rewards).cuda(), V,
                            otk.LossCfg(ent_coef=0.01), credit=credit)
        dl = torch.empty_like(lg)
        st.run([MicroBatch(0, N, lg, tg, old, ref, dl)])
    part = otk.otk_row_partials(ctx, lg, tg, 0, V)
    u = torch.rand(N, device="cuda")
    otk.otk_sample_tokens(ctx, lg, u)
    otk.otk_sample_tokens(ctx, lg, greedy=True)
    otk.otk_sample_tokens(ctx, lg[:3].contiguous(), u[:3].contiguous())   # clustered rows
from synth import make_lmhead
h, w, y = make_lmhead(300, 1000, 128, seed=4, device="cuda")
otk.otk_lmhead_logprob_fwd(ctx, h, w, y)
torch.cuda.synchronize()
ctx.check()
print("sanitize ok")
