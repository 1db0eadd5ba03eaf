"""One micro-batch of the math workload through otk_policy_loss_fwd_bwd, for ncu (not a bench)."""
import os, sys
sys.path.insert(0, os.getcwd())
import argparse
import numpy as np, torch
import paper_2601_07376_b200 as otk
from synth import make_batch, make_logits, make_noise
ap = argparse.ArgumentParser(); ap.add_argument("--rows", type=int, default=65536); ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--fwd", action="store_true"); ap.add_argument("--mask", default="data", choices=["data", "ones", "zeros"])
a = ap.parse_args()
torch.cuda.set_device(0)
ctx = otk.Context(0)
tb = make_batch("math")
db = otk.traj_batch_to_device(tb)
m = otk.otk_build_masks(ctx, db)
adv = otk.otk_group_advantages(ctx, torch.from_numpy(tb.group_id).cuda(), 64,
                               turn_offsets=torch.from_numpy(tb.turn_offsets).cuda(),
                               turn_rewards=torch.from_numpy(tb.turn_rewards).cuda())["adv"]
n = a.rows
lg, tg = make_logits(n, 151936, dtype="bf16", seed=5, device="cuda", rows_per_chunk=4096)
lp = otk.otk_logprob_entropy_fwd(ctx, lg, tg)["logp"]
old = lp + make_noise(n, 0.05, 1, device="cuda"); ref = lp + make_noise(n, 0.1, 2, device="cuda")
dl = torch.empty_like(lg)
lm = m["loss_mask"][:n].clone()
if a.mask == "ones": lm.fill_(1)
if a.mask == "zeros": lm.fill_(0)
for i in range(a.iters):
    if a.fwd:
        otk.otk_logprob_entropy_fwd(ctx, lg, tg)
    else:
        otk.otk_policy_loss_fwd_bwd(ctx, lg, tg, lm, m["row_traj"][:n], adv, old, ref, m["n_loss"],
                                    otk.LossCfg(), dlogits=dl, want_logp=False)
torch.cuda.synchronize(); ctx.check(); print("done")
