"""The README example (kept runnable: python scripts/readme_example.py on a GPU box)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2601_07376_b200 as otk
ctx = otk.Context(0)
# (1) + (2): masks and GRPO advantages from the FSM's segment lists (synth.make_batch shapes the paper's workloads)
from synth import make_batch, make_logits
tb = make_batch("tiny")
db = otk.traj_batch_to_device(tb)
m = otk.otk_build_masks(ctx, db)
a = otk.otk_group_advantages(ctx, torch.from_numpy(tb.group_id).cuda(), tb.num_groups,
                             turn_offsets=torch.from_numpy(tb.turn_offsets).cuda(),
                             turn_rewards=torch.from_numpy(tb.turn_rewards).cuda())
# (3) + (4): log-probs and the fused PPO-clip + KL loss with dlogits, over [N, V] logits
logits, targets = make_logits(tb.num_rows, 1024, dtype="bf16", seed=1, device="cuda")
old = otk.otk_logprob_entropy_fwd(ctx, logits, targets)["logp"]          # the fwd pool's old log-probs
out = otk.otk_policy_loss_fwd_bwd(ctx, logits, targets, m["loss_mask"], m["row_traj"], a["adv"], old,
                                  old, m["n_loss"], otk.LossCfg(kl_beta=0.04))
ctx.check()
print(otk.stats_dict(out["stats"]), out["dlogits"].shape)
