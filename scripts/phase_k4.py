"""Experiment: per-phase clock64 split of the fused loss kernel (build with -DOTK_PHASE_TIMING, OTK_LIB=...)."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2601_07376_b200 as otk
from synth import make_batch, make_logits, make_noise
ctx = otk.Context(0)
tb = make_batch("math"); db = otk.traj_batch_to_device(tb)
m = otk.otk_build_masks(ctx, db)
adv = otk.otk_group_advantages(ctx, torch.from_numpy(tb.group_id).cuda(), 64, turn_offsets=torch.from_numpy(tb.turn_offsets).cuda(),
                               turn_rewards=torch.from_numpy(tb.turn_rewards).cuda())["adv"]
n, V = 65536, 151936
lg, tg = make_logits(n, V, dtype="bf16", seed=5, device="cuda", rows_per_chunk=4096)
lp = otk.otk_logprob_entropy_fwd(ctx, lg, tg)["logp"]
o, r = lp + make_noise(n, 0.05, 1, device="cuda"), lp + make_noise(n, 0.1, 2, device="cuda")
dl = torch.empty_like(lg)
for mode in ("data", "ones"):
    lm = m["loss_mask"][:n].clone()
    if mode == "ones": lm.fill_(1)
    fn = getattr(otk._lib, "otk_debug_phase")
    buf = (C.c_ulonglong * 8)()
    otk.otk_policy_loss_fwd_bwd(ctx, lg, tg, lm, m["row_traj"][:n], adv, o, r, m["n_loss"], otk.LossCfg(), dlogits=dl)
    torch.cuda.synchronize(); fn(buf)
    for _ in range(3):
        otk.otk_policy_loss_fwd_bwd(ctx, lg, tg, lm, m["row_traj"][:n], adv, o, r, m["n_loss"], otk.LossCfg(), dlogits=dl)
    torch.cuda.synchronize(); fn(buf)
    tot = buf[0] + buf[1] + buf[2]
    print(mode, "warps", buf[3], "pass1+wait %.3f  rowtotal+loss %.3f  pass2 %.3f" % (buf[0] / tot, buf[1] / tot, buf[2] / tot))
ctx.check()
