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
# large sampled batch: one CTA per row (k_sample_tm), bf16 and fp32, a ragged vocabulary
for V, dtype in ((151936, "bf16"), (4100, "bf16"), (1003, "f32")):
    lg, _ = make_logits(400, V, ld=-(-V // 8) * 8, dtype=dtype, seed=2, device="cuda")
    otk.otk_sample_tokens(ctx, lg, torch.rand(400, device="cuda"), vocab=V)
# K4-VPF: two ranks co-scheduled on the GPU
lg, tg = make_logits(N, 4096, dtype="bf16", seed=3, device="cuda")
ctxs = [otk.Context(0), otk.Context(0)]
xs = otk.VpfExchange.local_group(ctxs, N, max_ctas=8)
m = otk.otk_build_masks(ctx, db)
a = otk.otk_group_advantages(ctx, torch.from_numpy(tb.group_id).cuda(), tb.num_groups,
                             turn_offsets=torch.from_numpy(tb.turn_offsets).cuda(),
                             turn_rewards=torch.from_numpy(tb.turn_rewards).cuda())
o = torch.zeros(N, device="cuda")
ss = [torch.cuda.Stream(), torch.cuda.Stream()]
torch.cuda.synchronize()
for k in range(2):
    otk.otk_policy_loss_fwd_bwd_vpf(ctxs[k], lg[:, 2048 * k:2048 * (k + 1)], tg, m["loss_mask"], m["row_traj"], a["adv"],
                                    o, o, m["n_loss"], otk.LossCfg(), 2048 * k, 4096, xs[k], stream=ss[k])
torch.cuda.synchronize()
for c in ctxs:
    c.check()
for x in xs:
    x.close()
from synth import make_lmhead
h, w, y = make_lmhead(300, 1000, 128, seed=4, device="cuda")
otk.otk_lmhead_logprob_fwd(ctx, h, w, y)
# the policy loss through the LM head (NEXT-1 fwd + bwd: x tiles, loss rows, dh split-K + reduce, dW), ragged shapes
h, w, y = make_lmhead(300, 1032, 192, seed=5, device="cuda")
mk = (torch.arange(300, device="cuda") % 3 != 0).to(torch.uint8)
rtj = torch.arange(300, device="cuda", dtype=torch.int32) // 100
lp = otk.otk_lmhead_logprob_fwd(ctx, h, w, y)["logp"]
nl = mk.sum().to(torch.int64).reshape(1)
for cfg in (otk.LossCfg(), otk.LossCfg(ent_coef=0.02)):
    otk.otk_lmhead_policy_loss_fwd_bwd(ctx, h, w, y, mk, rtj, torch.tensor([0.5, -0.3, 1.0], device="cuda",
                                       dtype=torch.float64), lp.contiguous(), lp.contiguous(), nl, cfg)
# decode-batch sampler (one row per cluster, ranges resident in registers, warp partials pushed over DSMEM) and
# the ring kernel with rows split over CTA clusters (48: C = 6, 100: C = 2)
for n in (1, 5, 37, 48, 100):
    lg, _ = make_logits(n, 151936, dtype="bf16", seed=6, device="cuda")
    otk.otk_sample_tokens(ctx, lg, torch.rand(n, device="cuda"))
    otk.otk_sample_tokens(ctx, lg, greedy=True)
# K4-VPF, grouped launch, lag-3 pipeline + collector warp (P = 8: <= 4-chunk shard rows)
lg8, tg8 = make_logits(N, 8 * 1024, dtype="bf16", seed=7, device="cuda")
ctx8 = [otk.Context(0) for _ in range(8)]
xs8 = otk.VpfExchange.local_group(ctx8, N)
b8 = [1024 * k for k in range(8)]
otk.otk_policy_loss_fwd_bwd_vpf_group(ctx8, [lg8[:, 1024 * k:1024 * (k + 1)] for k in range(8)], tg8, m["loss_mask"],
                                      m["row_traj"], a["adv"], o, o, m["n_loss"], otk.LossCfg(), b8, 8192, xs8)
torch.cuda.synchronize()
for c in ctx8:
    c.check()
for x in xs8:
    x.close()
torch.cuda.synchronize()
ctx.check()
print("sanitize ok")
