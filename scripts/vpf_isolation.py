import os, sys, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2601_07376_b200 as otk
from synth import make_batch, make_logits, make_noise
torch.cuda.set_device(0)
ctx = otk.Context(0)
tb = make_batch("math"); db = otk.traj_batch_to_device(tb)
m = otk.otk_build_masks(ctx, db)
adv = otk.otk_group_advantages(ctx, torch.from_numpy(tb.group_id).cuda(), 64, turn_offsets=torch.from_numpy(tb.turn_offsets).cuda(), turn_rewards=torch.from_numpy(tb.turn_rewards).cuda())["adv"]
n, V = 65536, 151936
lg, tg = make_logits(n, V, dtype="bf16", seed=5, device="cuda", rows_per_chunk=4096)
lp = otk.otk_logprob_entropy_fwd(ctx, lg, tg)["logp"]
o, r = lp + make_noise(n, 0.05, 1, device="cuda"), lp + make_noise(n, 0.1, 2, device="cuda")
dl = torch.empty_like(lg)
lm, rt = m["loss_mask"][:n].clone(), m["row_traj"][:n].clone()
cfg = otk.LossCfg(kl_beta=0.04); nl = m["n_loss"]
for P in (2, 4, 8):
    b = [V * k // P // 8 * 8 for k in range(P)] + [V]
    ctxs = [otk.Context(0) for _ in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    for mode in ("exchange", "isolated"):
        xs = otk.VpfExchange.local_group(ctxs, n, max_ctas=148 // P) if mode == "exchange" else \
            [otk.VpfExchange.local_group([c], n, max_ctas=148 // P)[0] for c in ctxs]
        def fn():
            main = torch.cuda.current_stream()
            for s_ in streams: s_.wait_stream(main)
            for q in range(P):
                otk.otk_policy_loss_fwd_bwd_vpf(ctxs[q], lg[:, b[q]:b[q + 1]], tg, lm, rt, adv, o, r, nl, cfg, b[q], V, xs[q],
                                                dlogits=dl[:, b[q]:b[q + 1]], stream=streams[q])
            for s_ in streams: main.wait_stream(s_)
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(8): fn()
        e1.record(); torch.cuda.synchronize()
        print(json.dumps(dict(P=P, mode=mode, ms=round(e0.elapsed_time(e1) / 8, 4))), flush=True)
        for x in xs: x.close()
