"""Time otk_policy_loss_fwd_bwd (and _fwd) alone on one math micro-batch: CUDA events, 2 cycled buffers.
Usage: OTK_LIB=path/to/libotk.so python scripts/perf_k4.py [--rows 65536] [--iters 10]"""
import os, sys, json, argparse
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2601_07376_b200 as otk
from synth import make_batch, make_logits, make_noise
ap = argparse.ArgumentParser(); ap.add_argument("--rows", type=int, default=65536); ap.add_argument("--iters", type=int, default=10); ap.add_argument("--mask", default="data", choices=["data", "ones", "zeros"])
ap.add_argument("--vocab", type=int, default=151936)
ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
ap.add_argument("--variant", default="", help="NEXT-4 loss variant: ent | dual | seqmean | seqsum | sft | turn")
a = ap.parse_args()
torch.cuda.set_device(0)
ctx = otk.Context(0)
tb = make_batch("math"); db = otk.traj_batch_to_device(tb)
m = otk.otk_build_masks(ctx, db)
adv = otk.otk_group_advantages(ctx, torch.from_numpy(tb.group_id).cuda(), 64, turn_offsets=torch.from_numpy(tb.turn_offsets).cuda(),
                               turn_rewards=torch.from_numpy(tb.turn_rewards).cuda())["adv"]
n, V = a.rows, a.vocab
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6532.2
bufs = [make_logits(n, V, dtype=a.dtype, seed=5 + k, device="cuda", rows_per_chunk=4096) for k in range(2)]
es = 2 if a.dtype == "bf16" else 4
olds = []
for lg, tg in bufs:
    lp = otk.otk_logprob_entropy_fwd(ctx, lg, tg)["logp"]
    olds.append((lp + make_noise(n, 0.05, 1, device="cuda"), lp + make_noise(n, 0.1, 2, device="cuda")))
dl = torch.empty_like(bufs[0][0])
lm, rt = m["loss_mask"][:n].clone(), m["row_traj"][:n]
if a.mask == "ones": lm.fill_(1)
if a.mask == "zeros": lm.fill_(0)
ntr = int(lm.sum())
alg = ntr * (2 * es * V + 21) + (n - ntr) * (es * V + 1)
kw = dict(ent=dict(ent_coef=0.01), dual=dict(dual_clip=3.0), seqmean=dict(reduction=1), seqsum=dict(reduction=2),
          sft=dict(sft=True)).get(a.variant, {})
cfg = otk.LossCfg(**kw, traj_loss_tokens=m["traj_loss_tokens"], n_active_traj=m["n_active_traj"])
adv_use = adv
if a.variant == "turn":   # turn-level credit: A read per row through the row's segment
    mt = otk.otk_build_masks(ctx, db, row_seg=True)
    tr = otk.otk_turn_returns(ctx, db, tb.num_segments, torch.from_numpy(tb.group_id).cuda(),
                              torch.from_numpy(tb.turn_offsets).cuda(), torch.from_numpy(tb.turn_rewards).cuda(), 0.9)
    adv_use = otk.otk_group_advantages(ctx, tr["seg_group"], 64, returns=tr["seg_return"], skip_ungrouped=True)["adv"]
    cfg = otk.LossCfg(adv_index=mt["row_seg"][:n].clone())
def run(k):
    lg, tg = bufs[k % 2]; o, r = olds[k % 2]
    otk.otk_policy_loss_fwd_bwd(ctx, lg, tg, lm, rt, adv_use, o, r, m["n_loss"], cfg, dlogits=dl, want_logp=False)
def runf(k):
    lg, tg = bufs[k % 2]
    otk.otk_logprob_entropy_fwd(ctx, lg, tg)
res = {}
for name, fn, by in (("bwd", run, alg), ("fwd", runf, n * (es * V + 12))):
    for k in range(3): fn(k)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for k in range(a.iters): fn(k)
    ev[1].record(); torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / a.iters
    res[name] = dict(ms=round(ms, 4), GBps=round(by / ms / 1e6, 1), frac=round(by / ms / 1e6 / peak, 4))
ctx.check()
print(json.dumps(dict(lib=os.environ.get("OTK_LIB", "default"), vocab=V, dtype=a.dtype, mask=a.mask, variant=a.variant or "default", ntr=ntr, **res)))
