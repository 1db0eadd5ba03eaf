"""Vocab-sharded fused loss on one math micro-batch, P ranks emulated on ONE GPU (each rank: own ctx, column shard),
three ways (CUDA events around all ranks' work, 2 cycled input buffers):
  unsharded : otk_policy_loss_fwd_bwd on the whole GPU (the reference point)
  gathered  : per rank otk_row_partials -> (stack = the all-gather) -> otk_policy_loss_fwd_bwd_partials (per-rank
              streams; each launch may use every SM)
  vpf       : otk_policy_loss_fwd_bwd_vpf_group (K4-VPF, the exchange inside the kernel): all ranks in ONE
              cooperative launch, 148 // P CTAs per rank
Throughput = logit rows of the micro-batch / time; GB/s = the unsharded algorithmic bytes / time.
Usage: python scripts/perf_vpf.py [--rows 65536] [--iters 10] [--ranks 2 4]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2601_07376_b200 as otk
from synth import make_batch, make_logits, make_noise

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=65536)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--ranks", type=int, nargs="+", default=[2, 4])
a = ap.parse_args()
torch.cuda.set_device(0)
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6532.2
ctx = otk.Context(0)
tb = make_batch("math")
db = otk.traj_batch_to_device(tb)
m = otk.otk_build_masks(ctx, db)
adv = otk.otk_group_advantages(ctx, torch.from_numpy(tb.group_id).cuda(), 64,
                               turn_offsets=torch.from_numpy(tb.turn_offsets).cuda(),
                               turn_rewards=torch.from_numpy(tb.turn_rewards).cuda())["adv"]
n, V = a.rows, 151936
bufs = [make_logits(n, V, dtype="bf16", seed=5 + k, device="cuda", rows_per_chunk=4096) for k in range(2)]
olds = []
for lg, tg in bufs:
    lp = otk.otk_logprob_entropy_fwd(ctx, lg, tg)["logp"]
    olds.append((lp + make_noise(n, 0.05, 1, device="cuda"), lp + make_noise(n, 0.1, 2, device="cuda")))
dl = torch.empty_like(bufs[0][0])
lm, rt = m["loss_mask"][:n].clone(), m["row_traj"][:n].clone()
ntr = int(lm.sum())
alg = ntr * (4 * V + 25) + (n - ntr) * (2 * V + 1)
cfg = otk.LossCfg(kl_beta=0.04)
nl = m["n_loss"]


def timed(fn, streams):
    main = torch.cuda.current_stream()
    for k in range(3):
        fn(k)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(main)
    for k in range(a.iters):
        for s in streams:               # every rank starts after the previous iteration of all ranks
            s.wait_stream(main)
        fn(k)
        for s in streams:
            main.wait_stream(s)
    ev[1].record(main)
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / a.iters


def report(name, P, ms, **kw):
    print(json.dumps(dict(path=name, ranks=P, rows=n, ntr=ntr, ms=round(ms, 4), tokens_per_s=round(n / ms * 1e3),
                          GBps=round(alg / ms / 1e6, 1), frac=round(alg / ms / 1e6 / peak, 4), **kw)), flush=True)


def unsharded(k):
    lg, tg = bufs[k % 2]
    o, r = olds[k % 2]
    otk.otk_policy_loss_fwd_bwd(ctx, lg, tg, lm, rt, adv, o, r, nl, cfg, dlogits=dl, want_logp=False)


report("unsharded", 1, timed(unsharded, []))

for P in a.ranks:
    b = [V * k // P // 8 * 8 for k in range(P)] + [V]
    ctxs = [otk.Context(0) for _ in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    xs = otk.VpfExchange.local_group(ctxs, n)
    # the gathered path needs contiguous shards (its binding takes [N, vocab_local] tensors)
    shards = [[bufs[j][0][:, b[k]:b[k + 1]].contiguous() for k in range(P)] for j in range(2)]
    dls = [torch.empty_like(shards[0][k]) for k in range(P)]
    parts = torch.empty((P, n, 4), dtype=torch.float32, device="cuda")
    outs = [dict(logp=torch.empty(n, device="cuda"), entropy=torch.empty(n, device="cuda"),
                 stats=torch.zeros(5, dtype=torch.float64, device="cuda")) for _ in range(P)]

    def vpf(k):   # all P ranks in one cooperative launch (k_rows_vpf_group)
        lg, tg = bufs[k % 2]
        o, r = olds[k % 2]
        otk.otk_policy_loss_fwd_bwd_vpf_group(ctxs, [lg[:, b[q]:b[q + 1]] for q in range(P)], tg, lm, rt, adv, o, r,
                                              nl, cfg, b[:P], V, xs, dlogits=[dl[:, b[q]:b[q + 1]] for q in range(P)],
                                              outs=outs)

    def gathered(k):
        tg = bufs[k % 2][1]
        o, r = olds[k % 2]
        main = torch.cuda.current_stream()
        for q in range(P):
            otk.otk_row_partials(ctxs[q], shards[k % 2][q], tg, b[q], V, row_mask=lm, logit_scale=1.0,
                                 partials=parts[q], stream=streams[q])
        for s in streams:                # the all-gather: every rank needs every partial
            main.wait_stream(s)
        for s in streams:
            s.wait_stream(main)
        for q in range(P):
            otk.otk_policy_loss_fwd_bwd_partials(ctxs[q], shards[k % 2][q], tg, lm, rt, adv, o, r, nl, cfg, b[q], V,
                                                 parts, dlogits=dls[q], stream=streams[q], **outs[q])

    ms_v = timed(vpf, streams)
    for c in ctxs:
        c.check()
    report("vpf", P, ms_v, ctas_per_rank=148 // P, launch="one grouped launch")
    ms_g = timed(gathered, streams)
    for c in ctxs:
        c.check()
    report("gathered", P, ms_g, max_ctas_per_rank="all (148 each, ranks time-share the SMs)")
    for x in xs:
        x.close()
