#!/usr/bin/env python
"""bench.py — one training step of the otk hot path (north_star (1)-(4)) on synthetic trajectories.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl otk|reference] [--config math]

A step = otk_build_masks + otk_group_advantages + otk_policy_loss_fwd_bwd over every micro-batch of
the batch (A3 runs fused inside A4), on BASELINE.json configs[1] ("math": 512 trajectories x T=2048,
V=151936 bf16 logits, N = 2^20 rows). Under torchrun (N > 1) the default layout is STRONG scaling of that one
global batch: dist.plan_batch_shards splits it into contiguous trajectory ranges balanced by HBM bytes (groups
straddle ranks: game / marl group ids are strided), and the step adds the batch-sharding exchanges (all-reduce
of the token count, all-gather of group returns so every rank computes the global group statistics, all-reduce
of the loss statistics). --layout weak gives every rank its own batch of the config instead. `--config game
--gpus 8` is BASELINE configs[2] (128 game trajectories batch-sharded over 8 GPUs).
Prints ONE JSON line on rank 0 (schema: the driver's bench contract).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "logit-tokens/s for fused logprob+GRPO loss fwd+bwd (V=151936), % HBM peak, 1/2/4/8 GPU"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="otk", choices=["otk", "reference"])
    ap.add_argument("--config", default="math")
    ap.add_argument("--micro-rows", type=int, default=65536)
    ap.add_argument("--logit-buffers", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--e2e-chunk", type=int, default=4096, help="rows per host-entry-point chunk (copy / compute overlap)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-parity", action="store_true", help="skip the parity block (SURVEY.md §8(d)(v))")
    ap.add_argument("--no-next", action="store_true",
                    help="skip the side measurements of the forward (3) and the SURVEY.md §8(f) rows")
    ap.add_argument("--vocab-ways", type=int, default=2,
                    help="--shard 2d / 2d-fused: vocab shards per row block (world = batch shards x vocab-ways)")
    ap.add_argument("--layout", default="strong", choices=["strong", "weak"],
                    help="batch sharding (N > 1): strong = ONE global batch of the config split into contiguous "
                         "trajectory ranges by dist.plan_batch_shards (groups straddle ranks; total work fixed); "
                         "weak = every rank its own batch of the config (rank-local groups)")
    ap.add_argument("--collectives", default="torch", choices=["torch", "otk"],
                    help="batch sharding's exchanges: torch.distributed (default) or the library's own NCCL "
                         "communicator (otk_comm_init + otk_batch_*, the C-ABI path)")
    ap.add_argument("--shard", default="batch", choices=["batch", "vocab", "vocab-fused", "2d", "2d-fused"],
                    help="batch: each rank owns whole trajectories (weak scaling); vocab: each rank owns V/N "
                         "columns of every row (strong scaling, row partials all-gathered); vocab-fused: the "
                         "same split with the exchange inside the loss kernel (K4-VPF, CUDA IPC peer buffers); "
                         "2d / 2d-fused: world / vocab-ways trajectory shards x vocab-ways column shards")
    return ap.parse_args()


# ------------------------------------------------------------------------------------------------
def shard_layout(args, world, rank):
    """(Pv vocab shards per row block, nb batch shards, b, v, batch group, vocab group) of this rank."""
    import torch.distributed as dist
    if args.shard in ("2d", "2d-fused"):
        if world == 1:
            return dict(Pv=1, nb=1, b=0, v=0, bg=None, vg=None)
        from paper_2601_07376_b200.dist import make_2d_groups
        b, v, bg, vg = make_2d_groups(args.vocab_ways)
        return dict(Pv=args.vocab_ways, nb=world // args.vocab_ways, b=b, v=v, bg=bg, vg=vg)
    if args.shard in ("vocab", "vocab-fused"):
        return dict(Pv=world, nb=1, b=0, v=rank, bg=None, vg=dist.group.WORLD if world > 1 else None)
    return dict(Pv=1, nb=world, b=rank, v=0, bg=dist.group.WORLD if world > 1 else None, vg=None)


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        backend = os.environ.get("OTK_DIST_BACKEND", "nccl")   # gloo: multi-rank functional runs on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        pg = dist.group.WORLD
    else:
        torch.cuda.set_device(0)
    return world, rank, local, pg


class ClockSampler:
    """Samples SM clock and clock-event reasons with NVML during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clocks"}

    def __init__(self, index):
        self.samples, self.reasons, self.stop = [], set(), threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml-unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------------------------------------
def build_workload(args, rank, world, device):
    """Synthetic inputs (untimed): this rank's trajectories, cycled logits buffers, per-row old/ref.
    batch sharding: rank-specific trajectories (seed + 1000 * rank), full-vocabulary logits.
    vocab sharding: the same trajectories and targets on every rank, logits columns [v0, v1) of this rank."""
    import paper_2601_07376_b200 as otk
    from paper_2601_07376_b200.dist import vocab_shard_bounds
    from paper_2601_07376_b200.step import MicroBatch, VocabShard
    from synth import CONFIGS, make_batch, make_logits, make_noise
    cfgw = CONFIGS[args.config]
    L = shard_layout(args, world, rank)
    vocab_mode = args.shard != "batch"
    brank = L["b"]
    strong = args.layout == "strong" and not vocab_mode
    tb_full, plan, b0 = None, None, 0
    if strong:   # one global batch, contiguous trajectory ranges balanced by HBM cost
        from paper_2601_07376_b200.dist import plan_batch_shards, traj_costs
        from synth import slice_batch
        tb_full = make_batch(args.config)
        plan = plan_batch_shards(traj_costs(tb_full, cfgw.V), world) if world > 1 else [(0, tb_full.num_traj)]
        b0, b1 = plan[rank]
        tb = slice_batch(tb_full, b0, b1)
    else:
        tb = make_batch(args.config, seed=cfgw.seed + 1000 * brank)
        tb.group_id = tb.group_id + np.int32(brank * cfgw.num_groups)   # this rank's groups (global ids)
    N, V = tb.num_rows, cfgw.V
    v0, v1 = vocab_shard_bounds(V, L["Pv"])[L["v"]]
    Vl = v1 - v0
    M = min(args.micro_rows, N)
    ctx = otk.Context(torch.cuda.current_device())
    dbatch = otk.traj_batch_to_device(tb, device)
    gid = torch.from_numpy(tb.group_id).to(device)
    toff = torch.from_numpy(tb.turn_offsets).to(device)
    trew = torch.from_numpy(tb.turn_rewards).to(device)
    nbuf = max(1, min(args.logit_buffers, (N + M - 1) // M))
    bufs, tgts = [], []
    for k in range(nbuf):
        lg, tg = make_logits(M, Vl, dtype=cfgw.dtype, seed=cfgw.seed * 100 + 10 * rank + k, device=device,
                             rows_per_chunk=4096)
        if vocab_mode:   # global targets, identical on every rank of the row block's vocab group
            g = torch.Generator(device=device)
            g.manual_seed(cfgw.seed * 100 + k + 7919 * brank)
            tg = torch.randint(0, V, (M,), generator=g, device=device, dtype=torch.int32)
        bufs.append(lg)
        tgts.append(tg)
    dlogits = torch.empty_like(bufs[0])
    vshard = VocabShard(ctx, v0, Vl, V, L["vg"]) if vocab_mode else None
    if args.shard.endswith("-fused"):   # K4-VPF: exchange buffers mapped once (setup, untimed)
        from paper_2601_07376_b200.step import VocabShardFused
        if L["vg"] is not None:
            from paper_2601_07376_b200.dist import open_vpf_exchange
            xchg = open_vpf_exchange(ctx, M, vshard.pg)
        else:
            xchg = otk.VpfExchange.local_group([ctx], M)[0]
        vshard = VocabShardFused(ctx, v0, Vl, V, xchg, vshard.pg)
    # old/ref = the fwd pool's log-probs (otk_logprob_entropy_fwd, or its vocab-sharded form) + synth noise
    if vocab_mode:
        base_logp = [vshard.forward(b, t)["logp"] for b, t in zip(bufs, tgts)]
    else:
        base_logp = [otk.otk_logprob_entropy_fwd(ctx, b, t)["logp"] for b, t in zip(bufs, tgts)]
    mbs = []
    for i, r0 in enumerate(range(0, N, M)):
        r1 = min(N, r0 + M)
        n = r1 - r0
        k = i % nbuf
        old = base_logp[k][:n] + make_noise(n, 0.05, 7000 + i, device=device)
        ref = base_logp[k][:n] + make_noise(n, 0.1, 9000 + i, device=device) if cfgw.kl_beta else None
        mbs.append(MicroBatch(r0, r1, bufs[k][:n], tgts[k][:n], old.contiguous(),
                              None if ref is None else ref.contiguous(), dlogits[:n]))
    ctx.check()
    return dict(otk=otk, cfgw=cfgw, tb=tb, ctx=ctx, dbatch=dbatch, gid=gid, toff=toff, trew=trew, bufs=bufs,
                tgts=tgts, mbs=mbs, N=N, V=V, Vl=Vl, v0=v0, M=M, dlogits=dlogits, vshard=vshard, L=L,
                strong=strong, tb_full=tb_full, plan=plan, b0=b0)


def algorithmic_bytes(V, n_train, n_masked, beta):
    """a trainable row reads + writes the V-wide bf16 row plus its side data
    (target 4, mask 1, row_traj 4, old 4, ref 4 if beta > 0); a masked row is only zero-filled (+ mask 1)."""
    side = 4 + 1 + 4 + 4 + (4 if beta else 0)
    return n_train * (4 * V + side) + n_masked * (2 * V + 1)


def run_otk(args):
    world, rank, local, pg = dist_setup(args)
    device = torch.device("cuda", torch.cuda.current_device())
    W = build_workload(args, rank, world, device)
    otk, ctx = W["otk"], W["ctx"]
    from paper_2601_07376_b200.step import PolicyLossStep
    cfgw = W["cfgw"]
    cfg = otk.LossCfg(kl_beta=cfgw.kl_beta)
    vocab_mode = args.shard != "batch"
    L = W["L"]
    bpg, nb, Pv = L["bg"], L["nb"], L["Pv"]
    if W["strong"]:
        counts = [e - s_ for s_, e in W["plan"]]
        g_groups = cfgw.num_groups
    else:
        counts = [W["tb"].num_traj] * nb
        g_groups = cfgw.num_groups * nb
    coll = "torch"
    if args.collectives == "otk" and bpg is not None and not vocab_mode:
        import torch.distributed as dist
        uid = [otk.otk_comm_unique_id() if dist.get_rank(bpg) == 0 else None]
        dist.broadcast_object_list(uid, src=dist.get_global_rank(bpg, 0), group=bpg)
        otk.otk_comm_init(ctx, uid[0], dist.get_world_size(bpg), dist.get_rank(bpg))
        coll = "otk"
    step = PolicyLossStep(ctx, W["dbatch"], W["gid"], cfgw.num_groups, W["toff"], W["trew"], W["Vl"], cfg,
                          process_group=bpg, global_num_traj=counts if bpg else None,
                          global_num_groups=g_groups if bpg else None, vocab_shard=W["vshard"], collectives=coll)
    stream = torch.cuda.current_stream()
    nmb = len(W["mbs"])
    # CUDA events around every loss launch of every timed step, on the launching stream
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nmb)]
          for _ in range(args.steps)]
    cur = {"s": 0}

    def on_launch(k, what):
        ev[cur["s"]][k][0 if what == "begin" else 1].record(stream)

    def barrier():
        if pg is not None:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step.run(W["mbs"])
    ctx.check()
    barrier()
    launches0 = ctx.launches
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for s in range(args.steps):
            cur["s"] = s
            step.run(W["mbs"], on_launch=on_launch)
        t1.record(stream)
        torch.cuda.synchronize()
    k4_ms_all = [[a.elapsed_time(b) for a, b in row] for row in ev]
    k4_ms = [sum(r[k] for r in k4_ms_all) / args.steps for k in range(nmb)]
    barrier()
    launches = ctx.launches - launches0
    elapsed = t0.elapsed_time(t1)
    if pg is not None:
        import torch.distributed as dist
        t = torch.tensor([elapsed], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    ms_per_step = elapsed / args.steps
    stats = otk.stats_dict(step.stats)
    ctx.check()

    # masks / token counts for the roofline bytes (from the device outputs; one D2H after timing)
    lm = step.masks["loss_mask"]
    n_train = [int(lm[mb.r0:mb.r1].sum()) for mb in W["mbs"]]
    n_rows = [mb.r1 - mb.r0 for mb in W["mbs"]]
    if args.shard.endswith("-fused"):   # one read + one write of the shard, 32 B per peer per trainable row
        Vl = W["Vl"]
        side = 4 + 1 + 4 + 4 + (4 if cfgw.kl_beta else 0) + 32 * (Pv - 1)
        bytes_k4 = [t * (4 * Vl + side) + (r - t) * (2 * Vl + 1) for t, r in zip(n_train, n_rows)]
        kname = "k_rows_tm<bf16,BWD_VPF> (otk_policy_loss_fwd_bwd_vpf, exchange in-kernel)"
    elif vocab_mode:   # row partials (read 2V_l) + all-gather + streaming pass 2 (read 2V_l, write 2V_l)
        Vl = W["Vl"]
        side = 4 + 1 + 4 + 4 + (4 if cfgw.kl_beta else 0) + 16 * Pv
        bytes_k4 = [t * (6 * Vl + side) + (r - t) * (2 * Vl + 1) for t, r in zip(n_train, n_rows)]
        kname = "k_rows_tm<bf16,PARTIAL> + all_gather + k_rows_stream<bf16> (vocab-sharded loss)"
    else:
        bytes_k4 = [algorithmic_bytes(W["V"], t, r - t, cfgw.kl_beta) for t, r in zip(n_train, n_rows)]
        kname = "k_rows_tm<bf16,BWD> (otk_policy_loss_fwd_bwd)"
    avg_bytes = sum(bytes_k4) / nmb
    avg_ms = sum(k4_ms) / nmb
    achieved = avg_bytes / (avg_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    total_rows = W["tb_full"].num_rows if W["strong"] else W["N"] * nb
    value = total_rows / (ms_per_step * 1e-3)
    step_bytes = sum(bytes_k4)
    per_rank = {"rows": [W["N"]], "GB": [step_bytes / 1e9], "trainable": [sum(n_train)], "ms_k4": [sum(k4_ms)]}
    if pg is not None:   # this step's per-rank work (load balance of the shard plan)
        import torch.distributed as dist
        t = torch.tensor([W["N"], step_bytes / 1e9, sum(n_train), sum(k4_ms)], dtype=torch.float64, device=device)
        allt = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        per_rank = {k: [float(a[i]) for a in allt] for i, k in enumerate(("rows", "GB", "trainable", "ms_k4"))}
    imbalance = max(per_rank["GB"]) / (sum(per_rank["GB"]) / len(per_rank["GB"]))
    if world == 1:
        par = "single GPU" + (f" ({args.shard} path, 1 shard)" if vocab_mode else "")
    elif W["strong"]:
        par = f"batch-shard dp{world}: one global batch, contiguous trajectory ranges (dist.plan_batch_shards)"
    else:
        fused = " (K4-VPF)" if args.shard.endswith("-fused") else ""
        par = (f"batch-shard dp{nb} x vocab-shard tp{Pv}{fused}" if args.shard.startswith("2d")
               else f"vocab-shard tp{world}{fused}" if vocab_mode else f"batch-shard dp{world}")
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if (W["strong"] or (nb == 1 and Pv > 1) or args.shard in ("vocab", "vocab-fused"))
                   else "weak",
        "vs_baseline": None, "dtype": cfgw.dtype, "data": "synthetic (seeded; SURVEY.md §8(d) recipe)",
        "config": {"workload": f"{args.config}: {cfgw.note}",
                   "global_batch_traj": W["tb_full"].num_traj if W["strong"] else W["tb"].num_traj * nb,
                   "layout": ("strong: one global batch split by dist.plan_batch_shards (HBM-cost balanced "
                              "contiguous trajectory ranges; groups span ranks)") if W["strong"] else
                             ("weak: every rank its own batch" if not vocab_mode else args.shard),
                   "rows_per_gpu": W["N"], "vocab": W["V"], "vocab_per_gpu": W["Vl"], "micro_batch_rows": W["M"],
                   "micro_batches": nmb, "parallelism": par,
                   "collectives": {"torch": "torch.distributed (NCCL)", "otk": "otk_comm_* / otk_batch_* (NCCL)"}[coll]
                   if world > 1 else None,
                   "l2": f"inputs >> L2: {len(W['bufs'])} logits buffers of "
                         f"{W['bufs'][0].numel() * W['bufs'][0].element_size() / 1e9:.1f} GB cycled",
                   "kl_beta": cfgw.kl_beta, "clip": [0.2, 0.2], "kl": "k3"},
        "trainable_rows_per_s": sum(n_train) * nb / (ms_per_step * 1e-3),
        "step_algorithmic_GBps": step_bytes / (ms_per_step * 1e-3) / 1e9,
        "roofline": {"bound": "hbm", "kernel": kname,
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "peak_source": peak_src,
                     "bytes_per_launch": avg_bytes, "avg_launch_ms": avg_ms,
                     "share_of_step": sum(k4_ms) / ms_per_step},
        "per_rank": per_rank, "imbalance_bytes_max_over_mean": imbalance,
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / args.steps,
        "loss": stats["loss"], "n_loss": stats["n_tokens"],
    }
    res["clocks"] = clk.summary()
    traffic = os.path.join(ROOT, "profiles", "k4_traffic.json")
    if os.path.exists(traffic) and not vocab_mode:
        try:
            tj = json.load(open(traffic))
            res["roofline"]["traffic"] = tj.get("traffic_bytes_per_launch")
            res["roofline"]["traffic_source"] = tj.get("source")
        except Exception:
            pass
    if not args.no_e2e and not vocab_mode:
        res["e2e"] = e2e(args, W, world, step, cfg)
    if rank == 0 and not args.no_cpu_baseline and not vocab_mode:
        res["cpu_baseline"], inp = cpu_baseline(args, W, cfg)
        if not args.no_parity:
            res["parity"] = parity_block(W, step, cfg, inp)
    if rank == 0 and world == 1 and not args.no_next and not vocab_mode:
        try:
            res["other_kernels"] = other_kernels(W, step, cfg)
        except Exception as e:  # side measurements never invalidate the headline line
            res["other_kernels"] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0:
        print(json.dumps(res), flush=True)
    if pg is not None:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------------------------------------
def other_kernels(W, step, cfg):
    """Side measurements (untimed for the headline, rank 0, N = 1): the forward (3) on one micro-batch, the
    rollout sampler (NEXT-3) on 4096- and 16-row decode batches, K4-VPF with P = 2, 4, 8 ranks emulated on this GPU,
    the fused LM-head forward (NEXT-1) at d = 3584 and the policy loss through the LM head (NEXT-1 fwd + bwd) at
    d = 1024 / 3584 against cuBLAS + (4) — CUDA events on the launching stream, inputs HBM-resident."""
    otk, ctx, V = W["otk"], W["ctx"], W["V"]
    hbm, _ = peaks()
    mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    bf16_peak = float(mp.get("bf16_tflops", 2250.0))               # burst (cuBLAS 8192^3, best of 10)
    bf16_sust = float(mp.get("bf16_tflops_sustained", bf16_peak))  # the same back to back for 4 s (power cap)
    bufs, tgts = W["bufs"], W["tgts"]

    def timed(fn, iters):
        for i in range(2):
            fn(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(iters):
            fn(i)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    out = {}
    M = bufs[0].shape[0]
    ms = timed(lambda i: otk.otk_logprob_entropy_fwd(ctx, bufs[i % len(bufs)], tgts[i % len(tgts)]), 4)
    gbs = M * (2 * V + 12) / ms / 1e6
    out["logprob_entropy_fwd"] = {"rows": M, "ms": ms, "GBps": gbs, "frac_hbm": gbs / hbm,
                                  "kernel": "k_rows_tm<bf16,FWD> (north_star (3))"}
    n = 4096
    u = torch.rand(n, device=bufs[0].device)
    for mode in ("sample", "greedy"):
        # row windows 4096 apart across the cycled buffers: no L2 reuse between iterations
        ms = timed(lambda i: otk.otk_sample_tokens(
            ctx, bufs[i % len(bufs)][(i * n) % (M - n):(i * n) % (M - n) + n], u, greedy=mode == "greedy"), 8)
        gbs = n * (2 * V + 12) / ms / 1e6
        out[f"sample_tokens_{mode}"] = {"rows": n, "us": ms * 1e3, "GBps": gbs, "frac_hbm": gbs / hbm,
                                        "kernel": ("k_sample" if mode == "greedy" else "k_sample_tm")
                                        + " (SURVEY.md §8(f) NEXT-3)"}
    # K4-VPF (vocab-sharded loss, exchange in-kernel): P = 2 ranks emulated on this GPU in ONE cooperative launch
    # (own ctx, column shard, 74 CTAs each) on micro-batch 0, against the unsharded loss on the same rows (measured
    # before the tensor-core benchmark below, whose power draw would slow whichever runs after it)
    mb = W["mbs"][0]
    lm, rt = step.masks["loss_mask"][mb.r0:mb.r1], step.masks["row_traj"][mb.r0:mb.r1]
    adv, nl = step.adv_out["adv"], step.masks["n_loss"]
    ms_u = timed(lambda i: otk.otk_policy_loss_fwd_bwd(ctx, mb.logits, mb.targets, lm, rt, adv, mb.old_logp,
                                                       mb.ref_logp, nl, cfg, dlogits=mb.dlogits, want_logp=False), 4)
    for P in (2, 4, 8):
        b = [V * k // P // 8 * 8 for k in range(P)] + [V]
        ctxs = [otk.Context(ctx.device) for _ in range(P)]
        xs = otk.VpfExchange.local_group(ctxs, M)

        def vpf(i):
            otk.otk_policy_loss_fwd_bwd_vpf_group(ctxs, [mb.logits[:, b[q]:b[q + 1]] for q in range(P)], mb.targets,
                                                  lm, rt, adv, mb.old_logp, mb.ref_logp, nl, cfg, b[:P], V, xs,
                                                  dlogits=[mb.dlogits[:, b[q]:b[q + 1]] for q in range(P)])
        ms_v = timed(vpf, 4)
        for c in ctxs:
            c.check()
        for x in xs:
            x.close()
        out[f"vocab_shard_vpf_p{P}_one_gpu"] = {
            "rows": M, "ms": ms_v, "ms_unsharded": ms_u, "vs_unsharded": ms_u / ms_v,
            "kernel": f"k_rows_vpf_group<bf16>: {P} ranks in one launch, {148 // P} CTAs each (DESIGN.md §7)"}
    # decode-sized sampling (k_sample_dec): 16 rows, windows cycled over the buffers (no L2 reuse); the 16 launches
    # replayed from a CUDA graph, so the time is the device's (the Python binding costs more than the kernel)
    n16 = 16
    u16 = torch.rand(n16, device=bufs[0].device)
    sl = [bufs[i % len(bufs)][(i * 4096) % (M - n16):(i * 4096) % (M - n16) + n16] for i in range(16)]
    o16 = dict(tokens=torch.empty(n16, dtype=torch.int32, device=u16.device),
               logp=torch.empty(n16, dtype=torch.float32, device=u16.device))
    for x in sl[:2]:
        otk.otk_sample_tokens(ctx, x, u16, out=o16)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    gs = torch.cuda.Stream()
    gs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(gs):
        with torch.cuda.graph(g, stream=gs):
            for x in sl:
                otk.otk_sample_tokens(ctx, x, u16, out=o16)
    torch.cuda.synchronize()
    g.replay()
    ms = timed(lambda i: g.replay(), 2) / len(sl)
    out["sample_tokens_decode16"] = {"rows": n16, "us": ms * 1e3, "GBps": n16 * (2 * V + 12) / ms / 1e6,
                                     "kernel": "k_sample_dec (one row per 8-CTA cluster; CUDA-graph replay)"}
    del g
    from synth import make_lmhead
    rows, d = 8192, 3584
    h, w, y = make_lmhead(rows, V, d, seed=1, device=bufs[0].device)
    ws = [None]

    def lm(i):
        o = otk.otk_lmhead_logprob_fwd(ctx, h, w, y, workspace=ws[0])
        ws[0] = o["workspace"]
    ms = timed(lm, 3)
    tf = 2.0 * rows * V * d / ms / 1e9
    out["lmhead_logprob_fwd"] = {"rows": rows, "hidden_dim": d, "ms": ms, "TFLOPs": tf, "frac_bf16": tf / bf16_peak,
                                 "kernel": "k_lmhead_fwd (tcgen05 cta_group::2; SURVEY.md §8(f) NEXT-1 fwd)"}
    del h, w, y, ws
    # NEXT-1 fwd + bwd: the policy loss and dh / dW through the LM head, on this library's tcgen05 kernels
    # (otk_lmhead_policy_loss_fwd_bwd) vs cuBLAS GEMMs around the loss kernel (4); same inputs, back to back
    from paper_2601_07376_b200.step import LMHeadPolicyLoss, LMHeadPolicyLossFused
    from synth import make_noise
    for d in (1024, 3584):
        h, w, y = make_lmhead(rows, V, d, seed=2, device=bufs[0].device)
        msk = (torch.arange(rows, device=h.device) % 2).to(torch.uint8)
        rtj = (torch.arange(rows, device=h.device, dtype=torch.int32) // 512)
        advl = torch.linspace(-1, 1, rows // 512 + 1, device=h.device, dtype=torch.float64)
        lp = otk.otk_lmhead_logprob_fwd(ctx, h, w, y)["logp"]
        old = (lp + make_noise(rows, 0.05, 1, device=h.device)).contiguous()
        ref = (lp + make_noise(rows, 0.1, 2, device=h.device)).contiguous()
        nlr = msk.sum().to(torch.int64).reshape(1)
        res = {}
        for name, cls in (("cublas_gemms_plus_k4", LMHeadPolicyLoss), ("fused_tcgen05", LMHeadPolicyLossFused)):
            st = cls(ctx)
            res[name] = timed(lambda i: st(h, w, y, msk, rtj, advl, old, ref, nlr, cfg), 3)
            del st
        tf = 3 * 2.0 * rows * V * d / res["fused_tcgen05"] / 1e9
        out[f"lmhead_policy_loss_d{d}"] = {
            "rows": rows, "hidden_dim": d, "ms": res, "speedup_fused": res["cublas_gemms_plus_k4"] / res["fused_tcgen05"],
            "fused_TFLOPs": tf, "fused_frac_bf16": tf / bf16_peak, "fused_frac_bf16_sustained": tf / bf16_sust,
            "cublas_TFLOPs": 3 * 2.0 * rows * V * d / res["cublas_gemms_plus_k4"] / 1e9,
            "kernel": "k_lmhead_fwd (x tiles) + k_lmhead_loss_rows + k_lmhead_bwd<dh, dW> (SURVEY.md §8(f) NEXT-1)"}
        del h, w, y
    ctx.check()
    return out


def e2e(args, W, world, step, cfg):
    """Same metric through the C-ABI host-buffer entry point (otk_policy_loss_fwd_bwd_host): every
    micro-batch's trainable logits rows + side arrays are copied H2D from pinned host memory inside the timed
    region (pipelined in 4096-row chunks on a copy stream), and the step's result comes back D2H: the gradient
    rows of every trainable token (cudaMemcpy2DAsync of [0, V) per run of trainable rows, on the execution
    stream, overlapping the next chunk's H2D) plus the loss statistics. Masked rows' gradient is zero by
    definition (loss_mask is on the host), so with zero_masked_rows = 0 it neither crosses PCIe nor is
    zero-filled on the device. The step's masks / advantages (device outputs of (1)-(2)) are inputs of this
    call and are staged once."""
    import dataclasses
    otk, ctx = W["otk"], W["ctx"]
    mbs = W["mbs"]
    N = W["N"]
    # pinned host buffers allocated directly (no pageable staging copy); with several ranks on one node, one host
    # logits buffer per rank (each rank's pinned footprint: 2 micro-batches = 40 GB at the math config)
    nbh = len(W["bufs"]) if world == 1 else 1
    host_bufs = []
    for b in W["bufs"][:nbh]:
        hb = torch.empty(b.shape, dtype=b.dtype, pin_memory=True)
        hb.copy_(b)
        host_bufs.append(hb)
    dl_host = torch.empty(W["bufs"][0].shape, dtype=W["bufs"][0].dtype, pin_memory=True)   # one micro-batch
    adv = step.masks_and_advantages()
    torch.cuda.synchronize()
    n_loss = int(step.masks["n_loss"].item())
    lm_h = step.masks["loss_mask"].cpu().pin_memory()
    rt_h = step.masks["row_traj"].cpu().pin_memory()
    adv_h = adv.cpu().pin_memory()
    side = [(mb.targets.cpu().pin_memory(), mb.old_logp.cpu().pin_memory(),
             None if mb.ref_logp is None else mb.ref_logp.cpu().pin_memory()) for mb in mbs]
    nb = len(host_bufs)
    hcfg = dataclasses.replace(cfg, zero_masked_rows=False)

    def one_step():
        tot = 0.0
        for i, mb in enumerate(mbs):
            tg, old, ref = side[i]
            n = mb.r1 - mb.r0
            s = otk.otk_policy_loss_fwd_bwd_host(ctx, host_bufs[i % nb][:n], tg, lm_h[mb.r0:mb.r1],
                                                 rt_h[mb.r0:mb.r1], adv_h, old, ref, n_loss, hcfg,
                                                 dlogits=dl_host[:n], rows_per_chunk=args.e2e_chunk)
            tot += s["loss"]
        return tot

    one_step()  # warm-up (allocates the staging buffers once)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        one_step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / args.e2e_steps
    # the returned gradient of the last micro-batch equals the device path's on a sampled trainable row
    mb = mbs[-1]
    n = mb.r1 - mb.r0
    tr = torch.nonzero(lm_h[mb.r0:mb.r1]).flatten()
    match = None
    if tr.numel():
        j = int(tr[tr.numel() // 2])
        ref_dev = otk.otk_policy_loss_fwd_bwd(ctx, mb.logits, mb.targets, step.masks["loss_mask"][mb.r0:mb.r1],
                                              step.masks["row_traj"][mb.r0:mb.r1], adv, mb.old_logp, mb.ref_logp,
                                              step.masks["n_loss"], cfg, dlogits=mb.dlogits, want_logp=False)
        torch.cuda.synchronize()
        match = bool(torch.equal(ref_dev["dlogits"][j].cpu(), dl_host[j]))
    row_bytes = W["bufs"][0].shape[1] * W["bufs"][0].element_size()
    side_b = 4 + 1 + 4 + 4 + (4 if mbs[0].ref_logp is not None else 0)
    # logits rows cross PCIe only when trainable (the C ABI copies the runs of loss_mask != 0 rows), and so do
    # their gradient rows on the way back
    n_train = int(lm_h.sum().item())
    h2d = n_train * row_bytes + N * side_b + len(mbs) * (adv_h.numel() * 8 + 8)
    d2h = n_train * W["V"] * W["bufs"][0].element_size() + len(mbs) * 40
    total = W["tb_full"].num_rows if W["strong"] else N * world
    return {"value": total / dt, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
            "h2d_GBps": h2d / dt / 1e9, "d2h_GBps": d2h / dt / 1e9,
            "dlogits_returned_equal_device": match,
            "path": "otk_policy_loss_fwd_bwd_host (C ABI, pinned host buffers, 4096-row chunks double-buffered; "
                    "logits of loss-masked rows are not copied; the gradient rows of trainable tokens come back "
                    "D2H into a pinned host buffer, masked rows' zero gradient is implied by loss_mask)",
            "clock": "host wall clock around the blocking C-ABI calls" + ("; rank 0" if world > 1 else "")}


def cpu_baseline(args, W, cfg, seconds=None):
    """The C float64 oracle (as it stands) on a bounded sample of the same workload, all host cores.
    Its inputs are the seeded generator's (logits, targets) plus masks / advantages / old / ref computed
    by the oracle itself — nothing from the CUDA path."""
    from oracle import oracle_cpu as OC
    from oracle import oracle_ref as O
    from synth import make_noise
    seconds = args.cpu_seconds if seconds is None else seconds
    tb, cfgw = W["tb"], W["cfgw"]
    mb = W["mbs"][0]
    m = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len, tb.terminated,
                      traj_agent=tb.traj_agent)
    if W["strong"]:   # this rank's shard of one global batch: global token count, group statistics over all ranks
        tf = W["tb_full"]
        m["n_loss"] = O.build_masks(tf.tok_offsets, tf.seg_offsets, tf.seg_source, tf.seg_agent, tf.seg_len,
                                    tf.terminated, traj_agent=tf.traj_agent)["n_loss"]
        adv = O.group_advantages(tf.group_id, O.episode_returns(tf.turn_offsets, tf.turn_rewards),
                                 cfgw.num_groups)["adv"][W["b0"]:W["b0"] + tb.num_traj]
    else:
        adv = O.group_advantages(tb.group_id - tb.group_id.min(), O.episode_returns(tb.turn_offsets, tb.turn_rewards),
                                 cfgw.num_groups)["adv"]
    ocfg = O.LossCfg(kl_beta=cfg.kl_beta)
    threads = os.cpu_count()
    done, ntrain, t_used, r0, block = 0, 0, 0.0, 0, 64
    olds, refs = [], []
    while t_used < seconds and r0 + block <= mb.r1 - mb.r0:
        lg = OC.bf16_bits(mb.logits[r0:r0 + block]) if cfgw.dtype == "bf16" else mb.logits[r0:r0 + block].cpu().numpy()
        tg = mb.targets[r0:r0 + block].cpu().numpy()
        base = OC.logprob_entropy(lg, tg)["logp"]
        old = (base + make_noise(block, 0.05, 7000 + r0).double().numpy()).astype(np.float32)
        ref = (base + make_noise(block, 0.1, 9000 + r0).double().numpy()).astype(np.float32) if cfg.kl_beta else None
        lm = m["loss_mask"][r0:r0 + block]
        olds.append(old)
        refs.append(ref)
        t = time.perf_counter()
        OC.policy_loss(lg, tg, lm, m["row_traj"][r0:r0 + block], adv, old, ref, m["n_loss"], ocfg)
        t_used += time.perf_counter() - t
        done += block
        ntrain += int(lm.sum())
        r0 += block
        block = min(block * 2, 1024)
    # the same oracle on ONE thread, on the first 256 rows (libgomp's thread count, then back)
    one = None
    try:
        import ctypes
        gomp = ctypes.CDLL("libgomp.so.1")
        n1 = min(256, mb.r1 - mb.r0)
        lg = OC.bf16_bits(mb.logits[:n1]) if cfgw.dtype == "bf16" else mb.logits[:n1].cpu().numpy()
        tg = mb.targets[:n1].cpu().numpy()
        base = OC.logprob_entropy(lg, tg)["logp"]
        old = (base + make_noise(n1, 0.05, 7000).double().numpy()).astype(np.float32)
        ref = (base + make_noise(n1, 0.1, 9000).double().numpy()).astype(np.float32) if cfg.kl_beta else None
        gomp.omp_set_num_threads(1)
        t = time.perf_counter()
        OC.policy_loss(lg, tg, m["loss_mask"][:n1], m["row_traj"][:n1], adv, old, ref, m["n_loss"], ocfg)
        one = n1 / (time.perf_counter() - t)
        gomp.omp_set_num_threads(threads)
    except OSError:
        pass
    res = {"value": done / t_used, "unit": UNIT, "cores": threads, "kind": "oracle", "value_1thread": one,
           "sample": f"first {done} rows of micro-batch 0 of the {args.config} workload ({ntrain} trainable): "
                     f"fused loss fwd+bwd with dlogits materialised, C float64 oracle (oracle/oracle_cpu.c, "
                     f"OpenMP {threads} threads), {t_used:.1f} s; value_1thread: the first 256 rows on one thread"}
    inputs = dict(rows=done, masks=m, adv=adv, old=np.concatenate(olds) if olds else None,
                  ref=np.concatenate(refs) if refs and cfg.kl_beta else None, ocfg=ocfg)
    return res, inputs


def parity_block(W, step, cfg, inp):
    """the CUDA path against the C float64 oracle on the cpu_baseline sample, every row
    (oracle/parity.py; error / tolerance ratios <= 1 pass). Masks and advantages over this rank's whole batch;
    the loss kernel (in the bench's launch configuration) re-run on the sampled rows of micro-batch 0 with the
    oracle's masks, advantages and old / ref (= oracle logp + noise) as inputs. Untimed, after the timed region."""
    from oracle import parity as P
    otk, ctx, cfgw = W["otk"], W["ctx"], W["cfgw"]
    m, n = inp["masks"], inp["rows"]
    dev = W["bufs"][0].device
    adv_gpu = step.adv_used.double().cpu().numpy()
    out = {"masks_bit_exact": bool(np.array_equal(step.masks["loss_mask"].cpu().numpy(), m["loss_mask"])
                                   and np.array_equal(step.masks["row_traj"].cpu().numpy(), m["row_traj"])
                                   and int(step.masks["n_loss"].item()) == m["n_loss"]),
           "adv_max_abs_err": float(np.max(np.abs(adv_gpu - inp["adv"]))),
           "adv_tol": P.ADV_TOL}
    out["adv_ratio"] = out["adv_max_abs_err"] / P.ADV_TOL
    if n == 0:
        return out
    mb = W["mbs"][0]
    lg, tg = mb.logits[:n], mb.targets[:n]
    lm, rt = m["loss_mask"][:n], m["row_traj"][:n]
    dl = W["dlogits"][:n]
    r = otk.otk_policy_loss_fwd_bwd(ctx, lg, tg, torch.from_numpy(lm).to(dev), torch.from_numpy(rt).to(dev),
                                    torch.from_numpy(inp["adv"]).to(dev), torch.from_numpy(inp["old"]).to(dev),
                                    None if inp["ref"] is None else torch.from_numpy(inp["ref"]).to(dev),
                                    torch.tensor([m["n_loss"]], dtype=torch.int64, device=dev), cfg, dlogits=dl)
    ctx.check()
    par = P.microbatch_parity(lg, tg, lm, rt, inp["adv"], inp["old"], inp["ref"], m["n_loss"], inp["ocfg"],
                              cfgw.dtype, W["V"], r["logp"], r["entropy"], dl, otk.stats_dict(r["stats"]))
    out.update(par)
    out["tolerances"] = {"logp": P.LOGP_TOL[cfgw.dtype], "entropy": P.LOGP_TOL[cfgw.dtype],
                         "dlogits_elem": f"{P.DL_REL[cfgw.dtype]:.4g}|ref| + dcoef|p-onehot| (+ target term)",
                         "dlogits_l1": P.DL_L1_REL[cfgw.dtype], "loss_rel": P.LOSS_REL, "adv": P.ADV_TOL}
    out["pass"] = bool(P.parity_ok(par) and out["masks_bit_exact"] and out["adv_ratio"] <= 1)
    return out


# ------------------------------------------------------------------------------------------------
def run_reference(args):
    """--impl reference: the float64 oracle as it stands on the host cores (the base contract's
    reference arm for this tier). Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle import oracle_cpu as OC
    from oracle import oracle_ref as O
    from synth import CONFIGS, make_batch, make_logits, make_noise
    cfgw = CONFIGS[args.config]
    tb = make_batch(args.config)
    V = cfgw.V
    rows = 256   # bounded per-step sample: the whole --steps/--warmup run stays within minutes
    m = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len, tb.terminated,
                      traj_agent=tb.traj_agent)
    R = O.episode_returns(tb.turn_offsets, tb.turn_rewards)
    adv = O.group_advantages(tb.group_id, R, cfgw.num_groups)["adv"]
    lg, tg = make_logits(rows, V, dtype=cfgw.dtype, seed=cfgw.seed * 100, device="cpu")
    bits = OC.bf16_bits(lg) if cfgw.dtype == "bf16" else lg.numpy()
    base = OC.logprob_entropy(bits, tg.numpy())["logp"]
    old = (base + make_noise(rows, 0.05, 7000).double().numpy()).astype(np.float32)
    ref = (base + make_noise(rows, 0.1, 9000).double().numpy()).astype(np.float32)
    ocfg = O.LossCfg(kl_beta=cfgw.kl_beta)

    def step():
        mm = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len, tb.terminated,
                           traj_agent=tb.traj_agent)
        aa = O.group_advantages(tb.group_id, O.episode_returns(tb.turn_offsets, tb.turn_rewards), cfgw.num_groups)
        OC.policy_loss(bits, tg.numpy(), mm["loss_mask"][:rows], mm["row_traj"][:rows], aa["adv"], old,
                       ref if cfgw.kl_beta else None, mm["n_loss"], ocfg)

    for _ in range(args.warmup):
        step()
    t = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t) / args.steps
    threads = os.cpu_count()
    sample = (f"per step: masks + advantages of the full {args.config} batch ({tb.num_traj} trajectories, "
              f"pure-Python oracle) + fused loss fwd+bwd of its first {rows} rows "
              f"({int(m['loss_mask'][:rows].sum())} trainable; C float64 oracle, OpenMP {threads} threads)")
    value = rows / dt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {cfgw.note}", "rows_per_step_sample": rows},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_otk(args)


if __name__ == "__main__":
    main()
