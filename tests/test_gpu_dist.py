"""Multi-rank step on the GPU (-m gpu): two processes share cuda:0 over gloo (NCCL refuses two ranks per
device, and the box has one GPU), running the product's batch- and vocab-sharded steps with the real kernels.
The sharded results must equal the unsharded step: advantages bit-exact, token counts exact, loss to fp64
summation order, dlogits of every shard equal to the unsharded columns within the bf16 tolerance."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch():
    from synth.trajectories import random_small_batch
    rng = np.random.default_rng(11)
    tb = random_small_batch(rng, 24, max_segs=8, max_len=40, num_groups=4)
    tb.group_id = (np.arange(24) % 4).astype(np.int32)      # every group straddles both ranks
    return tb


def _sub(tb, b0, b1):
    from tests.test_dist_gloo import _sub_batch
    return _sub_batch(tb, b0, b1)


def _worker(rank, world, port, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if mode == "2d":
        return _worker_2d(rank, world, q)
    torch.cuda.set_device(0)
    try:
        import paper_2601_07376_b200 as otk
        from paper_2601_07376_b200.dist import plan_batch_shards, traj_costs, vocab_shard_bounds
        from paper_2601_07376_b200.step import MicroBatch, PolicyLossStep, VocabShard
        from synth import make_logits, make_noise
        dev = "cuda"
        ctx = otk.Context(0)
        tb = _batch()
        V = 4096
        N = tb.num_rows
        logits, targets = make_logits(N, V, dtype="bf16", seed=3, device=dev)
        lp = otk.otk_logprob_entropy_fwd(ctx, logits, targets)["logp"]
        old = (lp + make_noise(N, 0.05, 1, device=dev)).contiguous()
        ref = (lp + make_noise(N, 0.1, 2, device=dev)).contiguous()
        cfg = otk.LossCfg()

        credit = "turn" if mode == "batch_turn" else "trajectory"

        def step_for(b, pg=None, counts=None, vshard=None, cols=(0, V), seg_counts=None):
            db = otk.traj_batch_to_device(b, dev)
            st = PolicyLossStep(ctx, db, torch.from_numpy(b.group_id).to(dev), 4,
                                torch.from_numpy(b.turn_offsets).to(dev), torch.from_numpy(b.turn_rewards).to(dev),
                                cols[1] - cols[0], cfg, process_group=pg, global_num_traj=counts,
                                global_num_groups=4 if pg is not None else None, vocab_shard=vshard,
                                credit=credit, gamma=0.9, global_num_segments=seg_counts)
            return st, db

        # unsharded reference on every rank
        st0, _ = step_for(tb)
        dl0 = torch.empty_like(logits)
        st0.run([MicroBatch(0, N, logits, targets, old, ref, dl0)])
        res = dict(rank=rank, ref_loss=otk.stats_dict(st0.stats), ref_adv=st0.adv_out["adv"].cpu().numpy())
        if mode in ("batch", "batch_turn"):
            plan = plan_batch_shards(traj_costs(tb, V), world)
            b0, b1 = plan[rank]
            loc = _sub(tb, b0, b1)
            r0, r1 = int(tb.tok_offsets[b0]), int(tb.tok_offsets[b1])
            st, _ = step_for(loc, pg=dist.group.WORLD, counts=[e - s for s, e in plan],
                             seg_counts=[int(tb.seg_offsets[e] - tb.seg_offsets[s]) for s, e in plan])
            dl = torch.empty_like(logits[r0:r1])
            adv = st.masks_and_advantages()
            if mode == "batch_turn":     # advantages live on segments: compare the rank's segment range
                b0, b1 = int(tb.seg_offsets[b0]), int(tb.seg_offsets[b1])
            st.loss(adv, [MicroBatch(0, r1 - r0, logits[r0:r1].contiguous(), targets[r0:r1].contiguous(),
                                     old[r0:r1].contiguous(), ref[r0:r1].contiguous(), dl)])
            res.update(adv=adv.cpu().numpy(), b0=b0, b1=b1, loss=otk.stats_dict(st.stats),
                       n_loss=int(st.masks["n_loss"].item()), n_loss_ref=int(st0.masks["n_loss"].item()),
                       dl_equal=bool(torch.equal(dl, dl0[r0:r1])))
        elif mode == "lmhead_vocab":
            from paper_2601_07376_b200.step import LMHeadVocabShard
            from synth import make_lmhead
            Vh = 20000
            h, w, yy = make_lmhead(300, Vh, 128, seed=5, device=dev)
            v0, v1 = vocab_shard_bounds(Vh, world)[rank]
            out = LMHeadVocabShard(ctx, v0, Vh, dist.group.WORLD).forward(h, w[v0:v1].contiguous(), yy)
            full = otk.otk_lmhead_logprob_fwd(ctx, h, w, yy)
            res.update(loss=res["ref_loss"], lm_err=float((out["logp"] - full["logp"]).abs().max()),
                       lm_logp=out["logp"].cpu().numpy())
        else:
            v0, v1 = vocab_shard_bounds(V, world)[rank]
            if mode == "vocab_fused":   # K4-VPF: peers' exchange buffers mapped through CUDA IPC handles
                from paper_2601_07376_b200.dist import open_vpf_exchange
                from paper_2601_07376_b200.step import VocabShardFused
                xchg = open_vpf_exchange(ctx, N, dist.group.WORLD)
                vs = VocabShardFused(ctx, v0, v1 - v0, V, xchg, dist.group.WORLD)
            else:
                vs = VocabShard(ctx, v0, v1 - v0, V, dist.group.WORLD)
            st, _ = step_for(tb, vshard=vs, cols=(v0, v1))
            shard = logits[:, v0:v1].contiguous()
            dl = torch.empty_like(shard)
            st.run([MicroBatch(0, N, shard, targets, old, ref, dl)])
            fwd = vs.forward(shard, targets)
            res.update(loss=otk.stats_dict(st.stats),
                       fwd_logp_err=float((fwd["logp"] - lp).abs().max()),
                       dl_err=float(((dl.float() - dl0[:, v0:v1].float()).abs()
                                     / (dl0[:, v0:v1].float().abs() * 2 ** -6 + 1e-6)).max()))
        ctx.check()
        q.put(res)
    finally:
        dist.destroy_process_group()


def _worker_2d(rank, world, q):
    """2-D sharding, world 4 = 2 trajectory shards x 2 vocab shards: PolicyLossStep with the batch group as its
    process group and a VocabShard over the vocab group; compared with the unsharded step on the same data."""
    torch.cuda.set_device(0)
    try:
        import paper_2601_07376_b200 as otk
        from paper_2601_07376_b200.dist import make_2d_groups, plan_batch_shards, traj_costs, vocab_shard_bounds
        from paper_2601_07376_b200.step import MicroBatch, PolicyLossStep, VocabShard
        from synth import make_logits, make_noise
        dev = "cuda"
        ctx = otk.Context(0)
        b, v, bg, vg = make_2d_groups(2)
        tb = _batch()
        V, N = 4096, tb.num_rows
        logits, targets = make_logits(N, V, dtype="bf16", seed=3, device=dev)
        lp = otk.otk_logprob_entropy_fwd(ctx, logits, targets)["logp"]
        old = (lp + make_noise(N, 0.05, 1, device=dev)).contiguous()
        ref = (lp + make_noise(N, 0.1, 2, device=dev)).contiguous()
        cfg = otk.LossCfg()

        def step_for(bb, pg=None, counts=None, vshard=None, Vl=V):
            db = otk.traj_batch_to_device(bb, dev)
            return PolicyLossStep(ctx, db, torch.from_numpy(bb.group_id).to(dev), 4,
                                  torch.from_numpy(bb.turn_offsets).to(dev), torch.from_numpy(bb.turn_rewards).to(dev),
                                  Vl, cfg, process_group=pg, global_num_traj=counts,
                                  global_num_groups=4 if pg is not None else None, vocab_shard=vshard)

        st0 = step_for(tb)
        dl0 = torch.empty_like(logits)
        st0.run([MicroBatch(0, N, logits, targets, old, ref, dl0)])
        plan = plan_batch_shards(traj_costs(tb, V), 2)
        b0, b1 = plan[b]
        r0, r1 = int(tb.tok_offsets[b0]), int(tb.tok_offsets[b1])
        v0, v1 = vocab_shard_bounds(V, 2)[v]
        st = step_for(_sub(tb, b0, b1), pg=bg, counts=[e - s for s, e in plan],
                      vshard=VocabShard(ctx, v0, v1 - v0, V, vg), Vl=v1 - v0)
        blk = logits[r0:r1, v0:v1].contiguous()
        dl = torch.empty_like(blk)
        st.run([MicroBatch(0, r1 - r0, blk, targets[r0:r1].contiguous(), old[r0:r1].contiguous(),
                           ref[r0:r1].contiguous(), dl)])
        ctx.check()
        ref_blk = dl0[r0:r1, v0:v1].float()
        q.put(dict(rank=rank, loss=otk.stats_dict(st.stats), ref_loss=otk.stats_dict(st0.stats),
                   adv=st.adv_g["adv"].cpu().numpy(), ref_adv=st0.adv_out["adv"].cpu().numpy(),
                   n_loss=int(st.masks["n_loss"].item()), n_loss_ref=int(st0.masks["n_loss"].item()),
                   dl_err=float(((dl.float() - ref_blk).abs() / (ref_blk.abs() * 2 ** -6 + 1e-6)).max())))
    finally:
        dist.destroy_process_group()


def test_2d_sharded_step_four_ranks_one_gpu():
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, "2d", q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in res:
        ref = r["ref_loss"]
        assert abs(r["loss"]["loss"] - ref["loss"]) <= 1e-5 * max(abs(ref["loss"]), 1e-6)
        assert r["loss"]["n_tokens"] == ref["n_tokens"] and r["n_loss"] == r["n_loss_ref"]
        assert np.array_equal(r["adv"], r["ref_adv"])      # global group statistics on every rank
        assert r["dl_err"] <= 1.0
    assert res[0]["loss"]["loss"] == res[1]["loss"]["loss"]   # the two vocab ranks of a row block agree


@pytest.mark.parametrize("mode", ["batch", "vocab", "batch_turn", "lmhead_vocab", "vocab_fused"])
def test_sharded_step_two_ranks_one_gpu(mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = res[0]["ref_loss"]
    for r in res:
        rel = abs(r["loss"]["loss"] - ref["loss"]) / max(abs(ref["loss"]), 1e-6)
        assert rel < 1e-5, (r["loss"], ref)
        assert r["loss"]["n_tokens"] == ref["n_tokens"]
    if mode in ("batch", "batch_turn"):
        for r in res:
            assert np.array_equal(r["adv"], r["ref_adv"][r["b0"]:r["b1"]])     # global group statistics
            assert r["n_loss"] == r["n_loss_ref"]                               # global token count
            assert r["dl_equal"]                                                # same kernel, same rows
    elif mode == "lmhead_vocab":
        for r in res:
            assert r["lm_err"] < 1e-5                                           # = the unsharded fused head
        assert np.array_equal(res[0]["lm_logp"], res[1]["lm_logp"])             # identical on every rank
    else:
        assert res[0]["loss"]["loss"] == res[1]["loss"]["loss"]                 # identical on every rank
        for r in res:
            assert r["fwd_logp_err"] < 1e-5 and r["dl_err"] <= 1.0
