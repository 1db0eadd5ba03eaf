"""Multi-rank host logic of the two sharding modes on CPU (gloo, world size 2) — DESIGN.md §7.

The product's shard planning and collectives (paper_2601_07376_b200.dist) run under gloo; the per-rank
compute is done by the float64 oracle standing in for the device kernels, and the sharded results must
equal the unsharded oracle: integers bit-exact, group statistics bit-exact (same inputs, same order),
floats to 1e-12.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_07376_b200.dist import (all_gather_group_returns, all_gather_vocab_partials, all_reduce_n_loss,
                                        all_reduce_stats, plan_batch_shards, traj_costs, vocab_shard_bounds)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sub_batch(tb, b0, b1):
    from synth import slice_batch
    return slice_batch(tb, b0, b1)


def _worker(rank, world, port, config, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle_ref as O
        from synth import make_batch
        tb = make_batch(config)
        V = 1000
        # ---- batch sharding: plan, local masks/returns (oracle stands in for the kernels), exchanges
        plan = plan_batch_shards(traj_costs(tb, 151936), world)
        b0, b1 = plan[rank]
        counts = [e - s for s, e in plan]
        loc = _sub_batch(tb, b0, b1)
        m_loc = O.build_masks(loc.tok_offsets, loc.seg_offsets, loc.seg_source, loc.seg_agent, loc.seg_len,
                              loc.terminated, traj_agent=loc.traj_agent)
        n_loss = torch.tensor([m_loc["n_loss"]], dtype=torch.int64)
        all_reduce_n_loss(n_loss)
        R_loc = torch.from_numpy(O.episode_returns(loc.turn_offsets, loc.turn_rewards))
        gid_g, ret_g = all_gather_group_returns(torch.from_numpy(loc.group_id), R_loc, counts)
        adv_g = O.group_advantages(gid_g.numpy(), ret_g.numpy(), tb.num_groups)["adv"]
        # ---- turn-level credit (R31): per-segment returns gathered with the per-rank SEGMENT counts
        seg_counts = [int(tb.seg_offsets[e] - tb.seg_offsets[s]) for s, e in plan]
        G_loc, grp_loc = O.turn_returns(loc.seg_offsets, loc.seg_source, loc.seg_agent, loc.turn_offsets,
                                        loc.turn_rewards, loc.group_id, 0.9, traj_agent=loc.traj_agent)
        sg_g, sr_g = all_gather_group_returns(torch.from_numpy(grp_loc), torch.from_numpy(G_loc), seg_counts)
        tadv_g = O.group_advantages(sg_g.numpy(), sr_g.numpy(), tb.num_groups, skip_ungrouped=True)["adv"]
        # ---- loss partial sums with the GLOBAL N, then all-reduce of the stats
        rng = np.random.default_rng(100 + rank)
        rows = np.flatnonzero(m_loc["loss_mask"])[:6]
        logits = rng.normal(scale=2.0, size=(len(rows), V))
        y = rng.integers(0, V, len(rows))
        lp = np.array([O.row_forward(logits[i], int(y[i]))[0] for i in range(len(rows))])
        adv_loc = adv_g[b0:b1]
        cfg = O.LossCfg(kl_beta=0.0)
        L = [O.row_loss_terms(lp[i], lp[i], None, float(adv_loc[m_loc["row_traj"][r]]), cfg)[0]
             for i, r in enumerate(rows)]
        stats = torch.tensor([math.fsum(L) / int(n_loss.item()), float(len(rows)), 0.0, 0.0, float(len(rows))],
                             dtype=torch.float64)
        all_reduce_stats(stats)
        # ---- vocab sharding: per-rank partials of the same rows, gathered in rank order
        vrng = np.random.default_rng(7)
        X = vrng.normal(scale=3.0, size=(5, 1003))
        X[2, 17] = -np.inf
        Y = vrng.integers(0, 1003, 5)
        v0, v1 = vocab_shard_bounds(1003, world)[rank]
        part = torch.tensor([O.shard_partials(X[j, v0:v1], int(Y[j]), v0) for j in range(5)], dtype=torch.float64)
        gathered = all_gather_vocab_partials(part)
        comb = [O.combine_partials([tuple(gathered[k, j].tolist()) for k in range(world)]) for j in range(5)]
        q.put(dict(rank=rank, n_loss=int(n_loss.item()), gid=gid_g.numpy(), ret=ret_g.numpy(), adv=adv_g,
                   plan=plan, stats=stats.numpy(), L=L, comb=comb, X=X, Y=Y, tadv=tadv_g,
                   loss_mask=m_loc["loss_mask"], row_traj=m_loc["row_traj"] + b0, adv_loc=adv_g[b0:b1]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("config", ["game", "marl", "math"])
def test_batch_and_vocab_sharding_gloo(config):
    from oracle import oracle_ref as O
    from synth import make_batch
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, config, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tb = make_batch(config)
    full = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len, tb.terminated,
                         traj_agent=tb.traj_agent)
    R = O.episode_returns(tb.turn_offsets, tb.turn_rewards)
    adv = O.group_advantages(tb.group_id, R, tb.num_groups)["adv"]
    # the shards' per-row labels, concatenated in rank order, are the unsharded ones (bit-exact), and every
    # rank's advantages of its own trajectories equal the unsharded oracle's (groups straddle the ranks: game
    # ids are b mod 16, marl agent * 8 + episode group)
    assert np.array_equal(np.concatenate([r["loss_mask"] for r in res]), full["loss_mask"])
    assert np.array_equal(np.concatenate([r["row_traj"] for r in res]), full["row_traj"])
    assert np.max(np.abs(np.concatenate([r["adv_loc"] for r in res]) - O.group_advantages(
        tb.group_id, O.episode_returns(tb.turn_offsets, tb.turn_rewards), tb.num_groups)["adv"])) <= 1e-6
    if config == "game":
        for g in range(tb.num_groups):            # every group really spans both ranks
            members = np.flatnonzero(tb.group_id == g)
            assert members.min() < res[0]["plan"][0][1] <= members.max()
    for r in res:
        assert r["n_loss"] == full["n_loss"]                       # global token count, bit-exact
        assert np.array_equal(r["gid"], tb.group_id)               # gathered in rank order
        assert np.array_equal(r["ret"], R)
        assert np.array_equal(r["adv"], adv)                       # identical stats on every rank
    G, grp = O.turn_returns(tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.turn_offsets, tb.turn_rewards,
                            tb.group_id, 0.9, traj_agent=tb.traj_agent)
    tadv = O.group_advantages(grp, G, tb.num_groups, skip_ungrouped=True)["adv"]
    for r in res:
        assert np.array_equal(r["tadv"], tadv)                     # turn-level: same segments, same order
    assert np.array_equal(res[0]["stats"], res[1]["stats"])
    want = (math.fsum(res[0]["L"]) + math.fsum(res[1]["L"])) / full["n_loss"]
    assert abs(res[0]["stats"][0] - want) < 1e-14
    for j in range(5):
        ref = O.row_forward(res[0]["X"][j], int(res[0]["Y"][j]))
        for r in res:
            assert abs(r["comb"][j][0] - ref[0]) < 1e-12 and abs(r["comb"][j][1] - ref[1]) < 1e-12


def test_plan_batch_shards_balanced():
    from synth import make_batch
    for name in ("math", "game", "marl"):
        tb = make_batch(name)
        c = traj_costs(tb, 151936)
        for world in (2, 4, 8):
            plan = plan_batch_shards(c, world)
            assert plan[0][0] == 0 and plan[-1][1] == len(c)
            assert all(a < b for a, b in plan) and all(plan[i][1] == plan[i + 1][0] for i in range(world - 1))
            loads = [c[a:b].sum() for a, b in plan]
            assert max(loads) <= c.sum() / world + c.max() + 1e-6   # within one trajectory of ideal
    with pytest.raises(ValueError):
        plan_batch_shards([1.0], 2)


def test_vocab_shard_bounds():
    for V, P in ((151936, 2), (151936, 4), (151936, 8), (1003, 3)):
        b = vocab_shard_bounds(V, P)
        assert b[0][0] == 0 and b[-1][1] == V
        assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
        assert all(x[0] % 8 == 0 for x in b)
    assert vocab_shard_bounds(151936, 4)[1] == (37984, 75968)


def _worker_2d(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle_ref as O
        from paper_2601_07376_b200.dist import make_2d_groups
        from synth import make_batch
        b, v, bg, vg = make_2d_groups(2)
        # group membership: sum of WORLD ranks inside each group
        t = torch.tensor([float(rank)])
        dist.all_reduce(t, group=bg)
        u = torch.tensor([float(rank)])
        dist.all_reduce(u, group=vg)
        # batch exchanges inside the batch group: n_loss of this rank's trajectory shard
        tb = make_batch("game")
        plan = plan_batch_shards(traj_costs(tb, 151936), 2)
        b0, b1 = plan[b]
        loc = _sub_batch(tb, b0, b1)
        m_loc = O.build_masks(loc.tok_offsets, loc.seg_offsets, loc.seg_source, loc.seg_agent, loc.seg_len,
                              loc.terminated, traj_agent=loc.traj_agent)
        n_loss = torch.tensor([m_loc["n_loss"]], dtype=torch.int64)
        all_reduce_n_loss(n_loss, bg)
        # row partials inside the vocab group: rows of batch shard b, columns of vocab shard v
        rng = np.random.default_rng(50 + b)
        X = rng.normal(scale=3.0, size=(4, 1003))
        Y = rng.integers(0, 1003, 4)
        v0, v1 = vocab_shard_bounds(1003, 2)[v]
        part = torch.tensor([O.shard_partials(X[j, v0:v1], int(Y[j]), v0) for j in range(4)], dtype=torch.float64)
        g = all_gather_vocab_partials(part, vg)
        comb = [O.combine_partials([tuple(g[k, j].tolist()) for k in range(2)]) for j in range(4)]
        q.put(dict(rank=rank, b=b, v=v, bsum=float(t.item()), vsum=float(u.item()), n_loss=int(n_loss.item()),
                   comb=comb, X=X, Y=Y))
    finally:
        dist.destroy_process_group()


def test_2d_batch_vocab_groups_gloo():
    """2-D sharding (world 4 = 2 batch x 2 vocab): group membership, the global token count over the batch
    group, and the rank-order combine of row partials over the vocab group equal the unsharded values."""
    from oracle import oracle_ref as O
    from synth import make_batch
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_2d, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tb = make_batch("game")
    full = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len, tb.terminated,
                         traj_agent=tb.traj_agent)
    for r in res:
        assert (r["b"], r["v"]) == divmod(r["rank"], 2)
        assert r["bsum"] == r["v"] + (2 + r["v"])          # batch group {v, 2 + v}
        assert r["vsum"] == 2 * r["b"] + (2 * r["b"] + 1)  # vocab group {2b, 2b + 1}
        assert r["n_loss"] == full["n_loss"]               # global count over the batch group
        for j in range(4):
            lp, H = O.row_forward(r["X"][j], int(r["Y"][j]))[:2]
            assert abs(r["comb"][j][0] - lp) < 1e-12 and abs(r["comb"][j][1] - H) < 1e-12


def _worker_vpf_setup(rank, world, port, q):
    """dist.open_vpf_exchange's host logic with the CUDA calls stubbed (CPU): every rank allocates its buffer,
    the 64-byte handles are all-gathered in rank order, and each rank maps the OTHER ranks' handles."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2601_07376_b200 as otk
        from paper_2601_07376_b200 import dist as D
        base = 0x10000 * (rank + 1)
        opened = []
        otk.otk_xchg_alloc = lambda ctx, n: base
        otk.otk_ipc_get_handle = lambda ptr: ptr.to_bytes(8, "little") * 8
        otk.otk_ipc_open = lambda h: (opened.append(h), 0x7000000 + int.from_bytes(h[:8], "little"))[1]
        x = D.open_vpf_exchange(object(), 1024)
        q.put(dict(rank=rank, ptrs=x.ptrs, nranks=x.nranks, me=x.rank, opened=[int.from_bytes(h[:8], "little")
                                                                               for h in opened]))
    finally:
        dist.destroy_process_group()


def test_open_vpf_exchange_host_logic_gloo():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_vpf_setup, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in res:
        k = r["rank"]
        assert r["me"] == k and r["nranks"] == world
        assert r["ptrs"][k] == 0x10000 * (k + 1)                                   # own buffer, unmapped
        assert r["opened"] == [0x10000 * (j + 1) for j in range(world) if j != k]  # peers, rank order
        assert all(r["ptrs"][j] == 0x7000000 + 0x10000 * (j + 1) for j in range(world) if j != k)


def _worker_layout(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import argparse
        import importlib.util
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
        bench = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(bench)
        out = {}
        for shard in ("batch", "vocab", "2d"):
            L = bench.shard_layout(argparse.Namespace(shard=shard, vocab_ways=2), world, rank)
            t = torch.tensor([float(rank)])
            if L["vg"] is not None:
                dist.all_reduce(t, group=L["vg"])
            out[shard] = (L["Pv"], L["nb"], L["b"], L["v"], float(t.item()))
        q.put(dict(rank=rank, out=out))
    finally:
        dist.destroy_process_group()


def test_bench_shard_layout_gloo():
    """bench.py's rank layout for --shard batch / vocab / 2d (world 4, 2 vocab ways): shard counts, this rank's
    (batch, vocab) index and the vocab group's membership."""
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_layout, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in res:
        k = r["rank"]
        assert r["out"]["batch"][:4] == (1, 4, k, 0)
        assert r["out"]["vocab"][:4] == (4, 1, 0, k) and r["out"]["vocab"][4] == 0 + 1 + 2 + 3
        b, v = divmod(k, 2)
        assert r["out"]["2d"][:4] == (2, 2, b, v) and r["out"]["2d"][4] == 2 * b + (2 * b + 1)
