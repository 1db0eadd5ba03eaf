"""Batch sharding through the library's own NCCL communicator (otk.h "Batch sharding"; SURVEY.md §8(e) BATCH):
otk_comm_* and otk_batch_* on one GPU (a one-rank communicator — NCCL refuses two ranks on one device, and the box
has one GPU; the multi-rank exchanges are the same calls with nranks > 1). The step with collectives="otk" must
equal the unsharded step exactly (the same kernels on the same data; the collectives are identities at one rank),
and the host-checked errors must come back as typed statuses."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import paper_2601_07376_b200 as otk
    torch.cuda.set_device(0)
    ctx = otk.Context(0)
    return otk, ctx


def _batch():
    from synth.trajectories import random_small_batch
    rng = np.random.default_rng(5)
    tb = random_small_batch(rng, 16, max_segs=8, max_len=40, num_groups=4)
    tb.group_id = (np.arange(16) % 4).astype(np.int32)
    return tb


def test_comm_errors_before_and_after_init(env):
    otk, _ = env
    ctx = otk.Context(0)          # a fresh ctx: no communicator
    t = torch.zeros(2, dtype=torch.int64, device="cuda")
    with pytest.raises(otk.OtkError) as e:
        otk.otk_batch_allreduce_i64(ctx, t)
    assert e.value.status == 13   # OTK_ERR_NO_COMM
    with pytest.raises(otk.OtkError):
        otk.otk_comm_size(ctx)
    uid = otk.otk_comm_unique_id()
    assert len(uid) == 128
    with pytest.raises(otk.OtkError) as e:
        otk.otk_comm_init(ctx, uid, 1, 1)           # rank outside [0, nranks)
    assert e.value.status == 2
    otk.otk_comm_init(ctx, uid, 1, 0)
    assert otk.otk_comm_size(ctx) == (1, 0)
    with pytest.raises(otk.OtkError) as e:
        otk.otk_comm_init(ctx, otk.otk_comm_unique_id(), 1, 0)   # already has one
    assert e.value.status == 1
    g = torch.zeros(3, dtype=torch.int32, device="cuda")
    r = torch.zeros(3, dtype=torch.float64, device="cuda")
    with pytest.raises(otk.OtkError) as e:
        otk.otk_batch_group_advantages(ctx, g, r, [4], 2)       # counts[rank] != local trajectories
    assert e.value.status == 2
    otk.otk_comm_destroy(ctx)
    with pytest.raises(otk.OtkError) as e:
        otk.otk_batch_allreduce_f64(ctx, torch.zeros(1, dtype=torch.float64, device="cuda"))
    assert e.value.status == 13


def test_comm_single_rank_collectives(env):
    otk, _ = env
    ctx = otk.Context(0)
    otk.otk_comm_init(ctx, otk.otk_comm_unique_id(), 1, 0)
    a = torch.tensor([3, -7, 1 << 40], dtype=torch.int64, device="cuda")
    b = torch.tensor([0.25, -1e300, 3.0], dtype=torch.float64, device="cuda")
    otk.otk_batch_allreduce_i64(ctx, a)
    otk.otk_batch_allreduce_f64(ctx, b)
    ctx.check()
    assert a.tolist() == [3, -7, 1 << 40] and b.tolist() == [0.25, -1e300, 3.0]
    gid = torch.tensor([0, 1, 0, 2, 1, 0], dtype=torch.int32, device="cuda")
    ret = torch.tensor([1.0, 0.0, -1.0, 2.0, 1.0, 0.5], dtype=torch.float64, device="cuda")
    o = otk.otk_batch_group_advantages(ctx, gid, ret, [6], 3)
    ref = otk.otk_group_advantages(ctx, gid, 3, returns=ret)
    ctx.check()
    assert torch.equal(o["gid_all"], gid) and torch.equal(o["ret_all"], ret)
    assert torch.equal(o["adv"], ref["adv"]) and torch.equal(o["group_mean"], ref["group_mean"])
    assert torch.equal(o["group_std"], ref["group_std"]) and torch.equal(o["group_size"], ref["group_size"])
    otk.otk_comm_destroy(ctx)


@pytest.mark.parametrize("credit", ["trajectory", "turn"])
def test_step_with_library_collectives_equals_unsharded(env, credit):
    otk, _ = env
    from paper_2601_07376_b200.step import MicroBatch, PolicyLossStep
    from synth import make_logits, make_noise
    ctx = otk.Context(0)
    otk.otk_comm_init(ctx, otk.otk_comm_unique_id(), 1, 0)
    tb = _batch()
    V, N, dev = 4096, tb.num_rows, "cuda"
    logits, targets = make_logits(N, V, dtype="bf16", seed=3, device=dev)
    lp = otk.otk_logprob_entropy_fwd(ctx, logits, targets)["logp"]
    old = (lp + make_noise(N, 0.05, 1, device=dev)).contiguous()
    ref = (lp + make_noise(N, 0.1, 2, device=dev)).contiguous()
    db = otk.traj_batch_to_device(tb, dev)
    out = {}
    for coll in ("none", "otk"):
        kw = {} if coll == "none" else dict(collectives="otk", global_num_traj=[tb.num_traj], global_num_groups=4,
                                            global_num_segments=[int(tb.seg_len.size)])
        st = PolicyLossStep(ctx, db, torch.from_numpy(tb.group_id).to(dev), 4, torch.from_numpy(tb.turn_offsets).to(dev),
                            torch.from_numpy(tb.turn_rewards).to(dev), V, otk.LossCfg(), credit=credit, gamma=0.9, **kw)
        dl = torch.empty_like(logits)
        adv = st.run([MicroBatch(0, N, logits, targets, old, ref, dl)])
        ctx.check()
        out[coll] = (otk.stats_dict(st.stats), dl, int(st.masks["n_loss"].item()))
    (s0, d0, n0), (s1, d1, n1) = out["none"], out["otk"]
    assert n0 == n1 > 0
    assert s0 == s1
    assert torch.equal(d0, d1)
    otk.otk_comm_destroy(ctx)
