"""CUDA path (through the C ABI) vs the float64 oracle, element by element (-m gpu).

Tolerances (north_star, DESIGN.md §3/§6): masks / row_traj / counts / group sizes bit-exact;
advantages 1e-6 abs; logp / entropy 2e-3 abs for bf16 logits (1e-5 for fp32); loss 1e-4 relative to
max(|loss|, sum m|L|/N); dlogits |d| <= rho |ref| + 1e-5 (|coef_j| + |dcoef_j/dlogp_j|) with rho = 2^-7 (bf16
output) or 1e-5 (fp32): the second term is the absolute error coef inherits from fp32 logp.
"""
import math

import numpy as np
import pytest
import torch

from oracle import oracle_ref as O
from synth import CONFIGS, make_batch
from tests.gpu_common import LOGP_TOL, check_dlogits_rows, dcoef_rows, near_kink, oracle_cfg, row_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def otk():
    import paper_2601_07376_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(otk):
    c = otk.Context(0)
    yield c
    c.close()


# ------------------------------------------------------------------------------------------ (1) masks
@pytest.mark.parametrize("name", list(CONFIGS))
def test_masks_bit_exact(otk, ctx, name):
    tb = make_batch(name)
    want = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len,
                         tb.terminated, traj_agent=tb.traj_agent)
    db = otk.traj_batch_to_device(tb)
    got = otk.otk_build_masks(ctx, db)
    ctx.check()
    for k in ("loss_mask", "response_mask", "row_traj", "traj_loss_tokens", "traj_source_counts"):
        assert np.array_equal(got[k].cpu().numpy(), want[k]), k
    assert int(got["n_loss"].item()) == want["n_loss"]


def test_masks_train_agent_and_errors(otk, ctx):
    from synth.trajectories import _pack, random_small_batch
    rng = np.random.default_rng(5)
    tb = random_small_batch(rng, 300, max_segs=40, max_len=30)   # > 256 segments per tile in some trajectories
    for ta in (-1, 0, 1):
        want = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len,
                             train_agent=ta)
        got = otk.otk_build_masks(ctx, otk.traj_batch_to_device(tb), ta)
        ctx.check()
        assert np.array_equal(got["loss_mask"].cpu().numpy(), want["loss_mask"])
        assert np.array_equal(got["response_mask"].cpu().numpy(), want["response_mask"])
    # > 256 segments in one trajectory (multi-tile scan)
    segs = [(int(rng.integers(0, 4)), int(rng.integers(0, 2)), int(rng.integers(1, 5))) for _ in range(700)]
    tb = _pack([segs, segs[:3]], [[0.0], [0.0]], [0, 0], 1)
    want = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len)
    got = otk.otk_build_masks(ctx, otk.traj_batch_to_device(tb))
    ctx.check()
    assert np.array_equal(got["loss_mask"].cpu().numpy(), want["loss_mask"])
    assert int(got["n_loss"].item()) == want["n_loss"]
    # unterminated -> error word, rows masked
    tb = _pack([[(0, -1, 3), (1, 0, 4)], [(0, -1, 2), (1, 0, 2)]], [[1.0], [0.0]], [0, 0], 1, terminated=[1, 0])
    got = otk.otk_build_masks(ctx, otk.traj_batch_to_device(tb))
    with pytest.raises(otk.OtkError) as e:
        ctx.check()
    assert e.value.name == "OTK_ERR_UNTERMINATED"
    assert got["loss_mask"].cpu().tolist()[7:] == [0, 0, 0, 0]
    # segment lengths that do not cover the rows
    tb = _pack([[(0, -1, 3), (1, 0, 4)]], [[1.0]], [0], 1)
    tb.tok_offsets[1] = 9
    got = otk.otk_build_masks(ctx, otk.traj_batch_to_device(tb))
    with pytest.raises(otk.OtkError) as e:
        ctx.check()
    assert e.value.name == "OTK_ERR_BAD_TRAJECTORY"
    assert int(got["loss_mask"].sum()) == 0
    # empty batch is a host-side error
    tb0 = otk.traj_batch_to_device(tb)
    tb0.num_traj = 0
    with pytest.raises(otk.OtkError) as e:
        otk.otk_build_masks(ctx, tb0)
    assert e.value.name == "OTK_ERR_EMPTY_GROUP"


# ------------------------------------------------------------------------------------------ (2) advantages
@pytest.mark.parametrize("name", list(CONFIGS))
@pytest.mark.parametrize("std_norm,unbiased", [(True, False), (True, True), (False, False)])
def test_advantages(otk, ctx, name, std_norm, unbiased):
    tb = make_batch(name)
    R = O.episode_returns(tb.turn_offsets, tb.turn_rewards)
    want = O.group_advantages(tb.group_id, R, tb.num_groups, std_norm=std_norm, unbiased=unbiased)
    dev = "cuda"
    got = otk.otk_group_advantages(ctx, torch.from_numpy(tb.group_id).to(dev), tb.num_groups,
                                   turn_offsets=torch.from_numpy(tb.turn_offsets).to(dev),
                                   turn_rewards=torch.from_numpy(tb.turn_rewards).to(dev),
                                   std_norm=std_norm, unbiased=unbiased)
    ctx.check()
    assert np.max(np.abs(got["returns"].cpu().numpy() - R)) < 1e-12
    assert np.max(np.abs(got["adv"].cpu().numpy() - want["adv"])) < 1e-6
    assert np.array_equal(got["group_size"].cpu().numpy(), want["group_size"])
    assert np.max(np.abs(got["group_mean"].cpu().numpy() - want["group_mean"])) < 1e-9
    if name == "marl":   # zero-sum => exact antisymmetry
        a = got["adv"].cpu().numpy()
        assert np.array_equal(a[0::2], -a[1::2])


def test_advantage_closed_forms_and_errors(otk, ctx):
    dev = "cuda"
    gid = torch.zeros(8, dtype=torch.int32, device=dev)
    for v in (0.0, 1.0, -0.5):
        got = otk.otk_group_advantages(ctx, gid, 1, returns=torch.full((8,), v, dtype=torch.float64, device=dev))
        assert bool((got["adv"] == 0).all())                 # constant group -> exactly 0
    R = torch.tensor([1.0, 1.0] + [0.0] * 6, dtype=torch.float64, device=dev)
    got = otk.otk_group_advantages(ctx, gid, 1, returns=R)
    a = got["adv"].cpu().numpy()
    assert abs(a[0] - math.sqrt(3)) < 1e-14 and abs(a[-1] + math.sqrt(1 / 3)) < 1e-14
    bad = torch.tensor([0, 3], dtype=torch.int32, device=dev)
    got = otk.otk_group_advantages(ctx, bad, 2, returns=torch.ones(2, dtype=torch.float64, device=dev))
    with pytest.raises(otk.OtkError) as e:
        ctx.check()
    assert e.value.name == "OTK_ERR_GROUP_RANGE"
    with pytest.raises(otk.OtkError):
        otk.otk_group_advantages(ctx, gid, 1)   # neither returns nor turn rewards


# ------------------------------------------------------------------------------------------ (3) forward
@pytest.mark.parametrize("V,ld,dtype,n", [(1024, 1024, "f32", 256), (1000, 1008, "bf16", 300), (4096, 4096, "bf16", 513),
                                          (151936, 151936, "bf16", 160), (33001, 33008, "bf16", 97),
                                          (151936, 151936, "f32", 40), (2, 8, "bf16", 33), (3, 4, "f32", 17),
                                          (262144, 262144, "bf16", 40), (300000, 300000, "f32", 12)])
def test_logprob_entropy_fwd(otk, ctx, V, ld, dtype, n):
    d, h = row_problem(n, V, dtype=dtype, ld=ld, seed=V + n, uniform_rows=(3,))
    rm = d["mask"] if n % 2 else None
    got = otk.otk_logprob_entropy_fwd(ctx, d["logits"], d["targets"], vocab=V, row_mask=rm, want_lse=True)
    ctx.check()
    want = O.logprob_entropy_fwd(h["wide"], h["targets"], row_mask=None if rm is None else h["mask"])
    tol = LOGP_TOL[dtype]
    assert np.max(np.abs(got["logp"].cpu().numpy() - want["logp"])) < tol
    assert np.max(np.abs(got["entropy"].cpu().numpy() - want["entropy"])) < tol
    assert np.max(np.abs(got["lse"].cpu().numpy() - want["lse"])) < tol
    if V == 151936:
        # uniform row: logp = -ln V (north_star pin), exact to fp32 accumulation
        assert abs(float(got["logp"][3]) + math.log(V)) < 1e-5


# ------------------------------------------------------------------------------------------ (4) loss + bwd
CASES = [
    # V, ld, dtype, n, kl_beta, kl_type, scale, zero_masked
    (1024, 1024, "f32", 256, 0.04, 3, 1.0, True),
    (1000, 1008, "bf16", 300, 0.04, 3, 1.0, True),
    (8, 8, "bf16", 64, 0.1, 1, 1.0, True),
    (4096, 4096, "bf16", 200, 0.04, 2, 1 / 0.7, True),
    (33001, 33008, "bf16", 120, 0.0, 3, 1.0, False),
    (151936, 151936, "bf16", 150, 0.04, 3, 1.0, True),
    (151936, 151936, "f32", 24, 0.04, 3, 1 / 0.7, True),
    (262144, 262144, "bf16", 40, 0.04, 3, 1.0, True),     # 3-CTA clusters (Gemma-class vocabulary)
    (300000, 300000, "f32", 10, 0.04, 3, 1.0, True),      # 6-CTA clusters
    (700003, 700008, "bf16", 8, 0.04, 3, 1.0, True),      # 7-CTA clusters (odd size, short last segment)
]


@pytest.mark.parametrize("V,ld,dtype,n,beta,kl_type,scale,zero_masked", CASES)
def test_policy_loss_fwd_bwd(otk, ctx, V, ld, dtype, n, beta, kl_type, scale, zero_masked):
    d, h = row_problem(n, V, dtype=dtype, ld=ld, seed=7 * V + n, force_clip=3, logit_scale=scale, uniform_rows=(1,))
    cfg = otk.LossCfg(kl_beta=beta, kl_type=kl_type, logit_scale=scale, zero_masked_rows=zero_masked)
    N = int(h["mask"].sum())
    n_loss = torch.tensor([N], dtype=torch.int64, device="cuda")
    dl = torch.full_like(d["logits"], 7.0)   # sentinel: masked rows stay 7 when zero_masked_rows = 0
    got = otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"], d["old"],
                                      d["ref"] if beta else None, n_loss, cfg, vocab=V, dlogits=dl)
    ctx.check()
    ocfg = oracle_cfg(cfg)
    want = O.policy_loss_fwd_bwd(h["wide"], h["targets"], h["mask"], h["row_traj"], h["adv"], h["old"],
                                 h["ref"] if beta else None, N, ocfg)
    tol = LOGP_TOL[dtype]
    glogp = got["logp"].cpu().numpy()
    assert np.max(np.abs(glogp - want["logp"])) < tol
    assert np.max(np.abs(got["entropy"].cpu().numpy() - want["entropy"])) < tol
    kinks = {j for j in range(n) if h["mask"][j] and near_kink(want["logp"][j], h["old"][j],
                                                               h["ref"][j] if beta else None,
                                                               h["adv"][h["row_traj"][j]], ocfg)}
    rows = [j for j in range(n) if h["mask"][j]]     # kink rows included: either branch must match in full
    dc = dcoef_rows(h, want["logp"], ocfg, N, beta)
    assert check_dlogits_rows(got["dlogits"], want["dlogits"], want["coef"], rows, dtype, V, dc, wide=h["wide"],
                              targets=h["targets"], scale=scale, h=h, cfg=ocfg) <= 1.0
    masked = [j for j in range(n) if not h["mask"][j]]
    gd = got["dlogits"].float().cpu()
    if zero_masked:
        assert all(bool((gd[j, :V] == 0).all()) for j in masked)
    else:
        assert all(bool((gd[j, :V] == 7).all()) for j in masked)
    if ld > V:
        assert bool((gd[:, V:] == 7).all())   # padding columns never written
    st = otk.stats_dict(got["stats"])
    scale_ = max(abs(want["loss"]), sum(abs(O.row_loss_terms(want["logp"][j], h["old"][j], h["ref"][j] if beta else None,
                                                             h["adv"][h["row_traj"][j]], ocfg)[0])
                                        for j in range(n) if h["mask"][j]) / max(N, 1))
    assert abs(st["loss"] - want["loss"]) <= 1e-4 * scale_          # L is continuous across the kinks
    assert abs(st["n_clipped"] - want["stats"]["n_clipped"]) <= len(kinks)
    assert st["n_tokens"] == N
    assert abs(st["entropy_sum"] - want["stats"]["entropy_sum"]) < tol * max(N, 1)
    # row sums of dlogits are 0 (softmax - onehot), up to bf16 rounding
    rs = gd[rows, :V].double().sum(dim=1).abs()
    coef = torch.tensor([abs(want["coef"][j]) for j in rows], dtype=torch.float64)
    assert bool((rs <= 1e-2 * coef + 1e-12).all())


def test_on_policy_bitwise_and_minus_mean_adv(otk, ctx):
    """old = the fwd pool's own logp (SPEC.md:501 on-policy): ratio is exactly 1, and with ref = logp
    and beta > 0 the KL is exactly 0, so loss = -sum m A / N (north_star pin)."""
    n, V = 300, 151936
    d, h = row_problem(n, V, seed=11)
    fwd = otk.otk_logprob_entropy_fwd(ctx, d["logits"], d["targets"])
    lp = fwd["logp"]
    N = int(h["mask"].sum())
    n_loss = torch.tensor([N], dtype=torch.int64, device="cuda")
    got = otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"], lp, lp,
                                      n_loss, otk.LossCfg())
    ctx.check()
    m = d["mask"].bool()
    assert torch.equal(got["logp"][m], lp[m])            # same reduction order: bitwise equal
    st = otk.stats_dict(got["stats"])
    want = -sum(h["adv"][h["row_traj"][j]] for j in range(n) if h["mask"][j]) / N
    # per-token terms are fp32 on the device (A rounded to fp32: 6e-8 relative), summed in fp64
    assert abs(st["loss"] - want) <= 1e-6 * max(1.0, abs(want))
    assert st["kl_sum"] == 0.0 and st["n_clipped"] == 0


def test_zero_loss_tokens_and_accumulate(otk, ctx):
    n, V = 64, 4096
    d, h = row_problem(n, V, seed=3)
    zero = torch.zeros(1, dtype=torch.int64, device="cuda")
    got = otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"], d["old"],
                                      d["ref"], zero, otk.LossCfg())
    ctx.check()
    assert bool((got["dlogits"] == 0).all()) and otk.stats_dict(got["stats"])["loss"] == 0.0
    # two half-batches accumulated == one full batch (micro-batching)
    N = int(h["mask"].sum())
    nl = torch.tensor([N], dtype=torch.int64, device="cuda")
    full = otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"], d["old"],
                                       d["ref"], nl, otk.LossCfg())
    stats = torch.zeros(5, dtype=torch.float64, device="cuda")
    for i, (a, b) in enumerate(((0, 30), (30, 64))):
        otk.otk_policy_loss_fwd_bwd(ctx, d["logits"][a:b], d["targets"][a:b], d["mask"][a:b], d["row_traj"][a:b],
                                    d["adv"], d["old"][a:b], d["ref"][a:b], nl, otk.LossCfg(), stats=stats,
                                    accumulate=i > 0)
    ctx.check()
    f, s = otk.stats_dict(full["stats"]), otk.stats_dict(stats)
    assert abs(f["loss"] - s["loss"]) < 1e-12 and f["n_tokens"] == s["n_tokens"] == N


def test_target_out_of_range(otk, ctx):
    n, V = 16, 1000
    d, h = row_problem(n, V, seed=2, mask_p=1.0)
    d["targets"][5] = V + 3
    nl = torch.tensor([n], dtype=torch.int64, device="cuda")
    got = otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"], d["old"],
                                      d["ref"], nl, otk.LossCfg())
    with pytest.raises(otk.OtkError) as e:
        ctx.check()
    assert e.value.name == "OTK_ERR_TARGET_RANGE"
    assert bool((got["dlogits"][5] == 0).all())


def test_host_validation(otk, ctx):
    d, h = row_problem(8, 64, seed=1)
    nl = torch.tensor([4], dtype=torch.int64, device="cuda")
    with pytest.raises(otk.OtkError) as e:   # KL on without a reference policy
        otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"], d["old"],
                                    None, nl, otk.LossCfg(kl_beta=0.1))
    assert e.value.name == "OTK_ERR_INVALID_ARG"
    with pytest.raises(otk.OtkError) as e:   # misaligned row stride (ld * 2 bytes not a multiple of 16)
        lg = torch.zeros((8, 63), dtype=torch.bfloat16, device="cuda")
        otk.otk_logprob_entropy_fwd(ctx, lg, d["targets"], vocab=60)
    assert e.value.name == "OTK_ERR_ALIGNMENT"
    with pytest.raises(otk.OtkError) as e:
        otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"], d["old"],
                                    d["ref"], nl, otk.LossCfg(), dlogits=d["logits"])
    assert e.value.name == "OTK_ERR_INVALID_ARG"


def test_deterministic(otk, ctx):
    n, V = 400, 151936
    d, h = row_problem(n, V, seed=21)
    nl = torch.tensor([int(h["mask"].sum())], dtype=torch.int64, device="cuda")
    outs = [otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"], d["old"],
                                        d["ref"], nl, otk.LossCfg()) for _ in range(2)]
    ctx.check()
    assert torch.equal(outs[0]["dlogits"], outs[1]["dlogits"])
    assert torch.equal(outs[0]["stats"], outs[1]["stats"])


# ------------------------------------------------------------------------------------------ vocab sharding
@pytest.mark.parametrize("P,V,dtype", [(2, 151936, "bf16"), (4, 151936, "bf16"), (3, 3000, "f32")])
def test_vocab_sharded_equals_oracle(otk, ctx, P, V, dtype):
    n = 96
    d, h = row_problem(n, V, dtype=dtype, seed=P * 100 + 5)
    bounds = [V * k // P // 8 * 8 for k in range(P)] + [V]
    parts = []
    shards = []
    for k in range(P):
        a, b = bounds[k], bounds[k + 1]
        sl = d["logits"][:, a:b].contiguous()
        shards.append((a, b, sl))
        parts.append(otk.otk_row_partials(ctx, sl, d["targets"], a, V))
    partials = torch.stack(parts).contiguous()
    comb = otk.otk_logprob_entropy_combine(ctx, partials)
    ctx.check()
    want = O.logprob_entropy_fwd(h["wide"], h["targets"])
    tol = LOGP_TOL[dtype]
    assert np.max(np.abs(comb["logp"].cpu().numpy() - want["logp"])) < tol
    assert np.max(np.abs(comb["entropy"].cpu().numpy() - want["entropy"])) < tol
    N = int(h["mask"].sum())
    nl = torch.tensor([N], dtype=torch.int64, device="cuda")
    cfg = otk.LossCfg()
    wl = O.policy_loss_fwd_bwd(h["wide"], h["targets"], h["mask"], h["row_traj"], h["adv"], h["old"], h["ref"], N,
                               oracle_cfg(cfg))
    dl = torch.empty_like(d["logits"])
    losses = []
    for (a, b, sl) in shards:
        r = otk.otk_policy_loss_fwd_bwd_partials(ctx, sl, d["targets"], d["mask"], d["row_traj"], d["adv"], d["old"],
                                                 d["ref"], nl, cfg, a, V, partials)
        dl[:, a:b] = r["dlogits"]
        losses.append(otk.stats_dict(r["stats"])["loss"])
    ctx.check()
    assert len(set(losses)) == 1                       # identical on every shard
    rows = [j for j in range(n) if h["mask"][j]]
    dc = dcoef_rows(h, wl["logp"], oracle_cfg(cfg), N, True)
    assert check_dlogits_rows(dl, wl["dlogits"], wl["coef"], rows, dtype, V, dc, wide=h["wide"], targets=h["targets"],
                              h=h, cfg=oracle_cfg(cfg)) <= 1.0
    assert abs(losses[0] - wl["loss"]) <= 1e-4 * max(abs(wl["loss"]), 1e-3)


# ------------------------------------------------------------------------------------------ host entry point
def test_host_entry_point_matches_device(otk, ctx):
    n, V = 300, 151936
    d, h = row_problem(n, V, seed=31)
    N = int(h["mask"].sum())
    nl = torch.tensor([N], dtype=torch.int64, device="cuda")
    dev = otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"], d["old"],
                                      d["ref"], nl, otk.LossCfg())
    hostd = {k: v.cpu().pin_memory() for k, v in d.items()}
    dl_host = torch.empty(d["logits"].shape, dtype=d["logits"].dtype).pin_memory()
    st = otk.otk_policy_loss_fwd_bwd_host(ctx, hostd["logits"], hostd["targets"], hostd["mask"], hostd["row_traj"],
                                          hostd["adv"], hostd["old"], hostd["ref"], N, otk.LossCfg(), dlogits=dl_host,
                                          rows_per_chunk=64)
    ctx.check()
    assert torch.equal(dl_host, dev["dlogits"].cpu())
    want = otk.stats_dict(dev["stats"])
    assert abs(st["loss"] - want["loss"]) < 1e-12 and st["n_tokens"] == want["n_tokens"]


# ------------------------------------------------------------------------------------------ numerics edge cases
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_extreme_rows(otk, ctx, dtype):
    """-inf logits, late maxima 40-90 nats above everything seen before (the kernel's overflow re-reference
    path), very negative rows, and the uniform row, for the forward and the fused loss."""
    import torch as T
    V = 151936
    n = 12
    rng = np.random.default_rng(77)
    x = rng.normal(scale=2.0, size=(n, V))
    x[0, rng.integers(0, V, 5000)] = -np.inf                 # sprinkled -inf
    x[1, : V // 2] = -np.inf                                  # the whole first half (first CTA segment) -inf
    x[2, V - 5] = 90.0                                        # max in the last chunk, far above the reference
    x[3, 70000] = 60.0
    x[3, 150000] = 120.0                                      # two late jumps
    x[4] -= 1e4                                               # very negative, finite
    x[5] = 0.0                                                # uniform
    x[6, 3] = 50.0                                            # early dominant token
    t = T.from_numpy(x).to(T.bfloat16 if dtype == "bf16" else T.float32)
    wide = t.to(T.float64).numpy()
    y = rng.integers(0, V, n)
    y[1] = V - 7                                              # target in the finite half
    y[2] = V - 5
    y[3] = 3
    tg = T.from_numpy(y.astype(np.int32)).cuda()
    lg = t.cuda()
    f = otk.otk_logprob_entropy_fwd(ctx, lg, tg)
    want = O.logprob_entropy_fwd(wide, y)
    # fp32 outputs of magnitude ~100 carry ~4e-6 of rounding alone: the fp32 tolerance scales as
    # 1e-5 + 2^-22 |value|
    tol = LOGP_TOL[dtype] + (2.0 ** -22 if dtype == "f32" else 0.0) * np.abs(want["logp"])
    assert np.all(np.abs(f["logp"].cpu().numpy() - want["logp"]) < tol)
    assert np.all(np.abs(f["entropy"].cpu().numpy() - want["entropy"]) < LOGP_TOL[dtype])
    mask = np.ones(n, np.uint8)
    rt = np.zeros(n, np.int32)
    adv = np.array([0.7])
    old = (want["logp"] + rng.normal(scale=0.05, size=n)).astype(np.float32)
    ref = (want["logp"] + rng.normal(scale=0.1, size=n)).astype(np.float32)
    cfg = otk.LossCfg()
    out = otk.otk_policy_loss_fwd_bwd(ctx, lg, tg, T.from_numpy(mask).cuda(), T.from_numpy(rt).cuda(),
                                      T.from_numpy(adv).cuda(), T.from_numpy(old).cuda(), T.from_numpy(ref).cuda(),
                                      T.tensor([n], dtype=T.int64, device="cuda"), cfg)
    ctx.check()
    assert T.equal(out["logp"], f["logp"])                   # same reduction order as the forward
    ocfg = oracle_cfg(cfg)
    w = O.policy_loss_fwd_bwd(wide, y, mask, rt, adv, old.astype(np.float64), ref.astype(np.float64), n, ocfg)
    h = dict(old=old.astype(np.float64), ref=ref.astype(np.float64), adv=adv, row_traj=rt, mask=mask)
    dc = dcoef_rows(h, w["logp"], ocfg, n, True)
    assert check_dlogits_rows(out["dlogits"], w["dlogits"], w["coef"], list(range(n)), dtype, V, dc, wide=wide,
                              targets=y, h=h, cfg=ocfg) <= 1.0
    assert not bool(T.isnan(out["dlogits"].float()).any())


# ------------------------------------------------------------------------------------------ A4 variants
VARIANTS = {
    "dual": dict(dual_clip=3.0),
    "ent": dict(ent_coef=0.05),
    "seqmean": dict(reduction=1),
    "seqsum": dict(reduction=2),
    "sft": dict(sft=True),
    "all": dict(ent_coef=0.02, dual_clip=2.5, reduction=1),
}


@pytest.mark.parametrize("dtype,V,n", [("bf16", 151936, 96), ("f32", 1000, 128)])
@pytest.mark.parametrize("variant", list(VARIANTS))
def test_policy_loss_variants(otk, ctx, variant, dtype, V, n):
    """NEXT-4 variants of (4) vs the oracle (tests/test_oracle_pins.py pins them)."""
    kw = VARIANTS[variant]
    d, h = row_problem(n, V, dtype=dtype, seed=hash_seed(variant, V), force_clip=4, B=7)
    if kw.get("dual_clip"):   # negative advantages with ratios past the cap on half of the rows
        h["adv"][:] = -np.abs(h["adv"]) - 0.2
        d["adv"] = torch.from_numpy(h["adv"]).cuda()
    N = int(h["mask"].sum())
    tt = np.bincount(h["row_traj"][h["mask"] == 1], minlength=7).astype(np.int64)
    na = int(np.count_nonzero(tt))
    cfg = otk.LossCfg(**kw, traj_loss_tokens=torch.from_numpy(tt).cuda(),
                      n_active_traj=torch.tensor([na], dtype=torch.int64, device="cuda"))
    out = otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"], d["old"],
                                      d["ref"], torch.tensor([N], dtype=torch.int64, device="cuda"), cfg, vocab=V)
    ctx.check()
    ocfg = O.LossCfg(**{k: v for k, v in kw.items()})
    want = O.policy_loss_fwd_bwd(h["wide"], h["targets"], h["mask"], h["row_traj"], h["adv"], h["old"], h["ref"], N,
                                 ocfg, traj_tokens=tt, n_active=na)
    W = O.row_weights(h["mask"], h["row_traj"], ocfg.reduction, N, tt, na)
    rows = [j for j in range(n) if h["mask"][j]]
    dc = dcoef_rows(h, want["logp"], ocfg, N, True, W=W)
    worst = check_dlogits_rows(out["dlogits"], want["dlogits"], want["coef"], rows, dtype, V, dc, wide=h["wide"],
                               targets=h["targets"], h=h, cfg=ocfg, W=W,
                               ent=(ocfg.ent_coef, W) if ocfg.ent_coef else None)
    assert worst <= 1.0, worst
    st = otk.stats_dict(out["stats"])
    scale = max(abs(want["loss"]), float(np.sum(W * np.abs([O.row_loss_terms(want["logp"][j], h["old"][j],
                                                                             h["ref"][j], h["adv"][h["row_traj"][j]],
                                                                             ocfg)[0] - ocfg.ent_coef *
                                                            want["entropy"][j] if h["mask"][j] else 0.0
                                                            for j in range(n)]))))
    assert abs(st["loss"] - want["loss"]) <= 1e-4 * scale, (st["loss"], want["loss"])


def hash_seed(name, V):
    return sum(ord(c) for c in name) * 7 + V % 1000
