"""Degenerate and empty inputs through the C ABI (-m gpu): zero rows, every row masked (N_loss = 0), a
one-token vocabulary, empty trajectories — each against the oracle or the closed form."""
import math

import numpy as np
import pytest
import torch

from oracle import oracle_ref as O

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


def test_zero_rows_every_entry_point(otk, ctx):
    V = 4096
    lg = torch.empty((0, V), dtype=torch.bfloat16, device="cuda")
    tg = torch.empty(0, dtype=torch.int32, device="cuda")
    assert otk.otk_logprob_entropy_fwd(ctx, lg, tg)["logp"].numel() == 0
    assert otk.otk_sample_tokens(ctx, lg, torch.empty(0, device="cuda"))["tokens"].numel() == 0
    assert otk.otk_row_partials(ctx, lg, tg, 0, V).numel() == 0
    h = torch.empty((0, 64), dtype=torch.bfloat16, device="cuda")
    w = torch.zeros((V, 64), dtype=torch.bfloat16, device="cuda")
    assert otk.otk_lmhead_logprob_fwd(ctx, h, w, tg)["logp"].numel() == 0
    # the loss over zero rows still writes the (zero) stats when not accumulating, and keeps them otherwise
    stats = torch.full((5,), 3.0, dtype=torch.float64, device="cuda")
    e = torch.empty(0, device="cuda")
    args = (lg, tg, torch.empty(0, dtype=torch.uint8, device="cuda"), torch.empty(0, dtype=torch.int32, device="cuda"),
            torch.zeros(1, dtype=torch.float64, device="cuda"), e, e, torch.zeros(1, dtype=torch.int64, device="cuda"))
    otk.otk_policy_loss_fwd_bwd(ctx, *args, otk.LossCfg(), stats=stats, accumulate=True)
    assert stats.tolist() == [3.0] * 5
    otk.otk_policy_loss_fwd_bwd(ctx, *args, otk.LossCfg(), stats=stats, accumulate=False)
    assert stats.tolist() == [0.0] * 5
    ctx.check()


def test_all_rows_masked(otk, ctx):
    """N_loss = 0 (R17): loss 0, every dlogits row 0, no trainable tokens."""
    from synth import make_logits
    n, V = 64, 4096
    lg, tg = make_logits(n, V, dtype="bf16", seed=2, device="cuda")
    dl = torch.full_like(lg, 5.0)
    out = otk.otk_policy_loss_fwd_bwd(ctx, lg, tg, torch.zeros(n, dtype=torch.uint8, device="cuda"),
                                      torch.zeros(n, dtype=torch.int32, device="cuda"),
                                      torch.ones(1, dtype=torch.float64, device="cuda"),
                                      torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda"),
                                      torch.zeros(1, dtype=torch.int64, device="cuda"), otk.LossCfg(), dlogits=dl)
    ctx.check()
    st = otk.stats_dict(out["stats"])
    assert st["loss"] == 0.0 and st["n_tokens"] == 0.0
    assert bool((dl == 0).all())


def test_one_token_vocabulary(otk, ctx):
    """V = 1: the only token has probability 1 — logp = 0 and entropy = 0 (to fp32 rounding of s*x), the sampler
    returns it, and the gradient row is coef * (1 - 1) = 0."""
    n = 16
    lg = torch.randn((n, 8), device="cuda").to(torch.bfloat16)     # ld = 8 (16-byte rows), vocab = 1
    tg = torch.zeros(n, dtype=torch.int32, device="cuda")
    f = otk.otk_logprob_entropy_fwd(ctx, lg, tg, vocab=1)
    assert float(f["logp"].abs().max()) < 1e-6 and float(f["entropy"].abs().max()) < 1e-6
    s = otk.otk_sample_tokens(ctx, lg, torch.rand(n, device="cuda"), vocab=1)
    assert int(s["tokens"].max()) == 0 and float(s["logp"].abs().max()) < 1e-6
    dl = torch.full_like(lg, 9.0)
    otk.otk_policy_loss_fwd_bwd(ctx, lg, tg, torch.ones(n, dtype=torch.uint8, device="cuda"),
                                torch.zeros(n, dtype=torch.int32, device="cuda"),
                                torch.ones(1, dtype=torch.float64, device="cuda"), torch.zeros(n, device="cuda"),
                                torch.zeros(n, device="cuda"), torch.full((1,), n, dtype=torch.int64, device="cuda"),
                                otk.LossCfg(), vocab=1, dlogits=dl)
    ctx.check()
    # coef * expm1(logp) with logp ~ 1e-8 of rounding: zero within the dlogits tolerance (1e-5 |coef|)
    assert float(dl[:, 0].float().abs().max()) < 1e-6 and bool((dl[:, 1:] == 9.0).all())   # columns >= vocab untouched


def test_empty_trajectories_in_batch(otk, ctx):
    """Trajectories with no segments and no rows sit between normal ones: masks, counts, returns exact."""
    from synth.trajectories import _pack
    C, A, Ob = O.CONTEXT, O.ACTION, O.OBSERVATION
    tb = _pack([[(C, -1, 3), (A, 0, 4)], [], [(C, -1, 2), (A, 0, 2), (Ob, -1, 1)], []],
               [[1.0], [], [0.5], [2.0]], [0, 0, 1, 1], 2)
    db = otk.traj_batch_to_device(tb)
    m = otk.otk_build_masks(ctx, db, row_seg=True)
    ctx.check()
    om = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len, tb.terminated)
    for k in ("loss_mask", "row_traj", "row_seg", "traj_loss_tokens"):
        assert np.array_equal(m[k].cpu().numpy(), om[k]), k
    assert int(m["n_active_traj"].item()) == 2
    a = otk.otk_group_advantages(ctx, torch.from_numpy(tb.group_id).cuda(), 2,
                                 turn_offsets=torch.from_numpy(tb.turn_offsets).cuda(),
                                 turn_rewards=torch.from_numpy(tb.turn_rewards).cuda())
    want = O.group_advantages(tb.group_id, O.episode_returns(tb.turn_offsets, tb.turn_rewards), 2)["adv"]
    assert np.max(np.abs(a["adv"].cpu().numpy() - want)) < 1e-6


def test_binding_rejects_malformed_arrays(otk, ctx):
    """The binding checks dtype / size / device of every per-row array before the C call (a short array
    would otherwise be read out of bounds by the kernels)."""
    from synth import make_logits
    n, V = 32, 1024
    lg, tg = make_logits(n, V, dtype="bf16", seed=3, device="cuda")
    with pytest.raises(ValueError):
        otk.otk_logprob_entropy_fwd(ctx, lg, tg.long())                       # int64 targets
    with pytest.raises(ValueError):
        otk.otk_logprob_entropy_fwd(ctx, lg, tg[:-1].contiguous())            # short targets
    args = dict(loss_mask=torch.ones(n, dtype=torch.uint8, device="cuda"),
                row_traj=torch.zeros(n, dtype=torch.int32, device="cuda"),
                adv=torch.ones(1, dtype=torch.float64, device="cuda"),
                old_logp=torch.zeros(n - 1, device="cuda"), ref_logp=None,
                n_loss=torch.full((1,), n, dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError):
        otk.otk_policy_loss_fwd_bwd(ctx, lg, tg, cfg=otk.LossCfg(kl_beta=0.0), **args)   # short old_logp
    with pytest.raises(ValueError):
        otk.otk_sample_tokens(ctx, lg, torch.rand(n, device="cuda", dtype=torch.float64))   # float64 uniforms


@pytest.mark.parametrize("dtype,V", [("bf16", 151936), ("f32", 151936), ("bf16", 262144), ("bf16", 33001)])
def test_targets_on_segment_boundaries(otk, ctx, dtype, V):
    """Targets on the first / last column of every CTA's column segment (row clusters split the vocabulary):
    logp and the target column of dlogits (coef * (p_y - 1)) against the oracle."""
    from synth import make_logits, make_noise
    seg = None
    for c in range(1, 9):      # the row kernel's split: fewest CTAs whose segment fits 18 x 12 KB
        s = ((V + c - 1) // c + 7) // 8 * 8
        if s * (2 if dtype == "bf16" else 4) <= 18 * 12288 and (c - 1) * s < V:
            seg = s
            break
    cols = sorted({0, V - 1} | {k * seg for k in range(1, (V + seg - 1) // seg)} |
                  {k * seg - 1 for k in range(1, (V + seg - 1) // seg)} | {7, 8, V - 8})
    n = len(cols)
    ld = -(-V // 8) * 8                      # 16-byte rows
    lg, _ = make_logits(n, V, ld=ld, dtype=dtype, seed=V % 1000 + 3, device="cpu")
    tg = torch.tensor(cols, dtype=torch.int32)
    wide = lg.double().numpy()[:, :V]
    olp = np.array([O.row_forward(wide[j], cols[j])[0] for j in range(n)])
    f = otk.otk_logprob_entropy_fwd(ctx, lg.cuda(), tg.cuda(), vocab=V)
    ctx.check()
    assert np.max(np.abs(f["logp"].cpu().numpy() - olp)) < (2e-3 if dtype == "bf16" else 1e-5)
    old = (olp + make_noise(n, 0.05, 1).double().numpy()).astype(np.float32)
    adv = torch.tensor([0.7], dtype=torch.float64)
    out = otk.otk_policy_loss_fwd_bwd(ctx, lg.cuda(), tg.cuda(), torch.ones(n, dtype=torch.uint8).cuda(),
                                      torch.zeros(n, dtype=torch.int32).cuda(), adv.cuda(),
                                      torch.from_numpy(old).cuda(), None,
                                      torch.tensor([n], dtype=torch.int64).cuda(), otk.LossCfg(kl_beta=0.0), vocab=V)
    ctx.check()
    want = O.policy_loss_fwd_bwd(wide, np.array(cols), np.ones(n, np.uint8), np.zeros(n, np.int32), adv.numpy(),
                                 old.astype(np.float64), None, n, O.LossCfg(kl_beta=0.0))
    from tests.gpu_common import check_dlogits_rows, dcoef_rows
    h = dict(old=old.astype(np.float64), ref=np.zeros(n), adv=adv.numpy(), row_traj=np.zeros(n, np.int32),
             mask=np.ones(n, np.uint8))
    ocfg = O.LossCfg(kl_beta=0.0)
    dc = dcoef_rows(h, want["logp"], ocfg, n, 0.0)
    assert check_dlogits_rows(out["dlogits"], want["dlogits"], want["coef"], list(range(n)), dtype, V, dc, wide=wide,
                              targets=np.array(cols), h=h, cfg=ocfg) <= 1.0


def test_adv_index_out_of_range_is_a_data_error(otk, ctx):
    """a row whose row_traj (or adv_index) points outside adv is OTK_ERR_GROUP_RANGE, that row is treated
    as loss-masked (zero gradient, logp 0, not counted), and every other row equals a call with valid indices."""
    from tests.gpu_common import row_problem
    n, V = 64, 4096
    d, h = row_problem(n, V, seed=12, mask_p=1.0, B=4)
    nl = torch.tensor([n], dtype=torch.int64, device="cuda")
    good = otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"], d["old"],
                                       d["ref"], nl, otk.LossCfg())
    ctx.check()
    for field in ("row_traj", "adv_index"):
        rt = d["row_traj"].clone()
        cfg = otk.LossCfg()
        if field == "row_traj":
            rt[9] = 4                                   # adv has 4 entries
        else:
            ai = d["row_traj"].clone()
            ai[9] = -1
            cfg = otk.LossCfg(adv_index=ai)
        bad = otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], rt, d["adv"], d["old"], d["ref"],
                                          nl, cfg)
        with pytest.raises(otk.OtkError, match="OTK_ERR_GROUP_RANGE"):
            ctx.check()
        assert bool((bad["dlogits"][9] == 0).all()) and float(bad["logp"][9]) == 0.0
        keep = torch.ones(n, dtype=torch.bool, device="cuda")
        keep[9] = False
        assert torch.equal(bad["dlogits"][keep], good["dlogits"][keep])
        assert torch.equal(bad["logp"][keep], good["logp"][keep])
        assert otk.stats_dict(bad["stats"])["n_tokens"] == n - 1


def test_host_entry_point_writes_vocab_columns_and_trainable_rows_only(otk, ctx):
    """the host-buffer entry point writes only columns [0, vocab) of dlogits_host, and with
    zero_masked_rows = 0 only the trainable rows (masked rows keep the caller's bytes)."""
    from tests.gpu_common import row_problem
    n, V, ld = 300, 1000, 1008
    d, h = row_problem(n, V, ld=ld, seed=14)
    N = int(h["mask"].sum())
    hostd = {k: v.cpu().pin_memory() for k, v in d.items()}
    for zero in (True, False):
        cfg = otk.LossCfg(zero_masked_rows=zero)
        dl_host = torch.full(d["logits"].shape, 7.0, dtype=d["logits"].dtype).pin_memory()
        st = otk.otk_policy_loss_fwd_bwd_host(ctx, hostd["logits"], hostd["targets"], hostd["mask"], hostd["row_traj"],
                                              hostd["adv"], hostd["old"], hostd["ref"], N, cfg, vocab=V,
                                              dlogits=dl_host, rows_per_chunk=64)
        dev = otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"],
                                          d["old"], d["ref"], torch.tensor([N], dtype=torch.int64, device="cuda"),
                                          otk.LossCfg(), vocab=V)
        ctx.check()
        assert bool((dl_host[:, V:] == 7.0).all())
        m = torch.from_numpy(h["mask"]).bool()
        assert torch.equal(dl_host[m, :V], dev["dlogits"][:, :V].cpu()[m])
        assert bool((dl_host[~m, :V] == (0.0 if zero else 7.0)).all())
        assert st["n_tokens"] == N
