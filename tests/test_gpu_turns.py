"""Turn-level credit assignment (R31) on the GPU vs the oracle (-m gpu).

row_seg and seg_group bit-exact; seg_return 1e-12 relative (float64, Horner vs exact sum); segment
advantages 1e-6 abs (north_star (2)); the step's loss / dlogits with A read through row_seg within the
tolerances of tests/test_gpu_parity.py.
"""
import numpy as np
import pytest
import torch

from oracle import oracle_ref as O
from synth import CONFIGS, make_batch, make_logits, make_noise
from synth.trajectories import random_small_batch
from tests.gpu_common import check_dlogits_rows, dcoef_rows, oracle_cfg

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


def _batches():
    out = [(n, make_batch(n)) for n in CONFIGS]
    rng = np.random.default_rng(4)
    out.append(("random", random_small_batch(rng, 40, max_segs=9, max_len=7, num_groups=3)))
    return out


@pytest.mark.parametrize("gamma", [1.0, 0.9, 0.0])
@pytest.mark.parametrize("idx", range(len(CONFIGS) + 1))
def test_turn_returns_and_advantages(otk, ctx, idx, gamma):
    name, tb = _batches()[idx]
    db = otk.traj_batch_to_device(tb)
    S = tb.num_segments
    m = otk.otk_build_masks(ctx, db, row_seg=True)
    tr = otk.otk_turn_returns(ctx, db, S, torch.from_numpy(tb.group_id).cuda(),
                              torch.from_numpy(tb.turn_offsets).cuda(), torch.from_numpy(tb.turn_rewards).cuda(), gamma)
    a = otk.otk_group_advantages(ctx, tr["seg_group"], tb.num_groups, returns=tr["seg_return"], skip_ungrouped=True)
    ctx.check()
    om = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len, tb.terminated,
                       traj_agent=tb.traj_agent)
    assert np.array_equal(m["row_seg"].cpu().numpy(), om["row_seg"])
    G, grp = O.turn_returns(tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.turn_offsets, tb.turn_rewards,
                            tb.group_id, gamma, traj_agent=tb.traj_agent)
    assert np.array_equal(tr["seg_group"].cpu().numpy(), grp)
    g = tr["seg_return"].cpu().numpy()
    assert np.all(np.abs(g - G) <= 1e-12 * np.maximum(1.0, np.abs(G)))
    want = O.group_advantages(grp, G, tb.num_groups, skip_ungrouped=True)
    assert np.max(np.abs(a["adv"].cpu().numpy() - want["adv"])) < 1e-6
    assert np.array_equal(a["group_size"].cpu().numpy(), want["group_size"])


def test_turn_returns_errors(otk, ctx):
    tb = make_batch("tiny")
    db = otk.traj_batch_to_device(tb)
    args = (torch.from_numpy(tb.turn_offsets).cuda(), torch.from_numpy(tb.turn_rewards).cuda())
    with pytest.raises(otk.OtkError):
        otk.otk_turn_returns(ctx, db, tb.num_segments, torch.from_numpy(tb.group_id).cuda(), *args, gamma=1.5)
    gid = torch.full((tb.num_traj,), -1, dtype=torch.int32, device="cuda")
    otk.otk_turn_returns(ctx, db, tb.num_segments, gid, *args, gamma=1.0)
    with pytest.raises(otk.OtkError) as e:
        ctx.check()
    assert e.value.status == 10          # OTK_ERR_GROUP_RANGE
    otk.otk_turn_returns(ctx, db, tb.num_segments + 1, torch.from_numpy(tb.group_id).cuda(), *args, gamma=1.0,
                         out=dict(seg_return=torch.empty(tb.num_segments + 1, dtype=torch.float64, device="cuda"),
                                  seg_group=torch.empty(tb.num_segments + 1, dtype=torch.int32, device="cuda")))
    with pytest.raises(otk.OtkError) as e:
        ctx.check()
    assert e.value.status == 7           # OTK_ERR_BAD_TRAJECTORY: seg_offsets[B] != num_segments


@pytest.mark.parametrize("dtype,V,gamma", [("f32", 1024, 0.9), ("bf16", 3000, 1.0)])
def test_turn_level_step(otk, ctx, dtype, V, gamma):
    """The whole step with credit="turn" against the oracle chain (O1 row_seg, O6, O2, O4 with adv_index)."""
    from paper_2601_07376_b200.step import MicroBatch, PolicyLossStep
    rng = np.random.default_rng(17)
    tb = random_small_batch(rng, 12, max_segs=7, max_len=30, num_groups=3)
    N = tb.num_rows
    cfg = otk.LossCfg(kl_beta=0.04)
    db = otk.traj_batch_to_device(tb)
    st = PolicyLossStep(ctx, db, torch.from_numpy(tb.group_id).cuda(), tb.num_groups,
                        torch.from_numpy(tb.turn_offsets).cuda(), torch.from_numpy(tb.turn_rewards).cuda(), V, cfg,
                        credit="turn", gamma=gamma)
    logits, targets = make_logits(N, V, dtype=dtype, seed=23, device="cpu")
    wide = logits.double().numpy()
    y = targets.numpy()
    olp = np.array([O.row_forward(wide[j], int(y[j]))[0] for j in range(N)])
    old = (olp + make_noise(N, 0.05, 5).double().numpy()).astype(np.float32)
    ref = (olp + make_noise(N, 0.1, 6).double().numpy()).astype(np.float32)
    dl = torch.empty_like(logits, device="cuda")
    st.run([MicroBatch(0, N // 2, logits[:N // 2].cuda(), targets[:N // 2].cuda(),
                       torch.from_numpy(old[:N // 2]).cuda(), torch.from_numpy(ref[:N // 2]).cuda(), dl[:N // 2]),
            MicroBatch(N // 2, N, logits[N // 2:].cuda(), targets[N // 2:].cuda(),
                       torch.from_numpy(old[N // 2:]).cuda(), torch.from_numpy(ref[N // 2:]).cuda(), dl[N // 2:])])
    ctx.check()
    om = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len, tb.terminated)
    G, grp = O.turn_returns(tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.turn_offsets, tb.turn_rewards,
                            tb.group_id, gamma)
    adv_seg, _ = O.turn_level_advantages(om["row_seg"], G, grp, tb.num_groups)
    assert np.max(np.abs(st.adv_out["adv"].cpu().numpy() - adv_seg)) < 1e-6
    ocfg = oracle_cfg(cfg)
    n_loss = om["n_loss"]
    want = O.policy_loss_fwd_bwd(wide, y, om["loss_mask"], om["row_traj"], adv_seg, old.astype(np.float64),
                                 ref.astype(np.float64), n_loss, ocfg, adv_index=om["row_seg"])
    stats = otk.stats_dict(st.stats)
    terms = [abs(O.row_loss_terms(want["logp"][j], float(old[j]), float(ref[j]), adv_seg[om["row_seg"][j]],
                                  ocfg)[0]) for j in range(N) if om["loss_mask"][j]]
    assert abs(stats["loss"] - want["loss"]) <= 1e-4 * max(abs(want["loss"]), sum(terms) / max(n_loss, 1))
    assert stats["n_tokens"] == n_loss
    # dlogits: the oracle's, with per-row advantage taken through row_seg
    h = dict(old=old.astype(np.float64), ref=ref.astype(np.float64), adv=adv_seg, row_traj=om["row_seg"],
             mask=om["loss_mask"])
    rows = [j for j in range(N) if om["loss_mask"][j]]
    dc = dcoef_rows(h, want["logp"], ocfg, n_loss, True)
    assert check_dlogits_rows(dl, want["dlogits"], want["coef"], rows, dtype, V, dc, wide=wide, targets=y, h=h,
                              cfg=ocfg) <= 1.0
    assert bool((dl[torch.from_numpy(om["loss_mask"] == 0).cuda()] == 0).all())
