"""Full-size parity (-m gpu): BASELINE configs at V = 151936 in the launch configuration bench.py times
(65,536-row micro-batches of the fused loss), every row against the C float64 oracle (oracle/parity.py).
Inputs come from the seeded generator and the oracle only (old / ref = oracle logp + noise)."""
import math

import numpy as np
import pytest
import torch

from oracle import oracle_ref as O
from synth import CONFIGS, make_batch, make_logits, make_noise
from tests.gpu_common import LOGP_TOL, oracle_cfg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def otk():
    import paper_2601_07376_b200 as m
    return m


@pytest.mark.parametrize("name", ["math", "game", "marl"])
def test_fullsize_microbatch(otk, name):
    """EVERY row of one 65,536-row micro-batch (the bench's launch configuration) against the C float64
    oracle: (3) logp / entropy, then (4) with old / ref = oracle logp + noise (nothing derived from the CUDA
    path): logp, entropy, each dlogits element and row L1 (oracle/parity.py tolerances), masked rows exactly 0,
    the micro-batch loss and the clipped / token counts."""
    from oracle import parity as P
    from paper_2601_07376_b200.step import PolicyLossStep
    cfgw = CONFIGS[name]
    V, M, dev = cfgw.V, 65536, "cuda"
    ctx = otk.Context(0)
    tb = make_batch(name)
    db = otk.traj_batch_to_device(tb)
    cfg = otk.LossCfg(kl_beta=cfgw.kl_beta)
    step = PolicyLossStep(ctx, db, torch.from_numpy(tb.group_id).to(dev), tb.num_groups,
                          torch.from_numpy(tb.turn_offsets).to(dev), torch.from_numpy(tb.turn_rewards).to(dev), V, cfg)
    adv = step.masks_and_advantages()
    ctx.check()
    om = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len, tb.terminated,
                       traj_agent=tb.traj_agent)
    assert np.array_equal(step.masks["loss_mask"].cpu().numpy(), om["loss_mask"])     # all 2^20 rows
    assert np.array_equal(step.masks["row_traj"].cpu().numpy(), om["row_traj"])
    assert int(step.masks["n_loss"].item()) == om["n_loss"]
    oadv = O.group_advantages(tb.group_id, O.episode_returns(tb.turn_offsets, tb.turn_rewards), tb.num_groups)["adv"]
    assert np.max(np.abs(adv.cpu().numpy() - oadv)) < 1e-6

    logits, targets = make_logits(M, V, dtype="bf16", seed=cfgw.seed * 100, device=dev, rows_per_chunk=4096)
    mask = om["loss_mask"][:M]
    rt = om["row_traj"][:M]
    # (3) on every row
    fwd = otk.otk_logprob_entropy_fwd(ctx, logits, targets)
    ctx.check()
    of = P.oracle_logp(logits, targets, V, "bf16")
    assert float(np.max(np.abs(fwd["logp"].double().cpu().numpy() - of["logp"]))) < LOGP_TOL["bf16"]
    assert float(np.max(np.abs(fwd["entropy"].double().cpu().numpy() - of["entropy"]))) < LOGP_TOL["bf16"]
    del fwd
    # (4) on every row, old / ref from the oracle's logp
    old = (of["logp"] + make_noise(M, 0.05, 11).double().numpy()).astype(np.float32)
    ref = (of["logp"] + make_noise(M, 0.1, 12).double().numpy()).astype(np.float32)
    dl = torch.empty_like(logits)
    out = otk.otk_policy_loss_fwd_bwd(ctx, logits, targets, step.masks["loss_mask"][:M], step.masks["row_traj"][:M],
                                      adv, torch.from_numpy(old).to(dev),
                                      torch.from_numpy(ref).to(dev) if cfgw.kl_beta else None,
                                      step.masks["n_loss"], cfg, dlogits=dl)
    ctx.check()
    st = otk.stats_dict(out["stats"])
    par = P.microbatch_parity(logits, targets, mask, rt, oadv, old, ref if cfgw.kl_beta else None, om["n_loss"],
                              oracle_cfg(cfg), "bf16", V, out["logp"], out["entropy"], dl, st)
    print(name, par)
    assert P.parity_ok(par), par
    assert par["trainable"] == int(mask.sum()) and par["rows"] == M
    ctx.close()


@pytest.mark.parametrize("P", [2, 4])
def test_fullsize_vpf_microbatch(otk, P):
    """K4-VPF at the bench's full size (one 65,536-row math micro-batch, V = 151936, P ranks emulated in one
    grouped launch, as perf_vpf.py times it): sampled rows against the oracle, and every row against the
    unsharded kernel (logp 1e-5, dlogits within bf16 rounding, identical loss stats up to fp64 summation)."""
    cfgw = CONFIGS["math"]
    V, M, dev = cfgw.V, 65536, "cuda"
    tb = make_batch("math")
    om = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len, tb.terminated,
                       traj_agent=tb.traj_agent)
    logits, targets = make_logits(M, V, dtype="bf16", seed=cfgw.seed * 100 + 1, device=dev, rows_per_chunk=4096)
    mask = om["loss_mask"][:M]
    rt = om["row_traj"][:M]
    oadv = O.group_advantages(tb.group_id, O.episode_returns(tb.turn_offsets, tb.turn_rewards), tb.num_groups)["adv"]
    tr = np.flatnonzero(mask)
    sample = sorted(set(tr[np.linspace(0, len(tr) - 1, 8).astype(int)].tolist()))
    y = targets.cpu().numpy()
    wide = {j: logits[j].double().cpu().numpy() for j in sample}
    base = np.zeros(M)
    for j in sample:
        base[j] = O.row_forward(wide[j], int(y[j]))[0]
    old = torch.from_numpy(base).float().to(dev) + make_noise(M, 0.05, 11, device=dev)
    ref = torch.from_numpy(base).float().to(dev) + make_noise(M, 0.1, 12, device=dev)
    d = dict(logits=logits, targets=targets, mask=torch.from_numpy(mask).to(dev),
             row_traj=torch.from_numpy(rt).to(dev), adv=torch.from_numpy(oadv).to(dev), old=old.contiguous(),
             ref=ref.contiguous())
    N = int(mask.sum())
    nl = torch.tensor([N], dtype=torch.int64, device=dev)
    cfg = otk.LossCfg(kl_beta=cfgw.kl_beta)
    ctxs = [otk.Context(0) for _ in range(P)]
    xchgs = otk.VpfExchange.local_group(ctxs, M)
    b = [V * k // P // 8 * 8 for k in range(P)] + [V]
    dl = torch.empty_like(logits)
    torch.cuda.synchronize()
    res = otk.otk_policy_loss_fwd_bwd_vpf_group(ctxs, [logits[:, b[k]:b[k + 1]] for k in range(P)], targets,
                                                d["mask"], d["row_traj"], d["adv"], d["old"], d["ref"], nl, cfg,
                                                b[:P], V, xchgs, dlogits=[dl[:, b[k]:b[k + 1]] for k in range(P)])
    torch.cuda.synchronize()
    for c in ctxs:
        c.check()
    full = otk.otk_policy_loss_fwd_bwd(ctxs[0], logits, targets, d["mask"], d["row_traj"], d["adv"], d["old"],
                                       d["ref"], nl, cfg)
    ctxs[0].check()
    for k in range(1, P):
        assert torch.equal(res[k]["logp"], res[0]["logp"]) and torch.equal(res[k]["stats"], res[0]["stats"])
    assert float((res[0]["logp"] - full["logp"]).abs().max()) < 1e-5
    sv, sf = otk.stats_dict(res[0]["stats"]), otk.stats_dict(full["stats"])
    assert abs(sv["loss"] - sf["loss"]) <= 1e-6 * max(abs(sf["loss"]), 1e-3) and sv["n_tokens"] == sf["n_tokens"] == N
    for r0 in range(0, M, 8192):   # every row vs the unsharded kernel, in blocks (memory)
        a = dl[r0:r0 + 8192].float()
        f = full["dlogits"][r0:r0 + 8192].float()
        assert float(((a - f).abs() / (f.abs() * 2 ** -6 + 1e-9)).max()) <= 1.0
    ocfg = oracle_cfg(cfg)
    for j in sample:
        lp = O.row_forward(wide[j], int(y[j]))[0]
        assert abs(float(res[0]["logp"][j]) - lp) < LOGP_TOL["bf16"]
    del full
    for x in xchgs:
        x.close()
