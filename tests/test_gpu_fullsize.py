"""Full-size parity (-m gpu): BASELINE configs at V = 151936 in the launch configuration bench.py times
(65,536-row micro-batches of the fused loss), checked on sampled rows the oracle computes one by one,
plus properties over every row. Inputs of every sampled row come from the seeded generator and the
oracle only (old/ref of sampled rows = oracle logp + noise)."""
import math

import numpy as np
import pytest
import torch

from oracle import oracle_ref as O
from synth import CONFIGS, make_batch, make_logits, make_noise
from tests.gpu_common import LOGP_TOL, check_dlogits_rows, dcoef_rows, oracle_cfg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def otk():
    import paper_2601_07376_b200 as m
    return m


@pytest.mark.parametrize("name,rows", [("math", 65536), ("game", 32768), ("marl", 32768)])
def test_fullsize_microbatch(otk, name, rows):
    from paper_2601_07376_b200.step import MicroBatch, PolicyLossStep
    cfgw = CONFIGS[name]
    V = cfgw.V
    ctx = otk.Context(0)
    tb = make_batch(name)
    db = otk.traj_batch_to_device(tb)
    dev = "cuda"
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

    # one micro-batch of logits (the bench's generator), sampled rows, and their oracle inputs
    M = rows
    logits, targets = make_logits(M, V, dtype="bf16", seed=cfgw.seed * 100, device=dev, rows_per_chunk=4096)
    mask = om["loss_mask"][:M]
    tr = np.flatnonzero(mask)
    ms = np.flatnonzero(mask == 0)
    sample = sorted(set(tr[np.linspace(0, len(tr) - 1, 12).astype(int)].tolist()
                        + ms[np.linspace(0, len(ms) - 1, 4).astype(int)].tolist() + [M - 1]))
    y = targets.cpu().numpy()
    wide = {j: logits[j].double().cpu().numpy() for j in sample}
    olp = {j: O.row_forward(wide[j], int(y[j]))[0] for j in sample}
    fwd = otk.otk_logprob_entropy_fwd(ctx, logits, targets)                            # (3) on every row
    for j in sample:
        lp, H, _, _ = O.row_forward(wide[j], int(y[j]))
        assert abs(float(fwd["logp"][j]) - lp) < LOGP_TOL["bf16"] and abs(float(fwd["entropy"][j]) - H) < LOGP_TOL["bf16"]
    n_old = make_noise(M, 0.05, 11, device=dev)
    n_ref = make_noise(M, 0.1, 12, device=dev)
    old = fwd["logp"] + n_old
    ref = fwd["logp"] + n_ref
    sidx = torch.tensor(sample, device=dev)
    olp_t = torch.tensor([olp[j] for j in sample], dtype=torch.float64)
    old[sidx] = (olp_t + n_old[sidx].double().cpu()).float().to(dev)
    ref[sidx] = (olp_t + n_ref[sidx].double().cpu()).float().to(dev)
    dl = torch.empty_like(logits)
    out = otk.otk_policy_loss_fwd_bwd(ctx, logits, targets, step.masks["loss_mask"][:M], step.masks["row_traj"][:M],
                                      adv, old, ref if cfgw.kl_beta else None, step.masks["n_loss"], cfg,
                                      dlogits=dl)
    ctx.check()
    ocfg = oracle_cfg(cfg)
    N = om["n_loss"]
    old_h, ref_h = old.double().cpu().numpy(), ref.double().cpu().numpy()
    want = O.policy_loss_fwd_bwd(lambda j: wide[j], y, om["loss_mask"], om["row_traj"], oadv, old_h,
                                 ref_h if cfgw.kl_beta else None, N, ocfg, rows=sample)
    h = dict(old=old_h, ref=ref_h, adv=oadv, row_traj=om["row_traj"], mask=np.zeros(M, np.uint8))
    h["mask"][[j for j in sample if mask[j]]] = 1
    dc = dcoef_rows(h, {j: want["logp"][j] for j in sample}, ocfg, N, cfgw.kl_beta)
    trows = [j for j in sample if mask[j]]
    assert check_dlogits_rows(dl, want["dlogits"], want["coef"], trows, "bf16", V, dc) <= 1.0
    for j in sample:
        assert abs(float(out["logp"][j]) - want["logp"][j]) < LOGP_TOL["bf16"]
        if not mask[j]:
            assert bool((dl[j] == 0).all())
    # properties over every row of the micro-batch
    m_t = step.masks["loss_mask"][:M].bool()
    assert bool((dl[~m_t] == 0).all())                                   # mask soundness
    st = otk.stats_dict(out["stats"])
    assert st["n_tokens"] == int(mask.sum())
    # loss = sum_j m_j L_j / N restated in float64 from the kernel's own per-row logp (property at any size)
    lp = out["logp"].double().cpu().numpy()[mask == 1]
    A = oadv[om["row_traj"][:M][mask == 1]]
    C = 20.0
    d = np.clip(lp - old_h[mask == 1], -C, C)
    r = np.exp(d)
    pg = np.maximum(-A * r, -A * np.clip(r, 0.8, 1.2))
    kl = 0.0
    if cfgw.kl_beta:
        dd = np.clip(ref_h[mask == 1] - lp, -C, C)
        kl = np.expm1(dd) - dd
    L = pg + cfgw.kl_beta * kl
    want_loss = math.fsum(L) / N
    assert abs(st["loss"] - want_loss) <= 1e-4 * max(abs(want_loss), np.abs(L).sum() / N)
    ctx.close()


@pytest.mark.parametrize("P", [2, 4])
def test_fullsize_vpf_microbatch(otk, P):
    """K4-VPF at the bench's full size (one 65,536-row math micro-batch, V = 151936, P ranks co-scheduled on the
    GPU in the perf_vpf.py launch configuration): sampled rows against the oracle, and every row against the
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
    streams = [torch.cuda.Stream() for _ in range(P)]
    xchgs = otk.VpfExchange.local_group(ctxs, M, max_ctas=148 // P)
    b = [V * k // P // 8 * 8 for k in range(P)] + [V]
    dl = torch.empty_like(logits)
    torch.cuda.synchronize()
    res = []
    for k in range(P):
        res.append(otk.otk_policy_loss_fwd_bwd_vpf(ctxs[k], logits[:, b[k]:b[k + 1]], targets, d["mask"],
                                                   d["row_traj"], d["adv"], d["old"], d["ref"], nl, cfg, b[k], V,
                                                   xchgs[k], dlogits=dl[:, b[k]:b[k + 1]], stream=streams[k]))
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
