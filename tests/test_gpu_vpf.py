"""K4-VPF (otk_policy_loss_fwd_bwd_vpf): the vocab-sharded fused loss with the row-partial exchange inside the
kernel (-m gpu). P ranks are emulated on the one GPU of the box in ONE cooperative launch
(otk_policy_loss_fwd_bwd_vpf_group): each rank its own ctx, column shard (a column slice of one [N, V] buffer)
and 148 // P CTAs, exchanging through plain device buffers instead of IPC-mapped peer buffers (the kernel code
and the per-rank parameters are the multi-GPU ones). Every rank's CTAs are resident together, so the test never
depends on separate launches being co-scheduled (which CUDA does not promise, and a profiler breaks).

Checks: logp / entropy bitwise equal on every rank AND to the gathered path (otk_row_partials -> stack ->
otk_policy_loss_fwd_bwd_partials: same partials, same rank-order combine); loss stats identical on every rank;
everything within the north_star tolerances of the float64 oracle; repeated calls (epoch parity) and CUDA-graph
replays (the epoch lives on the device) reproduce the same bits; a data error on one row leaves every other row
exact; a missing peer ends in OTK_ERR_PEER_TIMEOUT, not a hang."""
import numpy as np
import pytest
import torch

from oracle import oracle_ref as O
from tests.gpu_common import LOGP_TOL, check_dlogits_rows, dcoef_rows, oracle_cfg, row_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def otk():
    import paper_2601_07376_b200 as m
    return m


def _bounds(V, P):
    return [V * k // P // 8 * 8 for k in range(P)] + [V]


def _run_vpf(otk, ctxs, xchgs, streams, d, V, nl, cfg, dl, calls=1):
    """`calls` consecutive grouped launches (all P ranks in one launch each); `streams` is unused (kept for the
    call sites' symmetry with the per-rank form)."""
    P = len(ctxs)
    b = _bounds(V, P)
    torch.cuda.synchronize()
    outs = []
    for _ in range(calls):
        outs.append(otk.otk_policy_loss_fwd_bwd_vpf_group(
            ctxs, [d["logits"][:, b[k]:b[k + 1]] for k in range(P)], d["targets"], d["mask"], d["row_traj"],
            d["adv"], d["old"], d["ref"], nl, cfg, b[:P], V, xchgs, dlogits=[dl[:, b[k]:b[k + 1]] for k in range(P)]))
        torch.cuda.synchronize()
    for c in ctxs:
        c.check()
    return outs


@pytest.mark.parametrize("P,V,dtype,n", [(2, 151936, "bf16", 160), (4, 151936, "bf16", 96), (8, 151936, "bf16", 64),
                                         (2, 151936, "f32", 40), (3, 3000, "f32", 50)])
def test_vpf_equals_gathered_path_and_oracle(otk, P, V, dtype, n):
    d, h = row_problem(n, V, dtype=dtype, seed=P * 1000 + n)
    ctxs = [otk.Context(0) for _ in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    xchgs = otk.VpfExchange.local_group(ctxs, n, max_ctas=148 // P)
    N = int(h["mask"].sum())
    nl = torch.tensor([N], dtype=torch.int64, device="cuda")
    cfg = otk.LossCfg()
    dl = torch.full_like(d["logits"], 7.0)
    outs = _run_vpf(otk, ctxs, xchgs, streams, d, V, nl, cfg, dl, calls=3)
    res = outs[-1]
    # identical on every rank, and across the three calls (epochs 1, 2, 3: both buffer parities reused)
    for k in range(1, P):
        assert torch.equal(res[k]["logp"], res[0]["logp"]) and torch.equal(res[k]["entropy"], res[0]["entropy"])
        assert torch.equal(res[k]["stats"], res[0]["stats"])
    for c in range(2):
        for k in range(P):
            assert torch.equal(outs[c][k]["logp"], res[k]["logp"])
            assert torch.equal(outs[c][k]["stats"], res[k]["stats"])
    # gathered path: same partials, same combine -> bitwise-equal logp / entropy
    b = _bounds(V, P)
    parts = torch.stack([otk.otk_row_partials(ctxs[0], d["logits"][:, b[k]:b[k + 1]].contiguous(), d["targets"],
                                              b[k], V, row_mask=d["mask"]) for k in range(P)]).contiguous()
    g = otk.otk_policy_loss_fwd_bwd_partials(ctxs[0], d["logits"][:, b[0]:b[1]].contiguous(), d["targets"], d["mask"],
                                             d["row_traj"], d["adv"], d["old"], d["ref"], nl, cfg, b[0], V, parts)
    ctxs[0].check()
    assert torch.equal(g["logp"], res[0]["logp"]) and torch.equal(g["entropy"], res[0]["entropy"])
    sg, sv = otk.stats_dict(g["stats"]), otk.stats_dict(res[0]["stats"])
    assert abs(sg["loss"] - sv["loss"]) <= 1e-12 * max(1.0, abs(sg["loss"]))   # fp64 sums, CTA grouping differs
    assert sg["n_tokens"] == sv["n_tokens"] == N and sg["n_clipped"] == sv["n_clipped"]
    # oracle
    ocfg = oracle_cfg(cfg)
    want = O.policy_loss_fwd_bwd(h["wide"], h["targets"], h["mask"], h["row_traj"], h["adv"], h["old"], h["ref"], N,
                                 ocfg)
    tol = LOGP_TOL[dtype]
    m = h["mask"].astype(bool)
    assert np.max(np.abs(res[0]["logp"].cpu().numpy()[m] - want["logp"][m])) < tol
    assert np.max(np.abs(res[0]["entropy"].cpu().numpy()[m] - want["entropy"][m])) < tol
    assert abs(sv["loss"] - want["loss"]) <= 1e-4 * max(abs(want["loss"]), 1e-3)
    rows = [j for j in range(n) if h["mask"][j]]
    dc = dcoef_rows(h, want["logp"], ocfg, N, True)
    assert check_dlogits_rows(dl, want["dlogits"], want["coef"], rows, dtype, V, dc, wide=h["wide"],
                              targets=h["targets"], h=h, cfg=ocfg) <= 1.0
    gd = dl.float()
    masked = [j for j in range(n) if not h["mask"][j]]
    assert all(bool((gd[j] == 0).all()) for j in masked)          # every rank zero-filled its columns
    for x in xchgs:
        x.close()
    for c in ctxs:
        c.close()


def test_vpf_equals_unsharded_kernel_dlogits(otk):
    """The fused shard path writes the same dlogits as the unsharded loss within bf16 rounding, with a real
    KL term and a mix of clipped rows."""
    n, V, P = 200, 151936, 2
    d, h = row_problem(n, V, dtype="bf16", seed=77, force_clip=5)
    ctxs = [otk.Context(0) for _ in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    xchgs = otk.VpfExchange.local_group(ctxs, 4096, max_ctas=74)      # rows_cap > num_rows is fine
    N = int(h["mask"].sum())
    nl = torch.tensor([N], dtype=torch.int64, device="cuda")
    cfg = otk.LossCfg(kl_beta=0.04)
    dl = torch.empty_like(d["logits"])
    res = _run_vpf(otk, ctxs, xchgs, streams, d, V, nl, cfg, dl)[0]
    full = otk.otk_policy_loss_fwd_bwd(ctxs[0], d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"],
                                       d["old"], d["ref"], nl, cfg)
    ctxs[0].check()
    assert float((res[0]["logp"] - full["logp"]).abs().max()) < 1e-5
    a, bb = dl.float(), full["dlogits"].float()
    err = ((a - bb).abs() / (bb.abs() * 2 ** -6 + 1e-9)).max().item()
    assert err <= 1.0
    sv, sf = otk.stats_dict(res[0]["stats"]), otk.stats_dict(full["stats"])
    assert abs(sv["loss"] - sf["loss"]) <= 1e-5 * max(abs(sf["loss"]), 1e-3)
    assert sv["n_clipped"] == sf["n_clipped"] and sv["n_tokens"] == sf["n_tokens"]
    for x in xchgs:
        x.close()


def test_vpf_host_validation(otk):
    ctx = otk.Context(0)
    d, h = row_problem(8, 1024, dtype="bf16", seed=1)
    nl = torch.tensor([int(h["mask"].sum())], dtype=torch.int64, device="cuda")
    x = otk.VpfExchange.local_group([ctx, ctx], 4)          # rows_cap 4 < 8 rows
    with pytest.raises(otk.OtkError, match="OTK_ERR_SHAPE"):
        otk.otk_policy_loss_fwd_bwd_vpf(ctx, d["logits"][:, :512], d["targets"], d["mask"], d["row_traj"], d["adv"],
                                        d["old"], d["ref"], nl, otk.LossCfg(), 0, 1024, x[0])
    with pytest.raises(ValueError):
        otk.VpfExchange(0, 9, 4, [0] * 9)
    x[0].close()
    x[1].close()
    ctx.close()


def test_vpf_missing_peer_times_out(otk):
    """Only rank 0 of 2 runs: its CTAs give up after the timeout with OTK_ERR_PEER_TIMEOUT (sticky: later rows
    do not wait again), so a lost peer costs ~20 s, never a hang."""
    import time
    n, V = 16, 2048
    d, h = row_problem(n, V, dtype="bf16", seed=3, mask_p=1.0)
    ctxs = [otk.Context(0), otk.Context(0)]
    x = otk.VpfExchange.local_group(ctxs, n, max_ctas=8)
    nl = torch.tensor([n], dtype=torch.int64, device="cuda")
    t0 = time.time()
    otk.otk_policy_loss_fwd_bwd_vpf(ctxs[0], d["logits"][:, :1024], d["targets"], d["mask"], d["row_traj"],
                                    d["adv"], d["old"], d["ref"], nl, otk.LossCfg(), 0, V, x[0])
    torch.cuda.synchronize()
    dt = time.time() - t0
    with pytest.raises(otk.OtkError, match="OTK_ERR_PEER_TIMEOUT"):
        ctxs[0].check()
    assert 10 < dt < 60, dt
    for e in x:
        e.close()


def test_vpf_cuda_graph_replay(otk):
    """The grouped call captured in a CUDA graph and replayed three times: the device-resident epoch of every
    rank advances per replay, so every replay reproduces the eager bits."""
    n, V, P = 96, 151936, 2
    d, h = row_problem(n, V, dtype="bf16", seed=21)
    ctxs = [otk.Context(0) for _ in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    xchgs = otk.VpfExchange.local_group(ctxs, n, max_ctas=74)
    nl = torch.tensor([int(h["mask"].sum())], dtype=torch.int64, device="cuda")
    cfg = otk.LossCfg(kl_beta=0.04)
    dl = torch.empty_like(d["logits"])
    eager = _run_vpf(otk, ctxs, xchgs, streams, d, V, nl, cfg, dl)[0]
    eager = [{k: t.clone() for k, t in r.items() if k != "dlogits"} for r in eager]
    dl_eager = dl.clone()
    b = _bounds(V, P)
    graph = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(graph):
        outs = otk.otk_policy_loss_fwd_bwd_vpf_group(
            ctxs, [d["logits"][:, b[k]:b[k + 1]] for k in range(P)], d["targets"], d["mask"], d["row_traj"],
            d["adv"], d["old"], d["ref"], nl, cfg, b[:P], V, xchgs, dlogits=[dl[:, b[k]:b[k + 1]] for k in range(P)])
    for _ in range(3):
        dl.zero_()
        for o in outs:
            o["logp"].zero_()
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        for c in ctxs:
            c.check()
        for k in range(P):
            assert torch.equal(outs[k]["logp"], eager[k]["logp"])
            assert torch.equal(outs[k]["stats"], eager[k]["stats"])
        assert torch.equal(dl, dl_eager)
    for x in xchgs:
        x.close()


@pytest.mark.parametrize("case", ["zero_rows", "all_masked", "bad_target"])
def test_vpf_edges(otk, case):
    """Degenerate inputs keep every rank in lockstep: no rows, only loss-masked rows (zero-filled, no exchange),
    and an out-of-range target on a trainable row (skipped by every rank, OTK_ERR_TARGET_RANGE). A normal call
    on the same buffers afterwards still matches the gathered path (the call counters advanced together)."""
    n, V, P = 40, 4096, 2
    d, h = row_problem(n, V, dtype="bf16", seed=9, mask_p=0.0 if case == "all_masked" else 0.7)
    ctxs = [otk.Context(0) for _ in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    xchgs = otk.VpfExchange.local_group(ctxs, n, max_ctas=16)
    cfg = otk.LossCfg()
    b = _bounds(V, P)
    dl = torch.full_like(d["logits"], 7.0)
    if case == "zero_rows":
        e = {k: (t[:0] if isinstance(t, torch.Tensor) and t.dim() >= 1 and t.shape[0] == n else t)
             for k, t in d.items()}
        e["logits"] = d["logits"][:0]
        nl = torch.zeros(1, dtype=torch.int64, device="cuda")
        out = _run_vpf(otk, ctxs, xchgs, streams, e, V, nl, cfg, dl[:0])[0]
        for r in out:
            assert otk.stats_dict(r["stats"])["n_tokens"] == 0
    elif case == "all_masked":
        nl = torch.zeros(1, dtype=torch.int64, device="cuda")
        out = _run_vpf(otk, ctxs, xchgs, streams, d, V, nl, cfg, dl)[0]
        assert bool((dl == 0).all())
        for r in out:
            assert otk.stats_dict(r["stats"])["n_tokens"] == 0 and bool((r["logp"] == 0).all())
    else:
        j = int(np.flatnonzero(h["mask"])[0])
        bad = d["targets"].clone()
        bad[j] = V + 5
        e = dict(d, targets=bad)
        nl = torch.tensor([int(h["mask"].sum())], dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        out = otk.otk_policy_loss_fwd_bwd_vpf_group(
            ctxs, [e["logits"][:, b[k]:b[k + 1]] for k in range(P)], e["targets"], e["mask"], e["row_traj"],
            e["adv"], e["old"], e["ref"], nl, cfg, b[:P], V, xchgs, dlogits=[dl[:, b[k]:b[k + 1]] for k in range(P)])
        torch.cuda.synchronize()
        for c in ctxs:
            with pytest.raises(otk.OtkError, match="OTK_ERR_TARGET_RANGE"):
                c.check()
        assert bool((dl[j] == 0).all())
        # the data error must not end the other rows' waits — every other row equals the gathered path
        # on the same inputs (which also skips row j)
        gctx = otk.Context(0)
        parts = torch.stack([otk.otk_row_partials(gctx, e["logits"][:, b[k]:b[k + 1]].contiguous(), e["targets"],
                                                  b[k], V, row_mask=e["mask"]) for k in range(P)]).contiguous()
        g = otk.otk_policy_loss_fwd_bwd_partials(gctx, e["logits"][:, b[0]:b[1]].contiguous(), e["targets"],
                                                 e["mask"], e["row_traj"], e["adv"], e["old"], e["ref"], nl, cfg,
                                                 b[0], V, parts)
        torch.cuda.synchronize()
        with pytest.raises(otk.OtkError, match="OTK_ERR_TARGET_RANGE"):
            gctx.check()
        for k in range(P):
            assert torch.equal(out[k]["logp"], g["logp"]) and torch.equal(out[k]["entropy"], g["entropy"])
        # pass 2 differs in form (bf16 e from tensor memory x scale vs one fp32 exponential per element): the two
        # agree within bf16 rounding on every row, and row j is zero in both
        a_, g_ = dl[:, b[0]:b[1]].float(), g["dlogits"].float()
        assert float(((a_ - g_).abs() / (g_.abs() * 2 ** -6 + 1e-30)).max()) <= 1.0
        sv, sg = otk.stats_dict(out[0]["stats"]), otk.stats_dict(g["stats"])
        assert sv["n_tokens"] == sg["n_tokens"] == int(h["mask"].sum()) - 1
        gctx.close()
        keep = ctxs   # they own the exchange buffers; fresh contexts for the next call (the error word is sticky)
        ctxs = [otk.Context(0) for _ in range(P)]
    # a normal call afterwards, same buffers: equal to the gathered path
    nl = torch.tensor([int(h["mask"].sum())], dtype=torch.int64, device="cuda")
    out = _run_vpf(otk, ctxs, xchgs, streams, d, V, nl, cfg, dl)[0]
    parts = torch.stack([otk.otk_row_partials(ctxs[0], d["logits"][:, b[k]:b[k + 1]].contiguous(), d["targets"],
                                              b[k], V, row_mask=d["mask"]) for k in range(P)]).contiguous()
    g = otk.otk_policy_loss_fwd_bwd_partials(ctxs[0], d["logits"][:, b[0]:b[1]].contiguous(), d["targets"], d["mask"],
                                             d["row_traj"], d["adv"], d["old"], d["ref"], nl, cfg, b[0], V, parts)
    ctxs[0].check()
    assert torch.equal(g["logp"], out[0]["logp"]) and torch.equal(out[1]["logp"], out[0]["logp"])
    for x in xchgs:
        x.close()
