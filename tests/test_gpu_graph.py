"""The step is CUDA-graph capturable (otk.h conventions): masks, advantages and the fused loss
over two micro-batches captured once and replayed give exactly the eager results (-m gpu)."""
import numpy as np
import pytest
import torch

from synth import make_logits, make_noise
from synth.trajectories import random_small_batch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("credit", ["trajectory", "turn"])
def test_step_graph_replay_equals_eager(credit):
    import paper_2601_07376_b200 as otk
    from paper_2601_07376_b200.step import MicroBatch, PolicyLossStep
    ctx = otk.Context(0)
    rng = np.random.default_rng(3)
    tb = random_small_batch(rng, 16, max_segs=6, max_len=40, num_groups=4)
    N, V = tb.num_rows, 4096
    db = otk.traj_batch_to_device(tb)
    logits, targets = make_logits(N, V, dtype="bf16", seed=1, device="cuda")
    lp = otk.otk_logprob_entropy_fwd(ctx, logits, targets)["logp"]
    old = (lp + make_noise(N, 0.05, 1, device="cuda")).contiguous()
    ref = (lp + make_noise(N, 0.1, 2, device="cuda")).contiguous()
    h = N // 2

    def make_step():
        return PolicyLossStep(ctx, db, torch.from_numpy(tb.group_id).cuda(), 4,
                              torch.from_numpy(tb.turn_offsets).cuda(), torch.from_numpy(tb.turn_rewards).cuda(), V,
                              otk.LossCfg(), credit=credit, gamma=0.9)

    def mbs(dl):
        return [MicroBatch(0, h, logits[:h], targets[:h], old[:h], ref[:h], dl[:h]),
                MicroBatch(h, N, logits[h:], targets[h:], old[h:], ref[h:], dl[h:])]

    dl_e = torch.empty_like(logits)
    eager = make_step()
    eager.run(mbs(dl_e))
    torch.cuda.synchronize()
    dl_g = torch.zeros_like(logits)
    st = make_step()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):            # warm-up on the capture stream (occupancy queries, lazy init)
        st.run(mbs(dl_g))
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    dl_g.zero_()
    st.stats.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        st.run(mbs(dl_g))
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ctx.check()
    assert torch.equal(st.stats, eager.stats)
    assert torch.equal(dl_g, dl_e)
    ctx.close()


def test_lmhead_loss_and_decode_sampler_graph_replay():
    """otk_lmhead_policy_loss_fwd_bwd (5 launches, tensor maps as kernel parameters) and the decode sampler
    (clustered launch) captured once and replayed reproduce the eager outputs bit for bit (otk.h: every call is
    graph-capturable)."""
    import paper_2601_07376_b200 as otk
    from synth import make_lmhead
    ctx = otk.Context(0)
    N, V, d = 300, 2056, 192
    h, w, y = make_lmhead(N, V, d, seed=8, device="cuda")
    mk = (torch.arange(N, device="cuda") % 4 != 0).to(torch.uint8)
    rt = torch.arange(N, device="cuda", dtype=torch.int32) // 100
    adv = torch.tensor([0.3, -0.7, 1.1], device="cuda", dtype=torch.float64)
    lp = otk.otk_lmhead_logprob_fwd(ctx, h, w, y)["logp"]
    old = (lp + make_noise(N, 0.05, 1, device="cuda")).contiguous()
    nl = mk.sum().to(torch.int64).reshape(1)
    cfg = otk.LossCfg(kl_beta=0.04, ent_coef=0.01)
    eager = otk.otk_lmhead_policy_loss_fwd_bwd(ctx, h, w, y, mk, rt, adv, old, lp.contiguous(), nl, cfg)
    lg, _ = make_logits(12, 151936, dtype="bf16", seed=9, device="cuda")
    u = torch.rand(12, device="cuda")
    se = otk.otk_sample_tokens(ctx, lg, u)
    torch.cuda.synchronize()
    outs = dict(workspace=torch.empty_like(eager["workspace"]), dhidden=torch.empty_like(eager["dh"]),
                dweight=torch.empty_like(eager["dW"]), stats=torch.zeros_like(eager["stats"]))
    so = dict(tokens=torch.empty_like(se["tokens"]), logp=torch.empty_like(se["logp"]))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):   # warm-up on the capture stream
        otk.otk_lmhead_policy_loss_fwd_bwd(ctx, h, w, y, mk, rt, adv, old, lp.contiguous(), nl, cfg, **outs)
        otk.otk_sample_tokens(ctx, lg, u, out=so)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        got = otk.otk_lmhead_policy_loss_fwd_bwd(ctx, h, w, y, mk, rt, adv, old, lp.contiguous(), nl, cfg, **outs)
        otk.otk_sample_tokens(ctx, lg, u, out=so)
    for _ in range(2):
        outs["dhidden"].zero_()
        g.replay()
    torch.cuda.synchronize()
    ctx.check()
    assert torch.equal(got["dh"], eager["dh"]) and torch.equal(got["dW"], eager["dW"])
    assert torch.equal(got["stats"], eager["stats"])
    assert torch.equal(so["tokens"], se["tokens"]) and torch.equal(so["logp"], se["logp"])
    ctx.close()
