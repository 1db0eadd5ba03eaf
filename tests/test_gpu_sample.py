"""Rollout sampling kernel (R32) vs the oracle (-m gpu).

Greedy tokens are bit-exact (argmax, ties to the lowest id). A sampled token is an integer decided by
floating point: the kernel's fp32 cdf and the oracle's float64 cdf agree to ~1e-6, so the token must
equal the oracle's whenever u lies farther than TOL = 2e-5 from the boundaries of the oracle token's
cdf interval, and otherwise must be a token whose interval is within TOL of u (either neighbour of a
boundary is a correct draw). logp of the returned token within the forward tolerance (2e-3 bf16).
"""
import math

import numpy as np
import pytest
import torch

from oracle import oracle_ref as O
from synth import make_logits
from tests.gpu_common import LOGP_TOL

pytestmark = pytest.mark.gpu
TOL = 2e-5


@pytest.fixture(scope="module")
def otk():
    import paper_2601_07376_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(otk):
    c = otk.Context(0)
    yield c
    c.close()


def _cdf(x, s):
    z = s * np.asarray(x, np.float64)
    e = np.exp(z - z.max())
    return np.cumsum(e / math.fsum(e))


def _check_sampled(tok, lp, wide, u, s, dtype, rows):
    exact = 0
    for j in rows:
        t = int(tok[j])
        want, wlp = O.sample_token(wide[j], float(u[j]), s)
        cdf = _cdf(wide[j], s)
        lo = cdf[want - 1] if want > 0 else 0.0
        if t == want:
            exact += 1
        else:
            far = (u[j] - lo) > TOL and (cdf[want] - u[j]) > TOL
            assert not far, (j, t, want, u[j], lo, cdf[want])
            glo = cdf[t - 1] if t > 0 else 0.0
            assert glo - TOL <= u[j] <= cdf[t] + TOL, (j, t, want)
        z = s * wide[j]
        zl = z.max() + math.log(math.fsum(np.exp(z - z.max())))
        assert abs(float(lp[j]) - (z[t] - zl)) < LOGP_TOL[dtype], (j, float(lp[j]), z[t] - zl)
    return exact


@pytest.mark.parametrize("dtype,V,ld,n,scale", [("bf16", 151936, 151936, 384, 1.0), ("bf16", 151936, 151936, 300, 0.7),
                                                ("f32", 1000, 1000, 300, 1.0), ("bf16", 4100, 4104, 200, 1.3),
                                                ("bf16", 17, 24, 64, 1.0), ("f32", 50000, 50004, 64, 2.0),
                                                ("bf16", 262144, 262144, 64, 1.0)])
def test_sample_tokens_vs_oracle(otk, ctx, dtype, V, ld, n, scale):
    logits, _ = make_logits(n, V, ld=ld if ld != V else None, dtype=dtype, seed=V % 977 + n, device="cpu")
    wide = logits.double().numpy()[:, :V]
    rng = np.random.default_rng(V + n)
    u = rng.random(n).astype(np.float32)
    u[:4] = [0.0, np.float32(1.0 - 2 ** -24), 0.5, np.float32(1e-7)]      # edges of [0, 1)
    out = otk.otk_sample_tokens(ctx, logits.cuda(), torch.from_numpy(u).cuda(), logit_scale=scale, vocab=V)
    ctx.check()
    tok = out["tokens"].cpu().numpy()
    lp = out["logp"].cpu().numpy()
    assert np.all((tok >= 0) & (tok < V))
    rows = range(n) if V * n <= 4e7 else sorted(set(range(0, n, max(1, n // 64))) | {0, 1, 2, 3, n - 1})
    exact = _check_sampled(tok, lp, wide, u.astype(np.float64), scale, dtype, rows)
    assert exact >= 0.9 * len(rows)


def test_greedy_bit_exact(otk, ctx):
    n, V = 96, 151936
    logits, _ = make_logits(n, V, dtype="bf16", seed=5, device="cpu")
    x = logits.clone()
    x[1, :] = 0.0                                   # SPEC.md:316 zero weights -> token 0
    x[2, 77] = x[2, 150001] = x[2].max() + 1.0      # ties -> lowest id
    x[3, :] = float("-inf")
    x[3, 151935] = 1.0                              # the last column is the only finite one
    x[4, :] = float("-inf")                         # degenerate row: token 0, logp -inf
    x[5, 0:100] = float("-inf")
    out = otk.otk_sample_tokens(ctx, x.cuda(), greedy=True)
    ctx.check()
    tok = out["tokens"].cpu().numpy()
    wide = x.double().numpy()
    for j in range(n):
        if j == 4:
            assert tok[j] == 0 and out["logp"][j].item() == float("-inf")
            continue
        assert tok[j] == int(np.argmax(wide[j])), j
        assert abs(out["logp"][j].item() - O.sample_token(wide[j], 0.0, greedy=True)[1]) < LOGP_TOL["bf16"]
    assert tok[1] == 0 and tok[2] == 77 and tok[3] == 151935


def test_sample_masked_columns_never_drawn(otk, ctx):
    """-inf logits carry no mass: a draw never lands on them (also at u ~ 1)."""
    n, V = 256, 8192
    logits, _ = make_logits(n, V, dtype="bf16", seed=9, device="cpu")
    keep = torch.zeros(V, dtype=torch.bool)
    keep[torch.randperm(V, generator=torch.Generator().manual_seed(1))[:40]] = True
    logits[:, ~keep] = float("-inf")
    u = torch.rand(n, generator=torch.Generator().manual_seed(2))
    u[:3] = torch.tensor([0.0, 1.0 - 2 ** -24, 0.9999])
    out = otk.otk_sample_tokens(ctx, logits.cuda(), u.float().cuda())
    ctx.check()
    assert bool(keep[out["tokens"].cpu().long()].all())


def test_sample_empirical_distribution(otk, ctx):
    """frequencies of 2^16 draws (seeded uniforms) within 4 sigma of softmax(s x)."""
    V, n, s = 8, 1 << 16, 0.8
    x = torch.tensor([1.0, 0.0, -1.0, 2.0, 0.5, -3.0, 1.5, 0.25], dtype=torch.float32)
    logits = x.repeat(n, 1)
    u = torch.rand(n, generator=torch.Generator().manual_seed(3)).float()
    out = otk.otk_sample_tokens(ctx, logits.cuda(), u.cuda(), logit_scale=s)
    ctx.check()
    f = np.bincount(out["tokens"].cpu().numpy(), minlength=V) / n
    p = np.exp(s * x.double().numpy())
    p /= p.sum()
    assert np.all(np.abs(f - p) < 4 * np.sqrt(p * (1 - p) / n))


def test_sample_errors(otk, ctx):
    logits = torch.zeros(4, 64, device="cuda")
    with pytest.raises(ValueError):
        otk.otk_sample_tokens(ctx, logits)                       # uniforms required unless greedy
    with pytest.raises(otk.OtkError):
        otk.otk_sample_tokens(ctx, logits, torch.zeros(4, device="cuda"), logit_scale=0.0)
    otk.otk_sample_tokens(ctx, logits, torch.tensor([0.1, 1.5, 0.2, 0.3], device="cuda"))
    with pytest.raises(otk.OtkError) as e:
        ctx.check()
    assert e.value.status == 1                                   # OTK_ERR_INVALID_ARG: u outside [0, 1)


def test_temperature_argument(otk, ctx):
    """temperature = 1/logit_scale; temperature < 1e-6 is the greedy limit."""
    from synth import make_logits
    lg, _ = make_logits(64, 5000, dtype="bf16", seed=12, device="cuda")
    u = torch.rand(64, device="cuda")
    a = otk.otk_sample_tokens(ctx, lg, u, temperature=0.5)["tokens"]
    b = otk.otk_sample_tokens(ctx, lg, u, logit_scale=2.0)["tokens"]
    assert torch.equal(a, b)
    g = otk.otk_sample_tokens(ctx, lg, u, temperature=1e-7)["tokens"]
    assert torch.equal(g, otk.otk_sample_tokens(ctx, lg, greedy=True)["tokens"])


def test_greedy_without_logp_same_tokens(otk, ctx):
    """Greedy with logp not requested skips the exponentials: the same tokens (ties, -inf rows, degenerate rows)."""
    n, V = 700, 151936
    logits, _ = make_logits(n, V, dtype="bf16", seed=8, device="cpu")
    x = logits.clone()
    x[2, 77] = x[2, 150001] = x[2].max() + 1.0
    x[4, :] = float("-inf")
    x[5, 0:100] = float("-inf")
    xc = x.cuda()
    a = otk.otk_sample_tokens(ctx, xc, greedy=True)
    b = otk.otk_sample_tokens(ctx, xc, greedy=True, want_logp=False)
    c = otk.otk_sample_tokens(ctx, xc[:40].contiguous(), greedy=True, want_logp=False)   # cluster-split rows
    ctx.check()
    assert "logp" not in b
    assert torch.equal(a["tokens"], b["tokens"]) and torch.equal(a["tokens"][:40], c["tokens"])
    assert int(b["tokens"][4]) == 0 and int(b["tokens"][2]) == 77


@pytest.mark.parametrize("dtype,V", [("bf16", 151936), ("f32", 50000), ("bf16", 4100)])
def test_sampled_degenerate_rows_ring_kernel(otk, ctx, dtype, V):
    """>= 148 rows (the ring kernel): all -inf rows give token 0 / logp -inf; a single finite column is always
    drawn (first, last, and a middle column, for u = 0 and u -> 1); rows with huge logit ranges (overflow path)."""
    n = 200
    ld = -(-V // 8) * 8                                  # 16-byte rows
    logits, _ = make_logits(n, V, ld=ld if ld != V else None, dtype=dtype, seed=V % 101, device="cpu")
    x = logits.clone()[:, :V]
    x[0, :] = float("-inf")
    for j, col in ((1, 0), (2, V - 1), (3, V // 2), (4, 0), (5, V - 1)):
        x[j, :] = float("-inf")
        x[j, col] = 3.0
    x[6, : V // 2] = -80.0          # a large step inside the row: the warp reference is raised on overflow
    x[6, V // 2:] = 60.0
    x[7, :] = -200.0                 # all far below 0
    x[7, V - 3] = 150.0
    u = torch.rand(n, generator=torch.Generator().manual_seed(4)).float()
    u[1:4] = 0.0
    u[4:6] = 1.0 - 2 ** -24
    xp = torch.full((n, ld), float("nan"), dtype=x.dtype)   # padding columns never read
    xp[:, :V] = x
    out = otk.otk_sample_tokens(ctx, xp.cuda(), u.cuda(), vocab=V)
    ctx.check()
    tok = out["tokens"].cpu().numpy()
    lp = out["logp"].cpu().numpy()
    assert tok[0] == 0 and lp[0] == float("-inf")
    assert [int(t) for t in tok[1:6]] == [0, V - 1, V // 2, 0, V - 1]
    assert np.allclose(lp[1:6], 0.0, atol=1e-6)
    assert V // 2 <= tok[6] < V                   # all the mass sits in the upper half
    assert tok[7] == V - 3
    wide = x.double().numpy()
    rows = list(range(8, n, 7))
    exact = _check_sampled(tok, lp, wide, u.double().numpy(), 1.0, dtype, rows)
    assert exact >= 0.9 * len(rows)


@pytest.mark.parametrize("dtype,V,n", [("bf16", 151936, 16), ("bf16", 151936, 37), ("bf16", 151936, 1),
                                       ("f32", 50000, 30), ("bf16", 4100, 9), ("bf16", 17, 5),
                                       ("bf16", 151936, 33), ("f32", 151936, 16),
                                       ("bf16", 151936, 100), ("bf16", 151936, 148), ("f32", 151936, 96),
                                       ("bf16", 151936, 64)])   # >= 96 rows: the ring kernel, rows split by clusters
def test_decode_batches(otk, ctx, dtype, V, n):
    """Decode-sized batches (<= 49 rows: k_sample_dec, one row per cluster, each CTA's column range held in registers;
    96-148 rows: the ring kernel, each row split over a cluster of 2-3 CTAs):
    sampled draws vs the oracle, greedy bit-exact, degenerate rows, and single finite columns at the first / last
    column and at the boundaries between the cluster's CTA ranges (u = 0 and u -> 1)."""
    ld = -(-V // 8) * 8
    logits, _ = make_logits(n, V, ld=ld if ld != V else None, dtype=dtype, seed=V % 89 + n, device="cpu")
    x = logits.clone()[:, :V]
    C = min(8, 148 // n)
    es = 2 if dtype == "bf16" else 4
    per = -(-(-(-(V * es) // 16) // 64) // C) * 64 * 16 // es     # columns per CTA range (whole 1 KB segments)
    special = {}
    if n >= 5:
        x[0, :] = float("-inf")
        special[0] = None
        for j, col in ((1, 0), (2, V - 1), (3, min(per, V - 1)), (4, max(min(per, V - 1) - 1, 0))):
            x[j, :] = float("-inf")
            x[j, col] = 3.0
            special[j] = col
    if n >= 7:
        x[5, : V // 2] = -80.0
        x[5, V // 2:] = 60.0
        x[6, :] = -200.0
        x[6, V - 3] = 150.0
        special[6] = V - 3
    if n >= 16:   # the first column of CTA rank 1 for every cluster size the kernel may pick (3-8, by occupancy)
        for j, c in zip(range(8, 14), range(3, 9)):
            col = min(-(-(-(-(V * es) // 16) // 64) // c) * 64 * 16 // es, V - 1)
            x[j, :] = float("-inf")
            x[j, col] = 1.0
            special[j] = col
    if n >= 32:   # the ring kernel's cluster split (96-148 rows): first column of rank 1's 12 KB chunks, C = 2-8
        nch = -(-(-(-(V * es) // 16) * 16) // 12288)
        for j, c in zip(range(14, 21), range(2, 9)):
            col = min(-(-nch // c) * 12288 // es, V - 1)
            x[j, :] = float("-inf")
            x[j, col] = 1.0
            special[j] = col
    u = torch.rand(n, generator=torch.Generator().manual_seed(n)).float()
    if n >= 5:
        u[1:3] = 0.0
        u[3:5] = 1.0 - 2 ** -24
    xp = torch.full((n, ld), float("nan"), dtype=x.dtype)        # padding columns never read
    xp[:, :V] = x
    out = otk.otk_sample_tokens(ctx, xp.cuda(), u.cuda(), vocab=V)
    g = otk.otk_sample_tokens(ctx, xp.cuda(), greedy=True, vocab=V)
    ctx.check()
    tok, lp = out["tokens"].cpu().numpy(), out["logp"].cpu().numpy()
    gt, glp = g["tokens"].cpu().numpy(), g["logp"].cpu().numpy()
    wide = x.double().numpy()
    for j, col in special.items():
        if col is None:
            assert tok[j] == 0 and lp[j] == float("-inf") and gt[j] == 0 and glp[j] == float("-inf")
        else:
            assert tok[j] == col and gt[j] == col, (j, tok[j], gt[j], col)
    if n >= 7:
        assert V // 2 <= tok[5] < V
    rows = [j for j in range(n) if j not in special and j != 5]
    exact = _check_sampled(tok, lp, wide, u.double().numpy(), 1.0, dtype, rows)
    assert exact >= 0.9 * len(rows)
    for j in rows:
        assert gt[j] == int(np.argmax(wide[j])), j
        assert abs(float(glp[j]) - O.sample_token(wide[j], 0.0, greedy=True)[1]) < LOGP_TOL[dtype]


@pytest.mark.parametrize("n", [3, 200])
def test_greedy_rows_below_no_mass_threshold(otk, ctx, n):
    """R32: logits <= -1e30 carry no mass — a row of finite -1e31 logits is degenerate (token 0, logp -inf) in the
    decode kernel (3 rows) and the lane-strided kernel (200 rows) alike, for greedy and sampled draws."""
    x = torch.randn(n, 4096).to(torch.bfloat16)
    x[0, :] = -1e31
    xc = x.cuda()
    g = otk.otk_sample_tokens(ctx, xc, greedy=True)
    s = otk.otk_sample_tokens(ctx, xc, torch.full((n,), 0.5, device="cuda"))
    ctx.check()
    for o in (g, s):
        assert int(o["tokens"][0]) == 0 and float(o["logp"][0]) == float("-inf")
    assert int(g["tokens"][1]) == int(torch.argmax(x[1].float()))
