"""Pins of the float64 oracle to things other than itself (-m "not gpu").

Each test names what fixes the expected value: a SPEC.md/PAPER.md worked example (tests/golden/),
a closed form derived independently of the oracle's algorithm, brute force on tiny inputs, an
invariant, or a library routine (torch float64).
"""
import itertools
import math

import numpy as np
import pytest
import torch

from oracle import oracle_ref as O
from synth.trajectories import _pack, random_small_batch, make_batch, CONTEXT, ACTION, OBSERVATION, PAD
from tests.conftest import load_golden

CF = {k: float(v) for k, v in load_golden("closed_forms.txt").items()}


# ----------------------------------------------------------------------------- O1 masks
def _masks(tb, **kw):
    return O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len,
                         tb.terminated, traj_agent=tb.traj_agent, **kw)


def test_arith_worked_example():
    """SPEC.md:215/389-391/414: [CONTEXT "3+4=", ACTION "7\\n", OBSERVATION "done"]."""
    g = load_golden("arith_mask.txt")
    names = {"CONTEXT": CONTEXT, "ACTION": ACTION, "OBSERVATION": OBSERVATION}
    segs = []
    for part in g["segments"].split("|"):
        src, text = part.strip().split(":", 1)
        text = text.replace("\\n", "\n")
        segs.append((names[src], 0 if src == "ACTION" else -1, len(text)))
    tb = _pack([segs], [[float(g["turn_rewards"])]], [0], 1)
    m = _masks(tb)
    assert tb.num_rows == int(g["n_tokens"])
    assert "".join(map(str, m["loss_mask"])) == g["loss_mask"]
    assert "".join(map(str, m["response_mask"])) == g["response_mask"]
    c = m["traj_source_counts"][0]
    assert (c[CONTEXT], c[ACTION], c[OBSERVATION]) == (
        int(g["context_tokens"]), int(g["action_tokens"]), int(g["observation_tokens"]))
    assert m["n_loss"] == int(g["action_tokens"])


def _brute_tokens(segs):
    """Literal expansion: one (source, agent, segment-position) record per token."""
    toks = []
    for k, (s, a, L) in enumerate(segs):
        toks.extend([(s, a, k)] * L)
    return toks


@pytest.mark.parametrize("train_agent", [-1, 0, 1])
def test_masks_bruteforce_enumeration(train_agent):
    """Every sequence of <= 3 segments over {CTX, ACT(a0), ACT(a1), OBS, PAD} x len {1, 2}."""
    kinds = [(CONTEXT, -1), (ACTION, 0), (ACTION, 1), (OBSERVATION, -1), (PAD, -1)]
    cases = []
    for n in (1, 2, 3):
        for combo in itertools.product(kinds, repeat=n):
            for lens in itertools.product((1, 2), repeat=n):
                cases.append([(s, a, L) for (s, a), L in zip(combo, lens)])
    # pack many trajectories into one batch (exercises the CSR offsets too)
    tb = _pack(cases, [[0.0]] * len(cases), [0] * len(cases), 1)
    m = _masks(tb, train_agent=train_agent)
    row = 0
    for b, segs in enumerate(cases):
        for (s, a, k) in _brute_tokens(segs):
            want_loss = int(s == ACTION and (train_agent == -1 or a == train_agent))
            want_resp = int(not (k == 0 and s == CONTEXT) and s != PAD)
            assert m["loss_mask"][row] == want_loss
            assert m["response_mask"][row] == want_resp
            assert m["row_traj"][row] == b
            row += 1
        total = sum(L for _, _, L in segs)
        assert m["traj_source_counts"][b].sum() == total          # SPEC.md:91 partition
        assert m["traj_loss_tokens"][b] == sum(L for s, a, L in segs
                                                if s == ACTION and (train_agent == -1 or a == train_agent))
    assert row == tb.num_rows
    assert m["n_loss"] == int(m["loss_mask"].sum())


def test_masks_agent_views_partition_actions():
    """two agents' loss masks over a shared transcript are disjoint and cover ACTION."""
    tb = make_batch("marl")
    both = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len,
                         train_agent=-1)
    m0 = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len, train_agent=0)
    m1 = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len, train_agent=1)
    assert not np.any(m0["loss_mask"] & m1["loss_mask"])
    assert np.array_equal(m0["loss_mask"] | m1["loss_mask"], both["loss_mask"])
    view = _masks(tb)  # per-view agent: each view trains only its own agent's actions
    for b in range(tb.num_traj):
        r0, r1 = tb.tok_offsets[b], tb.tok_offsets[b + 1]
        src = m0 if tb.traj_agent[b] == 0 else m1
        assert np.array_equal(view["loss_mask"][r0:r1], src["loss_mask"][r0:r1])


def test_masks_errors():
    tb = _pack([[(CONTEXT, -1, 2), (ACTION, 0, 2)]], [[1.0]], [0], 1, terminated=[0])
    with pytest.raises(O.Unterminated):
        _masks(tb)
    tb = _pack([[(CONTEXT, -1, 2), (ACTION, 0, 2)]], [[1.0]], [0], 1)
    tb.tok_offsets[1] = 5   # rows != sum of segment lengths
    with pytest.raises(O.BadTrajectory):
        _masks(tb)
    with pytest.raises(O.EmptyGroup):
        O.build_masks(np.zeros(1, np.int64), np.zeros(1, np.int32), [], [], [])


@pytest.mark.parametrize("seed", range(5))
def test_masks_random_properties(seed):
    rng = np.random.default_rng(seed)
    tb = random_small_batch(rng, 20)
    m = _masks(tb)
    assert int(m["traj_source_counts"].sum()) == tb.num_rows
    for b in range(tb.num_traj):
        r0, r1 = tb.tok_offsets[b], tb.tok_offsets[b + 1]
        assert np.all(m["row_traj"][r0:r1] == b)
        assert m["loss_mask"][r0:r1].sum() == m["traj_source_counts"][b, ACTION]


# ----------------------------------------------------------------------------- O2 advantages
def test_constant_group_zero_advantage():
    """all returns equal -> A = 0 (exact for dyadic values)."""
    for v in (0.0, 1.0, -1.0, 0.5):
        a = O.group_advantages([0] * 8, [v] * 8, 1)["adv"]
        assert np.all(a == 0.0)
    a = O.group_advantages([0] * 3, [0.1] * 3, 1)["adv"]
    assert np.all(np.abs(a) <= 1e-15)


@pytest.mark.parametrize("k", range(1, 8))
def test_binary_group_closed_form(k):
    G = 8
    R = [1.0] * k + [0.0] * (G - k)
    pop = O.group_advantages([0] * G, R, 1)["adv"]
    smp = O.group_advantages([0] * G, R, 1, unbiased=True)["adv"]
    ap, an = math.sqrt((G - k) / k), -math.sqrt(k / (G - k))
    assert np.allclose(pop[:k], ap, rtol=0, atol=1e-14) and np.allclose(pop[k:], an, rtol=0, atol=1e-14)
    f = math.sqrt((G - 1) / G)
    assert np.allclose(smp[:k], ap * f, atol=1e-14) and np.allclose(smp[k:], an * f, atol=1e-14)
    if k == 2:
        assert abs(pop[0] - CF["binary_G8_k2_pop_pos"]) < 1e-14
        assert abs(pop[-1] - CF["binary_G8_k2_pop_neg"]) < 1e-14
        assert abs(smp[0] - CF["binary_G8_k2_sample_pos"]) < 1e-14
        assert abs(smp[-1] - CF["binary_G8_k2_sample_neg"]) < 1e-14


def test_two_member_group():
    a = O.group_advantages([0, 0], [0.0, 1.0], 1)["adv"]
    assert a.tolist() == [-1.0, 1.0]
    a = O.group_advantages([0, 0], [0.0, 1.0], 1, unbiased=True)["adv"]
    assert np.allclose(a, [-1 / math.sqrt(2), 1 / math.sqrt(2)], atol=1e-15)


@pytest.mark.parametrize("seed", range(4))
def test_advantage_invariants(seed):
    rng = np.random.default_rng(seed)
    G, B = 5, 60
    gid = rng.integers(0, G, B)
    R = rng.normal(size=B)
    out = O.group_advantages(gid, R, G)
    for g in range(G):
        a = out["adv"][gid == g]
        if len(a) >= 2:
            assert abs(a.sum()) < 1e-12                      # sum of centred values
            assert abs((a ** 2).sum() - len(a)) < 1e-10      # population: sum A^2 = n
        assert out["group_size"][g] == int((gid == g).sum())
    nostd = O.group_advantages(gid, R, G, std_norm=False)["adv"]
    for b in range(B):
        assert abs(nostd[b] - (R[b] - R[gid == gid[b]].mean())) < 1e-12


def test_degenerate_and_singleton_groups():
    a = O.group_advantages([0, 1, 1], [3.0, 2.0, 2.0 + 1e-9], 2)
    assert a["adv"][0] == 0.0                      # singleton group: R - mean = 0
    assert a["group_std"][1] < 1e-8               # std below the floor: divide by 1
    assert abs(a["adv"][2] - 0.5e-9) < 1e-15
    with pytest.raises(O.GroupRange):
        O.group_advantages([0, 2], [1.0, 2.0], 2)
    with pytest.raises(O.EmptyGroup):
        O.group_advantages([], [], 1)


def test_zero_sum_antisymmetry():
    """PAPER.md:263 / SPEC.md:230: zero-sum two-agent episodes => A(agent1) = -A(agent0) exactly."""
    tb = make_batch("marl")
    R = O.episode_returns(tb.turn_offsets, tb.turn_rewards)
    assert np.all(R[0::2] == -R[1::2])
    a = O.group_advantages(tb.group_id, R, tb.num_groups)["adv"]
    assert np.all(a[0::2] == -a[1::2])


def test_episode_returns_undiscounted():
    """return = sum over turns of the per-turn scores, undiscounted."""
    R = O.episode_returns(np.array([0, 3, 3, 5]), np.array([0.5, 0.0, -1.0, 0.25, 0.25]))
    assert R.tolist() == [-0.5, 0.0, 0.5]


# ----------------------------------------------------------------------------- O6 turn-level credit
def _one_traj(sources, agents, rewards, gid=0):
    from synth.trajectories import _pack
    segs = [(s, a, 3) for s, a in zip(sources, agents)]
    return _pack([segs], [rewards], [gid], 1)


def test_turn_returns_worked_example():
    """DESIGN.md R31 by hand: turns = trainable ACTION segments in order; G_k = sum_{j>=k} gamma^(j-k) r_j.
    Rewards [1, 0, 2] over 2 action turns (the third score lies past the last action and flows back)."""
    C, A_, Ob = O.CONTEXT, O.ACTION, O.OBSERVATION
    tb = _one_traj([C, A_, Ob, A_, Ob], [-1, 0, -1, 0, -1], [1.0, 0.0, 2.0])
    for gamma, want in ((0.5, [1.5, 1.0]), (1.0, [3.0, 2.0]), (0.0, [1.0, 0.0])):
        G, grp = O.turn_returns(tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.turn_offsets, tb.turn_rewards,
                                tb.group_id, gamma)
        assert G.tolist() == [0.0, want[0], 0.0, want[1], 0.0]
        assert grp.tolist() == [-1, 0, -1, 0, -1]
    # a turn with no score left (k >= R_b) has return 0
    tb = _one_traj([C, A_, A_, A_], [-1, 0, 0, 0], [4.0])
    G, _ = O.turn_returns(tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.turn_offsets, tb.turn_rewards,
                          tb.group_id, 0.9)
    assert G.tolist() == [0.0, 4.0, 0.0, 0.0]


def test_turn_returns_agent_views():
    """a view's turns are only its own agent's ACTION segments."""
    C, A_, Ob = O.CONTEXT, O.ACTION, O.OBSERVATION
    tb = _one_traj([C, A_, Ob, A_, Ob, A_], [-1, 0, -1, 1, -1, 0], [1.0, 2.0])
    for ta, want, units in ((0, [0.0, 2.0, 0.0, 0.0, 0.0, 2.0], (1, 5)), (1, [0.0, 0.0, 0.0, 2.0, 0.0, 0.0], (3,))):
        G, grp = O.turn_returns(tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.turn_offsets, tb.turn_rewards,
                                tb.group_id, 0.5, train_agent=ta)
        assert G.tolist() == want                       # agent 0: [1 + 0.5*2, 2]; agent 1: [1 + 0.5*2]
        assert np.flatnonzero(grp >= 0).tolist() == list(units)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_turn_returns_bellman_recursion(seed):
    """The reward-to-go satisfies G_k = r_k + gamma G_{k+1} (G_K = sum of the scores past the last turn,
    discounted) — a different formulation than the oracle's direct sum."""
    rng = np.random.default_rng(seed)
    C, A_, Ob = O.CONTEXT, O.ACTION, O.OBSERVATION
    K = int(rng.integers(1, 7))
    R = int(rng.integers(0, K + 3))
    r = rng.normal(size=R)
    srcs = [C] + [A_, Ob] * K
    tb = _one_traj(srcs, [-1] + [0, -1] * K, list(r))
    gamma = float(rng.uniform(0.5, 1.0))
    G, _ = O.turn_returns(tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.turn_offsets, tb.turn_rewards,
                          tb.group_id, gamma)
    Gt = G[1::2]
    nxt = 0.0
    for j in range(R - 1, K - 1, -1):          # scores past the last turn
        nxt = r[j] + gamma * nxt
    for k in range(K - 1, -1, -1):
        rk = r[k] if k < R else 0.0
        nxt = rk + gamma * nxt
        assert abs(Gt[k] - nxt) <= 1e-12 * max(1.0, abs(nxt))


def test_turn_level_reduces_to_trajectory_level():
    """One trainable ACTION turn per trajectory (single-turn math) and gamma = 1: turn-level credit IS
    trajectory-level GRPO, row by row, bit for bit (same values in the same order)."""
    from synth import make_batch
    tb = make_batch("math")
    m = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len, tb.terminated)
    G, grp = O.turn_returns(tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.turn_offsets, tb.turn_rewards,
                            tb.group_id, 1.0)
    adv_seg, adv_row = O.turn_level_advantages(m["row_seg"], G, grp, tb.num_groups)
    traj = O.group_advantages(tb.group_id, O.episode_returns(tb.turn_offsets, tb.turn_rewards), tb.num_groups)["adv"]
    tr = m["loss_mask"] == 1
    assert np.array_equal(adv_row[tr], traj[m["row_traj"]][tr])


def test_turn_level_group_worked_example_and_invariants():
    """Two trajectories of one group: turns G = [1.5, 1.0] and [0.5]; mean 1, population std sqrt(1/6), so
    A = [sqrt(1.5), 0, -sqrt(1.5)]. On the game workload every group's turn advantages have mean 0, std 1."""
    from synth.trajectories import _pack
    C, A_, Ob = O.CONTEXT, O.ACTION, O.OBSERVATION
    tb = _pack([[(C, -1, 2), (A_, 0, 2), (Ob, -1, 1), (A_, 0, 2)], [(C, -1, 2), (A_, 0, 3)]],
               [[1.0, 0.0, 2.0], [0.5]], [0, 0], 1)
    G, grp = O.turn_returns(tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.turn_offsets, tb.turn_rewards,
                            tb.group_id, 0.5)
    m = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len)
    adv_seg, adv_row = O.turn_level_advantages(m["row_seg"], G, grp, 1)
    s = math.sqrt(1.5)
    assert np.allclose(adv_seg, [0.0, s, 0.0, 0.0, 0.0, -s], atol=1e-15)
    assert np.allclose(adv_row, [0, 0, s, s, 0, 0, 0, 0, 0, -s, -s, -s], atol=1e-15)
    from synth import make_batch
    tb = make_batch("game")
    G, grp = O.turn_returns(tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.turn_offsets, tb.turn_rewards,
                            tb.group_id, 0.95)
    a = O.group_advantages(grp, G, tb.num_groups, skip_ungrouped=True)
    for g in range(tb.num_groups):
        x = a["adv"][grp == g]
        if a["group_std"][g] > 1e-8:
            assert abs(x.mean()) < 1e-12 and abs(x.std() - 1.0) < 1e-12
    assert np.all(a["adv"][grp < 0] == 0.0)


def test_loss_adv_index_plumbing():
    """adv_index selects the advantage per row: a segment-level array equal to the broadcast trajectory
    advantage gives the trajectory-level loss and gradient exactly."""
    from synth.trajectories import random_small_batch
    rng = np.random.default_rng(5)
    tb = random_small_batch(rng, 6, max_segs=5, max_len=6)
    m = O.build_masks(tb.tok_offsets, tb.seg_offsets, tb.seg_source, tb.seg_agent, tb.seg_len, tb.terminated)
    adv = rng.normal(size=tb.num_traj)
    seg_traj = np.repeat(np.arange(tb.num_traj), np.diff(tb.seg_offsets))
    adv_seg = adv[seg_traj]
    N = tb.num_rows
    X = rng.normal(size=(N, 50))
    y = rng.integers(0, 50, N)
    old = rng.normal(size=N) - 4.0
    a = O.policy_loss_fwd_bwd(X, y, m["loss_mask"], m["row_traj"], adv, old, None, m["n_loss"], O.LossCfg(kl_beta=0))
    b = O.policy_loss_fwd_bwd(X, y, m["loss_mask"], m["row_traj"], adv_seg, old, None, m["n_loss"],
                              O.LossCfg(kl_beta=0), adv_index=m["row_seg"])
    assert a["loss"] == b["loss"] and all(np.array_equal(a["dlogits"][j], b["dlogits"][j]) for j in range(N))


# ----------------------------------------------------------------------------- O3 forward
@pytest.mark.parametrize("V", [151936, 1024])
def test_uniform_row(V):
    """north_star: uniform logits give log-prob = -ln V (and entropy ln V)."""
    logp, H, lse, p = O.row_forward(np.zeros(V), 7)
    want = CF[f"uniform_logp_V{V}"]
    assert abs(logp - want) < 1e-12 and abs(H + want) < 1e-12
    assert abs(math.fsum(p) - 1) < 1e-12


@pytest.mark.parametrize("V,L", [(151936, 10), (1024, 5)])
def test_two_level_row(V, L):
    x = np.zeros(V)
    x[3] = L
    logp, H, _, _ = O.row_forward(x, 3)
    assert abs(logp - CF[f"twolevel_V{V}_L{L}_logp"]) < 1e-11
    assert abs(H - CF[f"twolevel_V{V}_L{L}_H"]) < 1e-11


def test_two_token_softplus():
    """V = 2: logp_y = -softplus(z_other - z_y)  (SPEC.md:327 two-token case)."""
    for a, b in [(0.3, -1.2), (5.0, 5.0), (-30.0, 12.0)]:
        logp, _, _, _ = O.row_forward(np.array([a, b]), 0)
        d = b - a
        want = -(max(d, 0.0) + math.log1p(math.exp(-abs(d))))
        assert abs(logp - want) < 1e-14


@pytest.mark.parametrize("seed", range(3))
def test_forward_vs_torch_float64(seed):
    """Library pin: torch.log_softmax / Categorical.entropy in float64 on CPU."""
    rng = np.random.default_rng(seed)
    x = rng.normal(scale=3.0, size=(6, 4099))
    t = torch.from_numpy(x)
    lsm = torch.log_softmax(t, dim=-1).numpy()
    ent = torch.distributions.Categorical(logits=t).entropy().numpy()
    for j in range(6):
        y = int(rng.integers(0, 4099))
        logp, H, lse, p = O.row_forward(x[j], y)
        assert abs(logp - lsm[j, y]) < 1e-12
        assert abs(H - ent[j]) < 1e-11
        assert np.allclose(np.log(p), lsm[j], atol=1e-12)


def test_forward_invariants():
    rng = np.random.default_rng(9)
    x = rng.normal(size=777) * 2
    base = O.row_forward(x, 5)
    shifted = O.row_forward(x + 123.25, 5)
    assert abs(base[0] - shifted[0]) < 1e-12 and abs(base[1] - shifted[1]) < 1e-12
    scaled = O.row_forward(x, 5, logit_scale=1 / 0.7)
    direct = O.row_forward(x / 0.7, 5)
    assert abs(scaled[0] - direct[0]) < 1e-13
    # sum_v exp(logp_v) = 1 over all targets (SPEC.md:308 normalisation)
    assert abs(math.fsum(math.exp(O.row_forward(x, v)[0]) for v in range(777)) - 1) < 1e-12
    # -inf entries contribute nothing: equal to the row with them removed
    xi = x.copy()
    xi[[1, 50, 600]] = -np.inf
    keep = np.setdiff1d(np.arange(777), [1, 50, 600])
    a = O.row_forward(xi, 5)
    b = O.row_forward(x[keep], int(np.searchsorted(keep, 5)))
    assert abs(a[0] - b[0]) < 1e-13 and abs(a[1] - b[1]) < 1e-13
    with pytest.raises(O.TargetRange):
        O.row_forward(x, 777)


# ----------------------------------------------------------------------------- O4 loss + grad
def _tiny_problem(rng, N=12, V=8, B=3, beta=0.04, kl_type=3, scale=1.0, delta_sd=0.05):
    x = rng.normal(scale=2.0, size=(N, V))
    y = rng.integers(0, V, N)
    mask = (rng.random(N) < 0.7).astype(np.uint8)
    row_traj = np.sort(rng.integers(0, B, N)).astype(np.int32)
    adv = rng.normal(size=B)
    cfg = O.LossCfg(kl_beta=beta, kl_type=kl_type, logit_scale=scale)
    logp = np.array([O.row_forward(x[j], int(y[j]), scale)[0] for j in range(N)])
    old = logp + rng.normal(scale=delta_sd, size=N)
    ref = logp + rng.normal(scale=0.1, size=N)
    return x, y, mask, row_traj, adv, old, ref, cfg


def test_on_policy_loss_is_minus_mean_advantage():
    """north_star: old = new makes the ratio 1, so (with ref = new, KL 0) loss = -sum m A / N."""
    rng = np.random.default_rng(1)
    x, y, mask, rt, adv, _, _, cfg = _tiny_problem(rng)
    logp = np.array([O.row_forward(x[j], int(y[j]))[0] for j in range(len(y))])
    N = int(mask.sum())
    out = O.policy_loss_fwd_bwd(x, y, mask, rt, adv, logp, logp, N, cfg)
    want = -math.fsum(adv[rt[j]] for j in range(len(y)) if mask[j]) / N
    assert abs(out["loss"] - want) < 1e-14
    assert out["stats"]["kl_sum"] == 0.0 and out["stats"]["n_clipped"] == 0


def test_balanced_groups_zero_loss():
    """Equal trainable length per trajectory of a full group + on-policy => loss = 0 (sum A = 0)."""
    rng = np.random.default_rng(2)
    B, T, V = 8, 5, 6
    R = rng.normal(size=B)
    adv = O.group_advantages([0] * B, R, 1)["adv"]
    x = rng.normal(size=(B * T, V))
    y = rng.integers(0, V, B * T)
    rt = np.repeat(np.arange(B), T).astype(np.int32)
    mask = np.tile([0, 1, 1, 1, 0], B).astype(np.uint8)
    logp = np.array([O.row_forward(x[j], int(y[j]))[0] for j in range(B * T)])
    out = O.policy_loss_fwd_bwd(x, y, mask, rt, adv, logp, None, int(mask.sum()), O.LossCfg(kl_beta=0.0))
    assert abs(out["loss"]) < 1e-15


def test_clip_closed_forms():
    cfg = O.LossCfg(kl_beta=0.0)
    for A in (0.7, 2.0):
        L, G, clipped, _ = O.row_loss_terms(math.log(1.5), 0.0, None, A, cfg)
        assert abs(L - CF["clip_pos_factor"] * A) < 1e-15 and G == 0.0 and clipped
    for A in (-0.7, -2.0):
        L, G, clipped, _ = O.row_loss_terms(math.log(0.5), 0.0, None, A, cfg)
        assert abs(L - CF["clip_neg_factor"] * A) < 1e-15 and G == 0.0 and clipped
    # inside the trust region: pg = -A r, gradient -A r
    L, G, clipped, _ = O.row_loss_terms(math.log(1.1), 0.0, None, 1.5, cfg)
    assert abs(L + 1.5 * 1.1) < 1e-14 and abs(G + 1.5 * 1.1) < 1e-14 and not clipped
    # A > 0 with r < 1 - eps is NOT clipped (min picks the unclipped term)
    L, G, clipped, _ = O.row_loss_terms(math.log(0.5), 0.0, None, 1.0, cfg)
    assert abs(L + 0.5) < 1e-15 and abs(G + 0.5) < 1e-15 and not clipped
    # ratio clamp: |logp - old| > C => r = e^C and zero gradient
    L, G, _, _ = O.row_loss_terms(30.0, 0.0, None, -1.0, O.LossCfg(kl_beta=0.0, clip_low=10.0))
    assert G == 0.0 and abs(L - math.exp(20.0)) < 1e-6


def test_kl_estimators():
    cfg = O.LossCfg(kl_beta=1.0, clip_low=0.2)
    L, G, _, kl = O.row_loss_terms(-1.0, -1.0, -0.9, 0.0, cfg)      # d = ref - logp = 0.1
    assert abs(kl - CF["k3_d0p1_value"]) < 1e-15 and abs(G - CF["k3_d0p1_grad"]) < 1e-15
    L, G, _, kl = O.row_loss_terms(-1.0, -1.0, -1.5, 0.0, O.LossCfg(kl_beta=1.0, kl_type=1))
    assert abs(kl - 0.5) < 1e-15 and G == 1.0
    L, G, _, kl = O.row_loss_terms(-1.0, -1.0, -1.5, 0.0, O.LossCfg(kl_beta=1.0, kl_type=2))
    assert abs(kl - 0.125) < 1e-15 and abs(G - 0.5) < 1e-15


@pytest.mark.parametrize("V,kl_type,scale,seed", [
    (2, 3, 1.0, 0), (3, 3, 1.0, 1), (8, 1, 1.0, 2), (8, 2, 1 / 0.7, 3), (32, 3, 1.0, 4), (32, 3, 1 / 0.7, 5)])
def test_gradient_finite_differences(V, kl_type, scale, seed):
    """analytic dlogits vs central finite differences of the loss (h = 1e-6)."""
    rng = np.random.default_rng(seed)
    x, y, mask, rt, adv, old, ref, cfg = _tiny_problem(rng, N=10, V=V, kl_type=kl_type, scale=scale)
    # force one clipped row and keep every row >= 1e-3 away from the clip / clamp kinks
    j0 = int(np.flatnonzero(mask)[0])
    logp0 = O.row_forward(x[j0], int(y[j0]), scale)[0]
    adv[rt[j0]] = abs(adv[rt[j0]]) + 0.1
    old[j0] = logp0 - math.log(1.5)
    N = int(mask.sum())
    out = O.policy_loss_fwd_bwd(x, y, mask, rt, adv, old, ref, N, cfg)
    for j in range(len(y)):
        if mask[j]:
            r = math.exp(out["logp"][j] - old[j])
            assert min(abs(r - 0.8), abs(r - 1.2)) > 1e-3
    h = 1e-6
    fd = np.zeros_like(x)
    for j in range(x.shape[0]):
        for v in range(V):
            xp, xm = x.copy(), x.copy()
            xp[j, v] += h
            xm[j, v] -= h
            fd[j, v] = (O.loss_only(xp, y, mask, rt, adv, old, ref, N, cfg)
                        - O.loss_only(xm, y, mask, rt, adv, old, ref, N, cfg)) / (2 * h)
    an = out["dlogits"]
    scale_ = np.max(np.abs(an))
    assert np.max(np.abs(an - fd)) <= 1e-6 * scale_ + 1e-12
    assert np.all(an[mask == 0] == 0.0)                        # mask soundness
    assert np.all(np.abs(an.sum(axis=1)) < 1e-15 + 1e-13 * scale_)   # rows sum to 0
    assert np.all(an[j0] == 0.0) or cfg.kl_beta != 0.0         # clipped row: only KL gradient


def test_sft_case_matches_torch_cross_entropy():
    """SPEC.md:503 SFT = update with A = 1: with old = logp, beta = 0, every row trainable,
    dlogits = d mean-CE / dz (torch float64 autograd, a library routine)."""
    rng = np.random.default_rng(7)
    N, V = 9, 17
    x = rng.normal(size=(N, V))
    y = rng.integers(0, V, N)
    logp = np.array([O.row_forward(x[j], int(y[j]))[0] for j in range(N)])
    out = O.policy_loss_fwd_bwd(x, y, np.ones(N, np.uint8), np.zeros(N, np.int32), np.ones(1),
                                logp, None, N, O.LossCfg(kl_beta=0.0))
    t = torch.from_numpy(x).requires_grad_(True)
    ce = torch.nn.functional.cross_entropy(t, torch.from_numpy(y))
    ce.backward()
    assert np.max(np.abs(out["dlogits"] - t.grad.numpy())) < 1e-16 + 1e-14
    assert abs(out["loss"] + 1.0) < 1e-15      # pg = -A r = -1 on every row


def test_zero_loss_tokens():
    rng = np.random.default_rng(3)
    x, y, mask, rt, adv, old, ref, cfg = _tiny_problem(rng)
    mask[:] = 0
    out = O.policy_loss_fwd_bwd(x, y, mask, rt, adv, old, ref, 0, cfg)
    assert out["loss"] == 0.0 and np.all(out["dlogits"] == 0.0)


# ----------------------------------------------------------------------------- O5 vocab shards
@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_vocab_shard_combine_equals_unsharded(P):
    rng = np.random.default_rng(P)
    V = 1000
    x = rng.normal(scale=3, size=V)
    x[[5, 400]] = -np.inf
    for y in (0, 333, 999):
        bounds = np.linspace(0, V, P + 1).astype(int)
        parts = [O.shard_partials(x[a:b], y, a) for a, b in zip(bounds[:-1], bounds[1:])]
        logp, H, lse = O.combine_partials(parts)
        ref = O.row_forward(x, y)
        assert abs(logp - ref[0]) < 1e-12 and abs(H - ref[1]) < 1e-12 and abs(lse - ref[2]) < 1e-12
    # an empty shard and an all -inf shard contribute nothing
    empty = O.shard_partials(x[:0], 3, 0)
    dead = O.shard_partials(np.full(4, -np.inf), 3, 0)
    assert empty == dead == (-math.inf, 0.0, 0.0, 0.0)
    got = O.combine_partials([empty, O.shard_partials(x, 3, 0), dead])
    assert abs(got[0] - O.row_forward(x, 3)[0]) < 1e-12


# ----------------------------------------------------------------------------- A4 variants (NEXT-4)
def test_dual_clip_closed_forms():
    """Dual-clip PPO (c = 3): for A < 0 the loss is capped at -c*A with zero gradient."""
    cfg = O.LossCfg(kl_beta=0.0, dual_clip=3.0)
    L, G, _, _ = O.row_loss_terms(math.log(5.0), 0.0, None, -1.0, cfg)     # pg = 5 > 3: capped
    assert abs(L - 3.0) < 1e-15 and G == 0.0
    L, G, _, _ = O.row_loss_terms(math.log(2.0), 0.0, None, -1.0, cfg)     # pg = 2 < 3: unchanged
    assert abs(L - 2.0) < 1e-15 and abs(G - 2.0) < 1e-15
    L, G, _, _ = O.row_loss_terms(math.log(5.0), 0.0, None, 1.0, cfg)      # A > 0: no dual clip
    assert abs(L + 1.2) < 1e-15 and G == 0.0


def _onpolicy(rng, tok_per_traj, V=6):
    rows = sum(tok_per_traj)
    x = rng.normal(size=(rows, V))
    y = rng.integers(0, V, rows)
    rt = np.repeat(np.arange(len(tok_per_traj)), tok_per_traj).astype(np.int32)
    lp = np.array([O.row_forward(x[j], int(y[j]))[0] for j in range(rows)])
    return x, y, rt, lp


def test_sequence_mean_reductions_closed_form():
    """seq-mean-token-mean: (1/B) sum_b mean_{j in b} L_j; seq-mean-token-sum: (1/B) sum_b sum_j L_j.
    On-policy, beta = 0: L_j = -A_b, so the losses are -(A0 + A1)/2 and -(A0*1 + A1*3)/2."""
    rng = np.random.default_rng(4)
    x, y, rt, lp = _onpolicy(rng, [1, 3])
    mask = np.ones(4, np.uint8)
    A = np.array([0.75, -0.25])
    base = dict(kl_beta=0.0)
    r1 = O.policy_loss_fwd_bwd(x, y, mask, rt, A, lp, None, 4, O.LossCfg(reduction=O.SEQ_MEAN_TOKEN_MEAN, **base))
    assert abs(r1["loss"] + (0.75 - 0.25) / 2) < 1e-15
    r2 = O.policy_loss_fwd_bwd(x, y, mask, rt, A, lp, None, 4, O.LossCfg(reduction=O.SEQ_MEAN_TOKEN_SUM, **base))
    assert abs(r2["loss"] + (0.75 * 1 - 0.25 * 3) / 2) < 1e-15
    r0 = O.policy_loss_fwd_bwd(x, y, mask, rt, A, lp, None, 4, O.LossCfg(**base))
    assert abs(r0["loss"] + (0.75 - 3 * 0.25) / 4) < 1e-15
    # equal lengths: seq-mean-token-mean == token-mean
    x, y, rt, lp = _onpolicy(rng, [2, 2, 2])
    m = np.ones(6, np.uint8)
    a = O.policy_loss_fwd_bwd(x, y, m, rt, np.array([1.0, -2.0, 0.5]), lp, None, 6, O.LossCfg(**base))
    b = O.policy_loss_fwd_bwd(x, y, m, rt, np.array([1.0, -2.0, 0.5]), lp, None, 6,
                              O.LossCfg(reduction=O.SEQ_MEAN_TOKEN_MEAN, **base))
    assert abs(a["loss"] - b["loss"]) < 1e-15 and np.allclose(a["dlogits"], b["dlogits"], atol=1e-16)


def test_entropy_bonus_vs_torch_autograd():
    """L = -c_H * H (A = 0 removes the PPO term): dlogits = w c_H s p (ln p + H), pinned to torch float64
    autograd of -c_H * w * H(softmax(s x)); a uniform row has zero entropy gradient."""
    rng = np.random.default_rng(8)
    N, V, c, s = 5, 9, 0.3, 1 / 0.7
    x = rng.normal(size=(N, V))
    x[2] = 0.0
    y = rng.integers(0, V, N)
    lp = np.array([O.row_forward(x[j], int(y[j]), s)[0] for j in range(N)])
    out = O.policy_loss_fwd_bwd(x, y, np.ones(N, np.uint8), np.zeros(N, np.int32), np.zeros(1), lp, None, N,
                                O.LossCfg(kl_beta=0.0, ent_coef=c, logit_scale=s))
    t = torch.from_numpy(x).requires_grad_(True)
    logp = torch.log_softmax(s * t, dim=-1)
    H = -(logp.exp() * logp).sum(dim=-1)
    (-c * H.sum() / N).backward()
    assert np.max(np.abs(out["dlogits"] - t.grad.numpy())) < 1e-15
    assert np.max(np.abs(out["dlogits"][2])) < 1e-17
    assert abs(out["loss"] + c * float(H.sum()) / N) < 1e-14


def test_sft_flag_matches_cross_entropy():
    """SPEC.md:503 SFT: L = -logp per token; token-mean equals torch cross_entropy (library pin)."""
    rng = np.random.default_rng(12)
    N, V = 7, 11
    x = rng.normal(size=(N, V))
    y = rng.integers(0, V, N)
    junk = rng.normal(size=N)                               # A / old must not matter in SFT mode
    out = O.policy_loss_fwd_bwd(x, y, np.ones(N, np.uint8), np.zeros(N, np.int32), np.array([-3.0]), junk, None,
                                N, O.LossCfg(kl_beta=0.0, sft=True))
    t = torch.from_numpy(x).requires_grad_(True)
    ce = torch.nn.functional.cross_entropy(t, torch.from_numpy(y))
    ce.backward()
    assert abs(out["loss"] - float(ce.detach())) < 1e-14
    assert np.max(np.abs(out["dlogits"] - t.grad.numpy())) < 1e-16 + 1e-14


@pytest.mark.parametrize("variant", ["dual", "ent", "seqmean", "seqsum", "sft"])
def test_variant_gradients_finite_differences(variant):
    rng = np.random.default_rng({"dual": 1, "ent": 2, "seqmean": 3, "seqsum": 4, "sft": 5}[variant])
    kw = dict(dual=dict(dual_clip=3.0), ent=dict(ent_coef=0.1), seqmean=dict(reduction=O.SEQ_MEAN_TOKEN_MEAN),
              seqsum=dict(reduction=O.SEQ_MEAN_TOKEN_SUM), sft=dict(sft=True))[variant]
    x, y, mask, rt, adv, old, ref, _ = _tiny_problem(rng, N=10, V=7)
    if variant == "dual":   # push some negative-advantage rows past the cap, away from the kink
        adv[:] = -np.abs(adv) - 0.2
        lp = np.array([O.row_forward(x[j], int(y[j]))[0] for j in range(10)])
        old = lp - np.where(np.arange(10) % 2 == 0, math.log(5.0), math.log(1.05))
    cfg = O.LossCfg(**kw)
    N = int(mask.sum())
    out = O.policy_loss_fwd_bwd(x, y, mask, rt, adv, old, ref, N, cfg)
    h = 1e-6
    fd = np.zeros_like(x)
    for j in range(x.shape[0]):
        for v in range(x.shape[1]):
            xp, xm = x.copy(), x.copy()
            xp[j, v] += h
            xm[j, v] -= h
            fd[j, v] = (O.loss_only(xp, y, mask, rt, adv, old, ref, N, cfg)
                        - O.loss_only(xm, y, mask, rt, adv, old, ref, N, cfg)) / (2 * h)
    sc = np.max(np.abs(out["dlogits"]))
    assert np.max(np.abs(out["dlogits"] - fd)) <= 1e-6 * sc + 1e-12
    assert abs(out["loss"] - O.loss_only(x, y, mask, rt, adv, old, ref, N, cfg)) < 1e-14


# ----------------------------------------------------------------------------- O7 sampling
def test_greedy_spec_examples():
    """zero weights -> token 0; single positive logit on 53 -> 53; ties -> lowest id."""
    x = np.zeros(128)
    assert O.sample_token(x, 0.3, greedy=True)[0] == 0
    x[53] = 2.0
    assert O.sample_token(x, 0.3, greedy=True)[0] == 53
    x = np.zeros(128)
    x[7] = x[9] = 1.5
    assert O.sample_token(x, 0.9, greedy=True)[0] == 7


def test_sample_two_token_closed_form():
    """V = 2: p_0 = 1 / (1 + e^{s (x_1 - x_0)}); token 0 iff u < p_0."""
    x = np.array([0.7, -0.4])
    for s in (1.0, 0.5, 3.0):
        p0 = 1.0 / (1.0 + math.exp(s * (x[1] - x[0])))
        assert O.sample_token(x, p0 - 1e-9, s)[0] == 0
        assert O.sample_token(x, p0 + 1e-9, s)[0] == 1
        t, lp = O.sample_token(x, p0 + 1e-9, s)
        assert abs(lp - math.log(1.0 - p0)) < 1e-12


def test_sample_uniform_row_is_floor():
    """Uniform logits: the inverse transform is t = floor(u V)."""
    V = 1000
    rng = np.random.default_rng(0)
    for u in rng.random(50):
        if abs(u * V - round(u * V)) > 1e-6:
            t, lp = O.sample_token(np.full(V, 0.25), u)
            assert t == int(math.floor(u * V)) and abs(lp + math.log(V)) < 1e-12


def test_sample_bruteforce_prefix_definition():
    """t = min{t : sum_{v<=t} p_v > u} by exactly rounded partial sums on small rows (-inf columns never drawn)."""
    rng = np.random.default_rng(1)
    for _ in range(40):
        V = int(rng.integers(2, 12))
        x = rng.normal(scale=2.0, size=V)
        x[rng.random(V) < 0.2] = -np.inf
        if np.all(np.isinf(x)):
            x[0] = 0.0
        u = float(rng.random())
        p = np.exp(x - x.max())
        p = p / math.fsum(p)
        want = next(t for t in range(V) if math.fsum(p[:t + 1]) > u)
        t, _ = O.sample_token(x, u)
        assert t == want and np.isfinite(x[t])


def test_sample_empirical_frequencies():
    """draws follow softmax(x / temperature): frequencies within 4 sigma over 20000 uniforms."""
    rng = np.random.default_rng(2)
    x = np.array([1.0, 0.0, -1.0, 2.0, 0.5])
    s = 0.7
    p = np.exp(s * x) / np.exp(s * x).sum()
    n = 20000
    t, _ = O.sample_tokens(np.tile(x, (n, 1)), rng.random(n), s)
    f = np.bincount(t, minlength=5) / n
    assert np.all(np.abs(f - p) < 4 * np.sqrt(p * (1 - p) / n))


def test_sample_temperature_is_logit_scale():
    """softmax(x / T): sampling x with scale s equals sampling s*x with scale 1."""
    rng = np.random.default_rng(3)
    x = rng.normal(size=300)
    for u in rng.random(20):
        assert O.sample_token(x, u, 2.5)[0] == O.sample_token(2.5 * x, u, 1.0)[0]


# ----------------------------------------------------------------------------- O8 LM head + forward
def test_lmhead_zero_weight_is_uniform():
    """W = 0: every logit is 0, so logp = -ln V and entropy = ln V (north_star's uniform pin)."""
    rng = np.random.default_rng(0)
    h = rng.normal(size=(3, 64))
    out = O.lmhead_logprob_fwd(h, np.zeros((1000, 64)), [0, 5, 999])
    for j in range(3):
        assert abs(out["logp"][j] + math.log(1000)) < 1e-12 and abs(out["entropy"][j] - math.log(1000)) < 1e-12


def test_lmhead_one_hot_hidden_reduces_to_forward():
    """h = e_k picks column k of W: the fused forward equals O3 on that column (a different code path)."""
    rng = np.random.default_rng(1)
    W = rng.normal(scale=2.0, size=(700, 32))
    for k, y, s in ((3, 10, 1.0), (31, 699, 0.7), (0, 0, 2.0)):
        h = np.zeros((1, 32))
        h[0, k] = 1.0
        out = O.lmhead_logprob_fwd(h, W, [y], s)
        lp, H, lse, _ = O.row_forward(W[:, k], y, s)
        assert out["logp"][0] == lp and out["entropy"][0] == H and out["lse"][0] == lse


def test_lmhead_vs_torch_float64():
    """Library pin: torch float64 matmul + log_softmax + entropy."""
    rng = np.random.default_rng(2)
    h = rng.normal(size=(5, 48))
    W = rng.normal(scale=0.3, size=(257, 48))
    y = rng.integers(0, 257, 5)
    out = O.lmhead_logprob_fwd(h, W, y, 1.3)
    z = 1.3 * (torch.from_numpy(h) @ torch.from_numpy(W).T)
    ls = torch.log_softmax(z, -1)
    for j in range(5):
        assert abs(out["logp"][j] - float(ls[j, y[j]])) < 1e-12
        assert abs(out["entropy"][j] + float((ls[j].exp() * ls[j]).sum())) < 1e-12
