"""Seeded synthetic trajectory batches shaped like the paper's agent workloads.

Recipe:
  * Table 1 scenarios: single-turn math, multi-turn gomoku, two-agent gomoku.
  * Segments follow the FSM of PAPER.md §2.2 (lines 163-179): a turn-0 CONTEXT segment (PENDING),
    then per turn an ACTION segment (GENERATING) and an OBSERVATION segment (INTERACTING);
    PAD rows fill each trajectory to T (packed-batch padding, reading R12).
  * Per-turn scores (SPEC.md:37-50 ``turn_rewards``); the episode return is built by the method,
    not here.

Layout (the C-ABI's ``otk_traj_batch``, include/otk.h): a CSR of segments per trajectory.
Source codes: 0 CONTEXT, 1 ACTION, 2 OBSERVATION, 3 PAD (data labels only).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

CONTEXT, ACTION, OBSERVATION, PAD = 0, 1, 2, 3
NO_AGENT = -1


@dataclass
class WorkloadConfig:
    name: str
    num_traj: int          # B (trajectories / agent-views)
    T: int                 # rows per trajectory (packed length incl. PAD)
    V: int                 # vocabulary
    dtype: str             # "bf16" | "f32"
    num_groups: int        # G
    group_size: int
    seed: int
    kl_beta: float         # 0 => no reference policy term
    note: str = ""

    @property
    def num_rows(self) -> int:
        return self.num_traj * self.T


# SURVEY.md §8(a)/(d) configuration table (BASELINE.json "configs").
CONFIGS: Dict[str, WorkloadConfig] = {
    "tiny": WorkloadConfig("tiny", 4, 64, 1024, "f32", 1, 4, 1, 0.04,
                           "1 group x 4 trajectories, 2 turns, T=64, V=1024, fp32 logits"),
    "math": WorkloadConfig("math", 512, 2048, 151936, "bf16", 64, 8, 2, 0.04,
                           "single-turn math GRPO: 64 prompts x group 8, T=2048, V=151936 bf16"),
    "game": WorkloadConfig("game", 128, 8192, 151936, "bf16", 16, 8, 3, 0.0,
                           "multi-turn gomoku-style game, 4-8 turns, env-token masking, T=8192, group 8"),
    "marl": WorkloadConfig("marl", 256, 4096, 151936, "bf16", 16, 16, 4, 0.04,
                           "two-agent episodes, interleaved turns, per-agent loss masks, T=4096, group 16"),
    "vp": WorkloadConfig("vp", 256, 16384, 151936, "bf16", 32, 8, 5, 0.04,
                         "vocab-parallel stress: 256 x T=16384, V=151936"),
}


@dataclass
class TrajBatch:
    """Host-side (numpy) segment CSR for B trajectories plus their rewards and group ids."""
    tok_offsets: np.ndarray        # int64 [B+1]
    seg_offsets: np.ndarray        # int32 [B+1]
    seg_source: np.ndarray         # uint8 [S]
    seg_agent: np.ndarray          # int16 [S]
    seg_len: np.ndarray            # int32 [S]
    terminated: np.ndarray         # uint8 [B]
    traj_agent: Optional[np.ndarray]  # int16 [B] or None (the agent each view trains)
    turn_offsets: np.ndarray       # int32 [B+1] CSR into turn_rewards
    turn_rewards: np.ndarray       # float64 [nnz] per-turn scores
    group_id: np.ndarray           # int32 [B]
    num_groups: int
    meta: dict = field(default_factory=dict)

    @property
    def num_traj(self) -> int:
        return int(self.tok_offsets.shape[0] - 1)

    @property
    def num_rows(self) -> int:
        return int(self.tok_offsets[-1])

    @property
    def num_segments(self) -> int:
        return int(self.seg_len.shape[0])


def _pack(trajs: List[List[tuple]], rewards: List[List[float]], group_id, num_groups,
          traj_agent=None, terminated=None, meta=None) -> TrajBatch:
    B = len(trajs)
    tok = np.zeros(B + 1, np.int64)
    sego = np.zeros(B + 1, np.int32)
    src, ag, ln = [], [], []
    for b, segs in enumerate(trajs):
        n = 0
        for (s, a, L) in segs:
            src.append(s); ag.append(a); ln.append(L); n += L
        tok[b + 1] = tok[b] + n
        sego[b + 1] = sego[b] + len(segs)
    to = np.zeros(B + 1, np.int32)
    rw = []
    for b, r in enumerate(rewards):
        rw.extend(r)
        to[b + 1] = to[b] + len(r)
    return TrajBatch(
        tok_offsets=tok, seg_offsets=sego,
        seg_source=np.asarray(src, np.uint8), seg_agent=np.asarray(ag, np.int16),
        seg_len=np.asarray(ln, np.int32),
        terminated=np.ones(B, np.uint8) if terminated is None else np.asarray(terminated, np.uint8),
        traj_agent=None if traj_agent is None else np.asarray(traj_agent, np.int16),
        turn_offsets=to, turn_rewards=np.asarray(rw, np.float64),
        group_id=np.asarray(group_id, np.int32), num_groups=int(num_groups), meta=meta or {})


def _fit(segs: List[tuple], T: int) -> List[tuple]:
    """Trim the segment list at T rows and pad the remainder with one PAD segment."""
    out, n = [], 0
    for (s, a, L) in segs:
        if n >= T:
            break
        L = min(L, T - n)
        out.append((s, a, L)); n += L
    if n < T:
        out.append((PAD, NO_AGENT, T - n))
    return out


def _u(rng, lo, hi):
    return int(rng.integers(lo, hi + 1))


def _tiny(rng, cfg):
    trajs, rewards = [], []
    for b in range(cfg.num_traj):
        segs = [(CONTEXT, NO_AGENT, _u(rng, 8, 16))]
        for _ in range(2):
            segs.append((ACTION, 0, _u(rng, 6, 12)))
            segs.append((OBSERVATION, NO_AGENT, _u(rng, 4, 8)))
        trajs.append(_fit(segs, cfg.T))
        rewards.append([float(rng.integers(-1, 2)) for _ in range(2)])
    gid = np.zeros(cfg.num_traj, np.int32)
    return _pack(trajs, rewards, gid, cfg.num_groups)


def _math(rng, cfg):
    T = cfg.T
    trajs, rewards, gid = [], [], []
    p_g = rng.uniform(0.0, 1.0, size=cfg.num_groups)
    for b in range(cfg.num_traj):
        g = b // cfg.group_size
        ctx = _u(rng, 64, 512)
        act = _u(rng, 256, T - ctx - 4)
        trajs.append(_fit([(CONTEXT, NO_AGENT, ctx), (ACTION, 0, act), (OBSERVATION, NO_AGENT, 4)], T))
        rewards.append([float(rng.random() < p_g[g])])
        gid.append(g)
    return _pack(trajs, rewards, gid, cfg.num_groups)


def _game(rng, cfg, turns=(4, 8)):
    T = cfg.T
    trajs, rewards, gid = [], [], []
    for b in range(cfg.num_traj):
        segs = [(CONTEXT, NO_AGENT, _u(rng, 256, 512))]
        nt = _u(rng, *turns)
        invalid_at = _u(rng, 0, nt - 1) if rng.random() < 0.1 else -1
        outcome = float(rng.choice([1.0, 0.0, -1.0], p=[0.4, 0.2, 0.4]))
        r = []
        for t in range(nt):
            segs.append((ACTION, 0, _u(rng, 400, 1000)))
            segs.append((OBSERVATION, NO_AGENT, _u(rng, 100, 200)))
            if t == invalid_at:
                r.append(-1.0)   # invalid move ends the episode with -1
                break
            r.append(outcome if t == nt - 1 else 0.0)
        # keep only turns whose ACTION survives the T cut (rewards attach to action tokens)
        fitted = _fit(segs, T)
        n_act = sum(1 for s in fitted if s[0] == ACTION)
        trajs.append(fitted)
        rewards.append(r[:n_act])
        gid.append(b % cfg.num_groups)  # strided: every group spans all batch shards
    return _pack(trajs, rewards, gid, cfg.num_groups)


def _marl(rng, cfg):
    """Two-agent zero-sum episodes; each episode appears once per agent (its own view)."""
    T = cfg.T
    E = cfg.num_traj // 2
    ep_groups = cfg.num_groups // 2
    per_group = max(1, E // ep_groups)
    trajs, rewards, gid, tagent = [], [], [], []
    for e in range(E):
        g = min(e // per_group, ep_groups - 1)
        segs = [(CONTEXT, NO_AGENT, _u(rng, 150, 300))]
        for _ in range(_u(rng, 4, 8)):
            for a in (0, 1):
                segs.append((ACTION, a, _u(rng, 120, 280)))
                segs.append((OBSERVATION, NO_AGENT, _u(rng, 40, 80)))
        fitted = _fit(segs, T)
        r0 = float(rng.integers(-1, 2))
        for a in (0, 1):
            n_act = sum(1 for s in fitted if s[0] == ACTION and s[1] == a)
            ra = r0 if a == 0 else -r0
            rewards.append([0.0] * (n_act - 1) + [ra] if n_act > 0 else [])
            trajs.append(fitted)
            gid.append(a * ep_groups + g)
            tagent.append(a)
    return _pack(trajs, rewards, gid, cfg.num_groups, traj_agent=tagent)


def make_batch(cfg: WorkloadConfig | str, seed: Optional[int] = None) -> TrajBatch:
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    rng = np.random.default_rng(cfg.seed if seed is None else seed)
    fn = {"tiny": _tiny, "math": _math, "game": _game, "marl": _marl,
          "vp": lambda r, c: _game(r, c, turns=(8, 16))}[cfg.name]
    tb = fn(rng, cfg)
    tb.meta.update(config=cfg.name, T=cfg.T, V=cfg.V)
    return tb


def random_small_batch(rng: np.random.Generator, B: int, max_segs: int = 6, max_len: int = 9,
                       n_agents: int = 2, num_groups: int = 2) -> TrajBatch:
    """Arbitrary (not FSM-shaped) small batches for property tests: any source order."""
    trajs, rewards, gid = [], [], []
    for b in range(B):
        ns = int(rng.integers(1, max_segs + 1))
        segs = []
        for _ in range(ns):
            s = int(rng.integers(0, 4))
            a = int(rng.integers(0, n_agents)) if s == ACTION else NO_AGENT
            segs.append((s, a, int(rng.integers(1, max_len + 1))))
        trajs.append(segs)
        rewards.append([float(x) for x in rng.normal(size=int(rng.integers(0, 3)))])
        gid.append(int(rng.integers(0, num_groups)))
    return _pack(trajs, rewards, gid, num_groups)


def concat_batches(parts: List[TrajBatch]) -> TrajBatch:
    trajs, rewards, gid, tag = [], [], [], []
    has_ag = any(p.traj_agent is not None for p in parts)
    for p in parts:
        for b in range(p.num_traj):
            s0, s1 = p.seg_offsets[b], p.seg_offsets[b + 1]
            trajs.append([(int(p.seg_source[i]), int(p.seg_agent[i]), int(p.seg_len[i]))
                          for i in range(s0, s1)])
            rewards.append(list(p.turn_rewards[p.turn_offsets[b]:p.turn_offsets[b + 1]]))
            gid.append(int(p.group_id[b]))
            tag.append(int(p.traj_agent[b]) if p.traj_agent is not None else -1)
    return _pack(trajs, rewards, gid, max(p.num_groups for p in parts),
                 traj_agent=tag if has_ag else None)


def slice_batch(tb: TrajBatch, b0: int, b1: int) -> TrajBatch:
    """Trajectories [b0, b1) of a batch as a batch of their own (offsets rebased; group ids stay global) — one
    rank's shard of a global batch under batch sharding (paper_2601_07376_b200.dist.plan_batch_shards)."""
    s0, s1 = int(tb.seg_offsets[b0]), int(tb.seg_offsets[b1])
    t0, t1 = int(tb.turn_offsets[b0]), int(tb.turn_offsets[b1])
    r0 = int(tb.tok_offsets[b0])
    return TrajBatch(tok_offsets=(tb.tok_offsets[b0:b1 + 1] - r0).astype(np.int64),
                     seg_offsets=(tb.seg_offsets[b0:b1 + 1] - s0).astype(np.int32),
                     seg_source=tb.seg_source[s0:s1].copy(), seg_agent=tb.seg_agent[s0:s1].copy(),
                     seg_len=tb.seg_len[s0:s1].copy(), terminated=tb.terminated[b0:b1].copy(),
                     traj_agent=None if tb.traj_agent is None else tb.traj_agent[b0:b1].copy(),
                     turn_offsets=(tb.turn_offsets[b0:b1 + 1] - t0).astype(np.int32),
                     turn_rewards=tb.turn_rewards[t0:t1].copy(), group_id=tb.group_id[b0:b1].copy(),
                     num_groups=tb.num_groups, meta=dict(tb.meta, shard=(b0, b1)))


def split_rows(num_rows: int, rows_per_chunk: int):
    """Row ranges [r0, r1) of the micro-batches a step is streamed in."""
    return [(r, min(r + rows_per_chunk, num_rows)) for r in range(0, num_rows, rows_per_chunk)]
