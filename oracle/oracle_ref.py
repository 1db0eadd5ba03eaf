"""Float64 reference ("oracle") for the OpenTinker policy-gradient hot path — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may use this
module. It shares no code with the CUDA path (paper_2601_07376_b200/) and imports nothing from it.

What it computes (PAPER.md = /root/reference/PAPER.md, SPEC.md = /root/reference/SPEC.md; the
paper names no RL algorithm, so steps O2-O4 follow the readings listed in DESIGN.md §3):

  O1 build_masks           PAPER.md:167-174 (§2.2 PENDING / GENERATING / INTERACTING token masking),
                           PAPER.md:192 (§2.3 independent per-agent policies).
  O2 episode_returns,      SPEC.md:95 (return = sum of per-turn scores, undiscounted)
     group_advantages      (A_i = (R_i - mean)/(std if std > 1e-8 else 1)), BASELINE.json north_star (2).
  O3 row_forward           north_star (3): log-softmax + gather + entropy over the vocabulary.
  O4 row_loss_terms,       north_star (4): PPO-clipped surrogate + KL penalty, token-mean reduction,
     policy_loss_fwd_bwd   dlogits = coef * (softmax - onehot); gradient pattern SPEC.md:323.
  O6 turn_returns,         turn-level credit (
     turn_level_advantages DESIGN.md R31): discounted reward-to-go per trainable ACTION turn.
  O7 sample_token           rollout sampling (R32):
                           inverse-transform softmax sampling with a given uniform, greedy argmax.
  O8 lmhead_logprob_fwd    LM head fused with O3 (R33): z = s h W^T, then O3.
  O5 shard_partials,       vocab-sharded forward (north_star "all-reduced row max/sum-exp"): per-shard
     combine_partials      partials combined exactly (DESIGN.md §3 R25).

Every step is the plain definition in float64: numpy vector ops per row (exp/log/max) and
math.fsum (exactly rounded) for every sum; no blocking, fusion or reordering.

Pins (tests/test_oracle_pins.py, -m "not gpu"): SPEC.md's ARITH worked example for O1, brute-force
segment enumeration, closed-form binary-group advantages, constant-group zero, zero-sum
antisymmetry, uniform / two-level / V=2 rows for O3, torch float64 log_softmax
(library routine), old=new and clip closed forms, k3 values, central finite differences of the
loss for the gradient, and the SFT case against torch float64 cross_entropy autograd; loss variants
(dual-clip / sequence-mean closed forms, entropy bonus vs torch autograd, finite differences); O6:
hand-worked reward-to-go, agent views, the Bellman recursion, reduction to trajectory-level GRPO,
a hand-worked group and per-group mean 0 / std 1; O7: SPEC.md greedy examples, V=2 closed form,
uniform row = floor(uV), exactly-rounded prefix brute force, empirical frequencies, temperature;
O8: W = 0 (uniform), one-hot h (reduces to O3), torch float64 matmul + log_softmax.
Parity unpinned: none of the functions; the CHOICE among readings R2, R14-R16 (std estimator,
clip epsilon, ratio clamp, KL estimator), R31 (turn units and discounting) and R32 (inverse transform
as the sampling scheme) cannot be pinned to anything the paper prints.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

# Segment sources (§2.2 states; SPEC.md:31 SegmentSource + PAD, R12)
CONTEXT, ACTION, OBSERVATION, PAD = 0, 1, 2, 3
ANY_AGENT = -1

KL_K1, KL_K2, KL_K3 = 1, 2, 3


class OracleError(Exception):
    code = "ERROR"


class EmptyGroup(OracleError):        # SPEC.md:324 errors: EmptyGroup
    code = "EMPTY_GROUP"


class Unterminated(OracleError):      # SPEC.md:324 errors: UnterminatedTrajectory
    code = "UNTERMINATED"


class BadTrajectory(OracleError):     # SPEC.md:79-87 validate_trajectory; SPEC.md:91 partition
    code = "BAD_TRAJECTORY"


class TargetRange(OracleError):
    code = "TARGET_RANGE"


class GroupRange(OracleError):
    code = "GROUP_RANGE"


# --------------------------------------------------------------------------------------------
# O1: loss / response masks
# --------------------------------------------------------------------------------------------
def build_masks(tok_offsets, seg_offsets, seg_source, seg_agent, seg_len, terminated=None,
                train_agent: int = ANY_AGENT, traj_agent=None):
    """Expand per-trajectory segment lists into per-row labels.

    PENDING (CONTEXT) tokens are "excluded from loss computation"; only GENERATING
    (ACTION) tokens are "trainable"; INTERACTING (OBSERVATION) tokens "are masked
    from the loss". Agents do not share gradients, so an ACTION row
    is trainable only for the agent that emitted it (train_agent, or traj_agent[b] per view).
    response_mask: every non-PAD row after the turn-0 CONTEXT (prompt) segment (R13).
    """
    tok_offsets = np.asarray(tok_offsets, np.int64)
    B = tok_offsets.shape[0] - 1
    if B < 1:
        raise EmptyGroup("no trajectories")
    N = int(tok_offsets[B])
    loss_mask = np.zeros(N, np.uint8)
    response_mask = np.zeros(N, np.uint8)
    row_traj = np.full(N, -1, np.int32)
    row_seg = np.full(N, -1, np.int32)
    traj_loss_tokens = np.zeros(B, np.int64)
    traj_source_counts = np.zeros((B, 4), np.int64)
    for b in range(B):
        if terminated is not None and not terminated[b]:
            raise Unterminated(f"trajectory {b} not terminated")
        ta = int(traj_agent[b]) if traj_agent is not None else int(train_agent)
        row = int(tok_offsets[b])
        s0, s1 = int(seg_offsets[b]), int(seg_offsets[b + 1])
        if s1 < s0:
            raise BadTrajectory(f"trajectory {b}: segment offsets decrease")
        for k in range(s0, s1):
            src, L, ag = int(seg_source[k]), int(seg_len[k]), int(seg_agent[k])
            if L <= 0 or src > PAD:
                raise BadTrajectory(f"trajectory {b}: bad segment {k}")
            trainable = src == ACTION and (ta == ANY_AGENT or ag == ta)
            is_prompt = (k == s0) and src == CONTEXT
            responding = (not is_prompt) and src != PAD
            if row + L > int(tok_offsets[b + 1]):
                raise BadTrajectory(f"trajectory {b}: segments exceed its rows")
            loss_mask[row:row + L] = 1 if trainable else 0
            response_mask[row:row + L] = 1 if responding else 0
            row_traj[row:row + L] = b
            row_seg[row:row + L] = k
            traj_source_counts[b, src] += L
            if trainable:
                traj_loss_tokens[b] += L
            row += L
        if row != int(tok_offsets[b + 1]):
            raise BadTrajectory(f"trajectory {b}: segment lengths != row count")
    return dict(loss_mask=loss_mask, response_mask=response_mask, row_traj=row_traj, row_seg=row_seg,
                traj_loss_tokens=traj_loss_tokens, traj_source_counts=traj_source_counts,
                n_loss=int(traj_loss_tokens.sum()))


# --------------------------------------------------------------------------------------------
# O2: returns and group-relative advantages  (north_star (2))
# --------------------------------------------------------------------------------------------
def episode_returns(turn_offsets, turn_rewards):
    """R_b = sum of the per-turn scores of trajectory b, undiscounted."""
    B = len(turn_offsets) - 1
    return np.array([math.fsum(turn_rewards[turn_offsets[b]:turn_offsets[b + 1]]) for b in range(B)],
                    np.float64)


def group_advantages(group_id, returns, num_groups: int, std_norm: bool = True, unbiased: bool = False,
                     std_floor: float = 1e-8, skip_ungrouped: bool = False):
    """A_b = (R_b - mean_g) / (std_g if std_g > std_floor else 1)   (R2-R4).

    mean_g and std_g over the trajectories of b's group g; std is the population std unless
    `unbiased` (then / (n_g - 1), and std_g = 0 when n_g <= 1). std_norm=False gives R_b - mean_g.
    skip_ungrouped: elements with a negative group id belong to no group and get A = 0 (turn-level
    credit, O6: the non-unit segments).
    """
    group_id = np.asarray(group_id)
    returns = np.asarray(returns, np.float64)
    B = returns.shape[0]
    if B < 1:
        raise EmptyGroup("no trajectories")
    if (not skip_ungrouped and np.any(group_id < 0)) or np.any(group_id >= num_groups):
        raise GroupRange("group id out of range")
    mean = np.zeros(num_groups)
    std = np.zeros(num_groups)
    size = np.zeros(num_groups, np.int32)
    for g in range(num_groups):
        Rg = [float(returns[b]) for b in range(B) if group_id[b] == g]
        n = len(Rg)
        size[g] = n
        if n == 0:
            continue
        mean[g] = math.fsum(Rg) / n
        denom = (n - 1) if unbiased else n
        if denom > 0:
            std[g] = math.sqrt(math.fsum((r - mean[g]) ** 2 for r in Rg) / denom)
    adv = np.zeros(B)
    for b in range(B):
        g = int(group_id[b])
        if g < 0:
            continue
        centred = float(returns[b]) - mean[g]
        if std_norm:
            adv[b] = centred / (std[g] if std[g] > std_floor else 1.0)
        else:
            adv[b] = centred
    return dict(adv=adv, group_mean=mean, group_std=std, group_size=size)


# --------------------------------------------------------------------------------------------
# O6: turn-level credit assignment  (R31)
# --------------------------------------------------------------------------------------------
def turn_returns(seg_offsets, seg_source, seg_agent, turn_offsets, turn_rewards, group_id, gamma: float = 1.0,
                 train_agent: int = ANY_AGENT, traj_agent=None):
    """Per-segment reward-to-go of the trainable ACTION turns.

    "rewards are associated with the corresponding action tokens": the k-th trainable
    ACTION segment of trajectory b (source ACTION, emitted by the agent trained on b; k = 0, 1, ...
    in segment order) is turn k, and its return is the discounted reward-to-go over b's per-turn
    scores r_{b,0..R_b-1} (SPEC.md:95 stores scores per turn; SPEC.md:364 lists discounting as the
    extension):   G_{b,k} = sum_{j=k}^{R_b-1} gamma^(j-k) r_{b,j}   (0 when k >= R_b).
    Returns seg_return[S] (0 for other segments) and seg_group[S] = group_id[b] for a turn, -1
    otherwise — the input of group_advantages(..., skip_ungrouped=True).
    """
    seg_offsets = np.asarray(seg_offsets)
    B = len(seg_offsets) - 1
    S = int(seg_offsets[B])
    seg_return = np.zeros(S)
    seg_group = np.full(S, -1, np.int32)
    for b in range(B):
        ta = int(traj_agent[b]) if traj_agent is not None else int(train_agent)
        r = [float(x) for x in turn_rewards[int(turn_offsets[b]):int(turn_offsets[b + 1])]]
        k = 0
        for s in range(int(seg_offsets[b]), int(seg_offsets[b + 1])):
            if int(seg_source[s]) == ACTION and (ta == ANY_AGENT or int(seg_agent[s]) == ta):
                seg_return[s] = math.fsum(gamma ** (j - k) * r[j] for j in range(k, len(r)))
                seg_group[s] = int(group_id[b])
                k += 1
    return seg_return, seg_group


def turn_level_advantages(tb_masks_row_seg, seg_return, seg_group, num_groups: int, **kw):
    """Row advantages of turn-level credit: A of the row's segment (group-normalised over the group's
    turns by group_advantages), i.e. the turn's advantage broadcast over its ACTION tokens."""
    adv_seg = group_advantages(seg_group, seg_return, num_groups, skip_ungrouped=True, **kw)["adv"]
    row_seg = np.asarray(tb_masks_row_seg)
    return adv_seg, np.where(row_seg >= 0, adv_seg[np.maximum(row_seg, 0)], 0.0)


# --------------------------------------------------------------------------------------------
# O3: per-row log-softmax + gather + entropy  (north_star (3))
# --------------------------------------------------------------------------------------------
def row_forward(x, y: int, logit_scale: float = 1.0):
    """z = s*x;  M = max z;  S = sum exp(z-M);  lse = M + ln S;  logp = z_y - lse;
    H = ln S - sum exp(z-M)(z-M) / S   (terms with exp(z-M) == 0 contribute 0).
    Returns (logp, H, lse, p) with p = exp(z - lse)."""
    z = float(logit_scale) * np.asarray(x, np.float64)
    V = z.shape[0]
    if not (0 <= y < V):
        raise TargetRange(f"target {y} outside [0, {V})")
    M = float(np.max(z))
    e = np.exp(z - M)
    S = math.fsum(e)
    lse = M + math.log(S)
    logp = float(z[y]) - lse
    nz = e > 0
    H = math.log(S) - math.fsum(e[nz] * (z[nz] - M)) / S
    p = np.exp(z - lse)
    return logp, H, lse, p


def logprob_entropy_fwd(logits, targets, row_mask=None, logit_scale: float = 1.0):
    """Rows with row_mask == 0 are skipped and reported as 0 (R26)."""
    logits = np.asarray(logits, np.float64)
    N = logits.shape[0]
    logp, H, lse = np.zeros(N), np.zeros(N), np.zeros(N)
    for j in range(N):
        if row_mask is not None and not row_mask[j]:
            continue
        logp[j], H[j], lse[j], _ = row_forward(logits[j], int(targets[j]), logit_scale)
    return dict(logp=logp, entropy=H, lse=lse)


# --------------------------------------------------------------------------------------------
# O4: PPO-clip + KL surrogate, token-mean, fused backward  (north_star (4))
# --------------------------------------------------------------------------------------------
TOKEN_MEAN, SEQ_MEAN_TOKEN_MEAN, SEQ_MEAN_TOKEN_SUM = 0, 1, 2


@dataclass
class LossCfg:
    clip_low: float = 0.2          # epsilon_low  (R14)
    clip_high: float = 0.2         # epsilon_high
    kl_beta: float = 0.04          # beta (R16); 0 => no KL term, ref unused
    kl_type: int = KL_K3
    log_ratio_clamp: float = 20.0  # C (R15)
    logit_scale: float = 1.0       # s = 1/temperature (R19)
    # A4 variants (R27-R30)
    ent_coef: float = 0.0          # entropy bonus c_H: L -= c_H * H
    dual_clip: float = 0.0         # c > 1 caps the loss of A < 0 tokens at -c*A (0 = off)
    sft: bool = False              # supervised mode: L = -logp, ignores A / old / clip
    reduction: int = TOKEN_MEAN    # TOKEN_MEAN | SEQ_MEAN_TOKEN_MEAN | SEQ_MEAN_TOKEN_SUM


def row_loss_terms(logp: float, old: float, ref: Optional[float], A: float, cfg: LossCfg):
    """Per-token surrogate L = pg + beta*KL and its derivative G = dL/dlogp.

    delta = clamp(logp - old, -C, C); r = exp(delta); rbar = min(max(r, 1-eps_lo), 1+eps_hi)
    pg = max(-A*r, -A*rbar); clipped <=> (A>0 and r>1+eps_hi) or (A<0 and r<1-eps_lo)
    dpg/dlogp = 0 if clipped or |logp-old| > C else -A*r
    dual clip (c > 1, A < 0): pg <- min(pg, -c*A), zero gradient where the cap is active
    sft: pg = -logp, dpg/dlogp = -1 (A, old and the clip are not used)
    k3: d = clamp(ref - logp, -C, C); KL = exp(d) - d - 1; dKL/dlogp = 0 if |ref-logp| > C else 1 - exp(d)
    k1: KL = logp - ref, dKL/dlogp = 1;   k2: KL = (logp-ref)^2/2, dKL/dlogp = logp - ref
    Returns (L, G, clipped, KL). The entropy bonus (-c_H * H) is added by the caller: it depends on the
    whole row, not on logp alone.
    """
    C = cfg.log_ratio_clamp
    clipped = False
    if cfg.sft:
        pg = -logp
        G = -1.0
    else:
        draw = logp - old
        delta = min(max(draw, -C), C)
        r = math.exp(delta)
        rbar = min(max(r, 1.0 - cfg.clip_low), 1.0 + cfg.clip_high)
        pg = max(-A * r, -A * rbar)
        clipped = (A > 0 and r > 1.0 + cfg.clip_high) or (A < 0 and r < 1.0 - cfg.clip_low)
        G = 0.0 if (clipped or abs(draw) > C) else -A * r
        if cfg.dual_clip > 0.0 and A < 0 and pg > -cfg.dual_clip * A:
            pg = -cfg.dual_clip * A
            G = 0.0
    kl = 0.0
    if cfg.kl_beta != 0.0:
        if cfg.kl_type == KL_K3:
            dr = ref - logp
            d = min(max(dr, -C), C)
            kl = math.exp(d) - d - 1.0
            Gk = 0.0 if abs(dr) > C else 1.0 - math.exp(d)
        elif cfg.kl_type == KL_K1:
            kl = logp - ref
            Gk = 1.0
        elif cfg.kl_type == KL_K2:
            kl = 0.5 * (logp - ref) ** 2
            Gk = logp - ref
        else:
            raise ValueError("kl_type")
        G += cfg.kl_beta * Gk
    L = pg + cfg.kl_beta * kl
    return L, G, bool(clipped), kl


def row_weights(loss_mask, row_traj, reduction: int, n_loss: int, traj_tokens=None, n_active=None):
    """w_j of loss = sum_j w_j L_j (R17, R29):
    token-mean: m_j / N; seq-mean-token-mean: m_j / (n_b * B_eff); seq-mean-token-sum: m_j / B_eff, with
    n_b the loss tokens of row j's trajectory and B_eff the trajectories with n_b > 0 (global values may be
    passed for sharded batches). Any zero denominator gives weight 0."""
    loss_mask = np.asarray(loss_mask)
    row_traj = np.asarray(row_traj)
    if reduction == TOKEN_MEAN:
        return np.where(loss_mask != 0, (1.0 / n_loss) if n_loss > 0 else 0.0, 0.0)
    if traj_tokens is None:
        traj_tokens = np.bincount(row_traj[loss_mask != 0], minlength=int(row_traj.max()) + 1)
    if n_active is None:
        n_active = int(np.count_nonzero(traj_tokens))
    w = np.zeros(len(loss_mask))
    for j in range(len(loss_mask)):
        if loss_mask[j] and n_active > 0:
            nb = traj_tokens[row_traj[j]]
            w[j] = 1.0 / (nb * n_active) if reduction == SEQ_MEAN_TOKEN_MEAN else 1.0 / n_active
    return w


def policy_loss_fwd_bwd(logits, targets, loss_mask, row_traj, adv, old_logp, ref_logp, n_loss: int,
                        cfg: LossCfg = LossCfg(), zero_masked_rows: bool = True,
                        rows: Optional[Sequence[int]] = None, traj_tokens=None, n_active=None, adv_index=None):
    """loss = sum_j w_j L_j with L_j = pg + beta*KL - c_H*H_j and w_j from row_weights (token-mean: m_j/N;
    N = n_loss, the global loss-token count; 0 => loss 0, grads 0)
    dlogits[j, v] = coef_j * (p_jv - [v == y_j]) + w_j c_H s p_jv (ln p_jv + H_j),  coef_j = -s * w_j * G_j
    (dH/dz_v = -p_v (ln p_v + H); z = s x).

    `rows` restricts the per-row outputs to a subset (sampled parity at full size); the loss and
    stats are then sums over that subset only. Rows with m_j == 0 get dlogits 0, logp 0, entropy 0.
    adv_index (turn-level credit, O6): A_j = adv[adv_index[j]] (the row's segment) instead of adv[row_traj[j]].
    """
    logits_is_array = not callable(logits)
    N_rows = len(targets)
    rows = range(N_rows) if rows is None else rows
    s = cfg.logit_scale
    W = row_weights(loss_mask, row_traj, cfg.reduction, n_loss, traj_tokens, n_active)
    out_dl, out_logp, out_H, out_coef = {}, {}, {}, {}
    terms, klterms, Hterms = [], [], []
    n_clipped = 0
    n_tok = 0
    for j in rows:
        x = logits[j] if logits_is_array else logits(j)
        m = int(loss_mask[j])
        if not m:
            out_dl[j] = np.zeros(len(x)) if zero_masked_rows else None
            out_logp[j], out_H[j], out_coef[j] = 0.0, 0.0, 0.0
            continue
        y = int(targets[j])
        logp, H, lse, p = row_forward(x, y, s)
        A = float(adv[int(row_traj[j]) if adv_index is None else int(adv_index[j])])
        ref = float(ref_logp[j]) if ref_logp is not None else None
        L, G, clipped, kl = row_loss_terms(logp, float(old_logp[j]), ref, A, cfg)
        L -= cfg.ent_coef * H
        w = float(W[j])
        coef = -s * w * G
        dl = coef * p
        dl[y] = coef * (p[y] - 1.0)
        if cfg.ent_coef != 0.0:
            with np.errstate(divide="ignore", invalid="ignore"):
                lnp = np.where(p > 0, np.log(np.where(p > 0, p, 1.0)), 0.0)
            dl = dl + w * cfg.ent_coef * s * p * (lnp + H)
        out_dl[j], out_logp[j], out_H[j], out_coef[j] = dl, logp, H, coef
        terms.append(w * L); klterms.append(kl); Hterms.append(H)
        n_clipped += int(clipped)
        n_tok += 1
    loss = math.fsum(terms)
    stats = dict(loss=loss, n_clipped=n_clipped, kl_sum=math.fsum(klterms),
                 entropy_sum=math.fsum(Hterms), n_tokens=n_tok)
    if logits_is_array and rows == range(N_rows):
        dl = np.stack([out_dl[j] for j in range(N_rows)]) if zero_masked_rows else None
        return dict(loss=loss, dlogits=dl, logp=np.array([out_logp[j] for j in range(N_rows)]),
                    entropy=np.array([out_H[j] for j in range(N_rows)]),
                    coef=np.array([out_coef[j] for j in range(N_rows)]), stats=stats)
    return dict(loss=loss, dlogits=out_dl, logp=out_logp, entropy=out_H, coef=out_coef, stats=stats)


def loss_only(logits, targets, loss_mask, row_traj, adv, old_logp, ref_logp, n_loss, cfg=LossCfg()):
    """The scalar loss alone (used by the finite-difference pin)."""
    s = cfg.logit_scale
    W = row_weights(loss_mask, row_traj, cfg.reduction, n_loss)
    terms = []
    for j in range(len(targets)):
        if not loss_mask[j]:
            continue
        logp, H, _, _ = row_forward(logits[j], int(targets[j]), s)
        ref = float(ref_logp[j]) if ref_logp is not None else None
        L, _, _, _ = row_loss_terms(logp, float(old_logp[j]), ref, float(adv[int(row_traj[j])]), cfg)
        terms.append(W[j] * (L - cfg.ent_coef * H))
    return math.fsum(terms)


# --------------------------------------------------------------------------------------------
# O5: vocab-sharded forward (north_star: vocab-sharding with all-reduced row max / sum-exp)
# --------------------------------------------------------------------------------------------
def shard_partials(x_shard, y: int, vocab_start: int, logit_scale: float = 1.0):
    """Partials of one vocab shard [vocab_start, vocab_start + len): (m, s, t, zy) with
    m = max z, s = sum exp(z-m), t = sum exp(z-m)(z-m), zy = z_y if y in the shard else 0."""
    z = float(logit_scale) * np.asarray(x_shard, np.float64)
    if z.shape[0] == 0:
        return (-math.inf, 0.0, 0.0, 0.0)
    m = float(np.max(z))
    if m == -math.inf:                      # every entry -inf: the shard holds no probability mass
        return (-math.inf, 0.0, 0.0, 0.0)
    e = np.exp(z - m)
    nz = e > 0
    s = math.fsum(e)
    t = math.fsum(e[nz] * (z[nz] - m))
    zy = float(z[y - vocab_start]) if vocab_start <= y < vocab_start + z.shape[0] else 0.0
    return (m, s, t, zy)


def combine_partials(parts):
    """M = max m_p; S = sum s_p e^{m_p-M}; T = sum e^{m_p-M}(t_p + (m_p-M) s_p);
    lse = M + ln S; H = ln S - T/S; logp = sum zy_p - lse.   Returns (logp, H, lse)."""
    M = max(p[0] for p in parts)
    w = [math.exp(p[0] - M) if p[0] != -math.inf else 0.0 for p in parts]
    S = math.fsum(wi * p[1] for wi, p in zip(w, parts))
    T = math.fsum(wi * (p[2] + (p[0] - M) * p[1]) for wi, p in zip(w, parts) if wi > 0)
    lse = M + math.log(S)
    H = math.log(S) - T / S
    logp = math.fsum(p[3] for p in parts) - lse
    return logp, H, lse


# --------------------------------------------------------------------------------------------
# O7: rollout-side token sampling (PAPER.md:170-171 GENERATING)
# --------------------------------------------------------------------------------------------
def sample_token(x, u: float, logit_scale: float = 1.0, greedy: bool = False):
    """One generated token from a row of logits (R32).

    sample ("samples from softmax(logits/temperature)"): inverse transform with the
    caller's uniform u in [0, 1): t = min{ t : sum_{v <= t} p_v > u }, p = softmax(s x), s = 1/temperature.
    greedy (SPEC.md:309-318 greedy_token; also the temperature < 1e-6 limit of SPEC.md:305): the argmax
    of the logits, ties to the lowest token id. Returns (t, log p_t) with p the softmax(s x) distribution.
    """
    z = float(logit_scale) * np.asarray(x, np.float64)
    M = float(np.max(z))
    e = np.exp(z - M)
    S = math.fsum(e)
    if greedy:
        t = int(np.argmax(np.asarray(x, np.float64)))          # first maximal index
    else:
        cdf = np.cumsum(e / S)
        t = int(np.searchsorted(cdf, u, side="right"))           # first t with cdf_t > u
        if t >= len(z):                                           # u beyond the rounded total mass
            t = int(np.flatnonzero(e > 0)[-1])
    return t, float(z[t]) - (M + math.log(S))


def sample_tokens(logits, u, logit_scale: float = 1.0, greedy: bool = False):
    logits = np.asarray(logits, np.float64)
    out = [sample_token(logits[j], float(u[j]) if u is not None else 0.0, logit_scale, greedy)
           for j in range(logits.shape[0])]
    return np.array([t for t, _ in out], np.int32), np.array([lp for _, lp in out])


# --------------------------------------------------------------------------------------------
# O8: LM head fused with O3 (PAPER.md:188 fwd pool; R33)
# --------------------------------------------------------------------------------------------
def lmhead_logprob_fwd(hidden, weight, targets, logit_scale: float = 1.0, rows=None):
    """z_j = s * h_j W^T (float64 matmul of the given values), then O3 row_forward on z_j.
    Returns dict(logp, entropy, lse) over `rows` (default all)."""
    h = np.asarray(hidden, np.float64)
    W = np.asarray(weight, np.float64)
    rows = range(h.shape[0]) if rows is None else rows
    out = {}
    for j in rows:
        z = W @ h[j]
        lp, H, lse, _ = row_forward(z, int(targets[j]), logit_scale)
        out[j] = (lp, H, lse)
    return dict(logp={j: v[0] for j, v in out.items()}, entropy={j: v[1] for j, v in out.items()},
                lse={j: v[2] for j, v in out.items()})
