"""One training step of the hot path (north_star (1)-(4)) over one batch of trajectories.

Sequences the C-ABI calls and, when a torch.distributed process group is given (batch sharding,
DESIGN.md §7), the exchanges between them:

  otk_build_masks            -> all_reduce(n_loss, SUM)            global token count (R17)
  otk_group_advantages       -> all_gather(group_id, return)       cross-shard group statistics;
     (local returns)            otk_group_advantages (global)      every rank computes identical stats
  otk_policy_loss_fwd_bwd x M micro-batches (stats accumulated on the device)
                             -> all_reduce(stats, SUM)             global loss on every rank

Turn-level credit (credit="turn", NEXT-2): otk_build_masks also writes row_seg; otk_turn_returns gives
the reward-to-go of every trainable ACTION turn (per segment), all_gather(seg_group, seg_return) when
batch-sharded, otk_group_advantages(skip_ungrouped) over the segments; the loss reads A by row_seg.

Vocab sharding (VocabShard): every rank holds all rows and a column range; per micro-batch
  otk_row_partials -> all_gather(16 B / row) -> otk_policy_loss_fwd_bwd_partials (identical stats on all ranks).
Fused vocab sharding (VocabShardFused, K4-VPF): one otk_policy_loss_fwd_bwd_vpf per micro-batch; the 16-byte
row partials travel between the ranks' kernels over peer memory (no collective call, one read of the shard).

No host synchronisation inside a step (n_loss and the stats never leave the device), so a step can be
captured in a CUDA graph. Everything arithmetic happens in libotk's kernels; this module only moves
pointers and calls collectives.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Tuple

import torch

from . import (Context, DeviceTrajBatch, LossCfg, STATS_FIELDS, otk_build_masks, otk_group_advantages,
               otk_batch_allreduce_f64, otk_batch_allreduce_i64, otk_batch_group_advantages, otk_comm_size,
               otk_logprob_entropy_combine, otk_policy_loss_fwd_bwd, otk_policy_loss_fwd_bwd_partials,
               otk_lmhead_row_partials, otk_policy_loss_fwd_bwd_vpf, otk_row_partials, otk_turn_returns,
               VpfExchange)


@dataclass
class MicroBatch:
    """Row range [r0, r1) of the step and the tensors the loss call reads for it."""
    r0: int
    r1: int
    logits: torch.Tensor            # [r1 - r0, ld]
    targets: torch.Tensor           # [r1 - r0] int32
    old_logp: torch.Tensor          # [r1 - r0] f32
    ref_logp: Optional[torch.Tensor]
    dlogits: torch.Tensor           # [r1 - r0, ld] output


class VocabShard:
    """(3) and (4) on a vocab shard [vocab_start, vocab_start + vocab_local) of every row:
    otk_row_partials (16 B per row) -> all_gather in rank order -> exact combine / streaming pass 2.
    Every rank ends with the same logp, entropy and loss statistics."""

    def __init__(self, ctx: Context, vocab_start: int, vocab_local: int, vocab_total: int, process_group=None):
        self.ctx, self.v0, self.vl, self.vt, self.pg = ctx, vocab_start, vocab_local, vocab_total, process_group

    def _gather(self, partials):
        if self.pg is None:
            return partials.unsqueeze(0)
        from .dist import all_gather_vocab_partials
        return all_gather_vocab_partials(partials, self.pg)

    def forward(self, logits: torch.Tensor, targets: torch.Tensor, row_mask=None, logit_scale: float = 1.0):
        part = otk_row_partials(self.ctx, logits, targets, self.v0, self.vt, vocab_local=self.vl, row_mask=row_mask,
                                logit_scale=logit_scale)
        return otk_logprob_entropy_combine(self.ctx, self._gather(part), row_mask=row_mask)

    def loss(self, logits, targets, loss_mask, row_traj, adv, old_logp, ref_logp, n_loss, cfg: LossCfg, *,
             dlogits=None, stats=None, accumulate=None):
        part = otk_row_partials(self.ctx, logits, targets, self.v0, self.vt, vocab_local=self.vl, row_mask=loss_mask,
                                logit_scale=cfg.logit_scale)
        return otk_policy_loss_fwd_bwd_partials(self.ctx, logits, targets, loss_mask, row_traj, adv, old_logp,
                                                ref_logp, n_loss, cfg, self.v0, self.vt, self._gather(part),
                                                vocab_local=self.vl, dlogits=dlogits, stats=stats,
                                                accumulate=accumulate)


class VocabShardFused(VocabShard):
    """VocabShard whose loss runs as K4-VPF (otk_policy_loss_fwd_bwd_vpf): the exchange of row partials is
    inside the kernel, over the VpfExchange's peer-mapped buffers (dist.open_vpf_exchange across processes,
    VpfExchange.local_group for ranks sharing one process). Same results as VocabShard (logp / entropy / stats
    bitwise equal). forward() is inherited (its exchange is the all-gather)."""

    def __init__(self, ctx: Context, vocab_start: int, vocab_local: int, vocab_total: int, xchg: VpfExchange,
                 process_group=None):
        super().__init__(ctx, vocab_start, vocab_local, vocab_total, process_group)
        self.xchg = xchg

    def loss(self, logits, targets, loss_mask, row_traj, adv, old_logp, ref_logp, n_loss, cfg: LossCfg, *,
             dlogits=None, stats=None, accumulate=None, stream=None):
        return otk_policy_loss_fwd_bwd_vpf(self.ctx, logits, targets, loss_mask, row_traj, adv, old_logp, ref_logp,
                                           n_loss, cfg, self.v0, self.vt, self.xchg, dlogits=dlogits, stats=stats,
                                           accumulate=accumulate, stream=stream)


class LMHeadVocabShard:
    """Tensor-parallel fused LM head (NEXT-1 forward): this rank holds rows [vocab_start, vocab_start +
    vocab_local) of W; otk_lmhead_row_partials (16 B per row) -> all_gather in rank order -> exact combine.
    Every rank ends with the same logp / entropy; the [N, V] logits exist nowhere."""

    def __init__(self, ctx: Context, vocab_start: int, vocab_total: int, process_group=None):
        self.ctx, self.v0, self.vt, self.pg = ctx, vocab_start, vocab_total, process_group
        self.workspace = None

    def forward(self, hidden: torch.Tensor, weight_shard: torch.Tensor, targets: torch.Tensor, row_mask=None,
                logit_scale: float = 1.0):
        part, self.workspace = otk_lmhead_row_partials(self.ctx, hidden, weight_shard, targets, self.v0, self.vt,
                                                       row_mask=row_mask, logit_scale=logit_scale,
                                                       workspace=self.workspace)
        if self.pg is None:
            gathered = part.unsqueeze(0)
        else:
            from .dist import all_gather_vocab_partials
            gathered = all_gather_vocab_partials(part, self.pg)
        return otk_logprob_entropy_combine(self.ctx, gathered, row_mask=row_mask)


class PolicyLossStep:
    def __init__(self, ctx: Context, batch: DeviceTrajBatch, group_id: torch.Tensor, num_groups: int,
                 turn_offsets: torch.Tensor, turn_rewards: torch.Tensor, vocab: int, cfg: LossCfg = LossCfg(), *,
                 train_agent: int = -1, std_norm: bool = True, unbiased: bool = False,
                 process_group=None, global_num_traj: Optional[Sequence[int]] = None,
                 global_num_groups: Optional[int] = None, vocab_shard: Optional[VocabShard] = None,
                 credit: str = "trajectory", gamma: float = 1.0,
                 global_num_segments: Optional[Sequence[int]] = None, collectives: str = "torch"):
        """process_group: batch sharding (this rank's trajectories; exchanges below). vocab_shard: vocab
        sharding (the rank holds a column range of the logits of its rows). Both: 2-D sharding — process_group
        is then the rank's batch group (same columns, other trajectories) and vocab_shard's group its vocab
        group (same rows, other columns); dist.make_2d_groups builds them.
        credit: "trajectory" (north_star (2): one A per trajectory) or "turn" (NEXT-2, R31: the
        discounted reward-to-go of each trainable ACTION turn, group-normalised over the group's turns,
        read per row through the row's segment). global_num_segments: per-rank segment counts (batch
        sharding with turn credit; default: every rank has this rank's count).
        collectives: who runs batch sharding's three exchanges — "torch" (torch.distributed on process_group) or
        "otk" (the library's own NCCL communicator on ctx, otk_comm_init: the C-ABI path a non-Python caller
        uses; process_group is then not needed)."""
        self.vshard = vocab_shard
        self.ctx, self.batch, self.cfg, self.vocab = ctx, batch, cfg, vocab   # (cfg may gain count pointers)
        self.group_id, self.num_groups = group_id, num_groups
        self.turn_offsets, self.turn_rewards = turn_offsets, turn_rewards
        self.train_agent, self.std_norm, self.unbiased = train_agent, std_norm, unbiased
        self.pg = process_group
        if collectives not in ("torch", "otk"):
            raise ValueError(f"collectives must be 'torch' or 'otk', not {collectives!r}")
        self.coll = collectives
        self.sharded = process_group is not None or collectives == "otk"
        if credit not in ("trajectory", "turn"):
            raise ValueError(f"credit must be 'trajectory' or 'turn', not {credit!r}")
        self.credit, self.gamma = credit, float(gamma)
        dev = batch.tok_offsets.device
        N, B = batch.num_rows, batch.num_traj
        S = int(batch.seg_len.numel())
        self.S = S
        self.masks = dict(loss_mask=torch.empty(N, dtype=torch.uint8, device=dev),
                          row_traj=torch.empty(N, dtype=torch.int32, device=dev),
                          traj_loss_tokens=torch.empty(B, dtype=torch.int64, device=dev),
                          n_loss=torch.empty(1, dtype=torch.int64, device=dev),
                          n_active_traj=torch.empty(1, dtype=torch.int64, device=dev))
        E = B
        if credit == "turn":     # advantages live on segments; rows find theirs through row_seg
            self.masks["row_seg"] = torch.empty(N, dtype=torch.int32, device=dev)
            self.turn_out = dict(seg_return=torch.empty(S, dtype=torch.float64, device=dev),
                                 seg_group=torch.empty(S, dtype=torch.int32, device=dev))
            E = S
        if cfg.reduction != 0:   # sequence-mean reductions read the per-trajectory token counts (R29)
            self.cfg = dataclasses.replace(cfg, traj_loss_tokens=self.masks["traj_loss_tokens"],
                                           n_active_traj=self.masks["n_active_traj"])
        G_loc = global_num_groups if (self.sharded and global_num_groups) else num_groups
        self.adv_out = dict(adv=torch.empty(E, dtype=torch.float64, device=dev),
                            returns=torch.empty(E, dtype=torch.float64, device=dev),
                            group_mean=torch.empty(G_loc, dtype=torch.float64, device=dev),
                            group_std=torch.empty(G_loc, dtype=torch.float64, device=dev),
                            group_size=torch.empty(G_loc, dtype=torch.int32, device=dev))
        self.stats = torch.zeros(len(STATS_FIELDS), dtype=torch.float64, device=dev)
        if self.sharded:
            if self.coll == "otk":
                self.world, self.rank = otk_comm_size(ctx)
            else:
                import torch.distributed as dist
                self.world = dist.get_world_size(self.pg)
                self.rank = dist.get_rank(self.pg)
            counts = list(global_num_traj) if global_num_traj is not None else [B] * self.world
            if credit == "turn":
                counts = list(global_num_segments) if global_num_segments is not None else [S] * self.world
            self.counts = counts
            self.b0 = sum(counts[:self.rank])
            self.E = E
            self.Bmax = max(counts)
            self.G_global = global_num_groups if global_num_groups is not None else num_groups
            Bg = sum(counts)
            self.gid_g = torch.empty(Bg, dtype=torch.int32, device=dev)
            self.ret_g = torch.empty(Bg, dtype=torch.float64, device=dev)
            self.adv_g = dict(adv=torch.empty(Bg, dtype=torch.float64, device=dev),
                              returns=torch.empty(Bg, dtype=torch.float64, device=dev),
                              group_mean=torch.empty(self.G_global, dtype=torch.float64, device=dev),
                              group_std=torch.empty(self.G_global, dtype=torch.float64, device=dev),
                              group_size=torch.empty(self.G_global, dtype=torch.int32, device=dev))

    # -- (1) + (2) --------------------------------------------------------------------------------
    def masks_and_advantages(self):
        """Steps (1) + (2). Returns the advantage array the loss indexes: per trajectory (row_traj), or per
        segment (row_seg) with credit="turn"."""
        otk_build_masks(self.ctx, self.batch, self.train_agent, response_mask=False, source_counts=False,
                        row_seg=self.credit == "turn", out=self.masks)
        if self.credit == "turn":
            return self._turn_advantages()
        if not self.sharded:
            otk_group_advantages(self.ctx, self.group_id, self.num_groups, turn_offsets=self.turn_offsets,
                                 turn_rewards=self.turn_rewards, std_norm=self.std_norm, unbiased=self.unbiased,
                                 out=self.adv_out)
            return self.adv_out["adv"]
        if self.coll == "otk":
            self._otk_counts()
            otk_group_advantages(self.ctx, self.group_id, self.G_global, turn_offsets=self.turn_offsets,
                                 turn_rewards=self.turn_rewards, out=self.adv_out)
            return self._otk_group_advantages(self.group_id, self.adv_out["returns"], False)
        from .dist import all_gather_group_returns, all_reduce_n_loss
        all_reduce_n_loss(self.masks["n_loss"], self.pg)
        if self.cfg.reduction != 0:
            all_reduce_n_loss(self.masks["n_active_traj"], self.pg)
        # local returns (group statistics of this call are discarded; ids are global), then the exchange
        otk_group_advantages(self.ctx, self.group_id, self.G_global, turn_offsets=self.turn_offsets,
                             turn_rewards=self.turn_rewards, out=self.adv_out)
        all_gather_group_returns(self.group_id, self.adv_out["returns"], self.counts, self.pg,
                                 out=(self.gid_g, self.ret_g))
        otk_group_advantages(self.ctx, self.gid_g, self.G_global, returns=self.ret_g, std_norm=self.std_norm,
                             unbiased=self.unbiased, out=self.adv_g)
        return self.adv_g["adv"][self.b0:self.b0 + self.batch.num_traj]

    def _turn_advantages(self):
        otk_turn_returns(self.ctx, self.batch, self.S, self.group_id, self.turn_offsets, self.turn_rewards,
                         self.gamma, self.train_agent, out=self.turn_out)
        seg_group, seg_return = self.turn_out["seg_group"], self.turn_out["seg_return"]
        if not self.sharded:
            otk_group_advantages(self.ctx, seg_group, self.num_groups, returns=seg_return, std_norm=self.std_norm,
                                 unbiased=self.unbiased, skip_ungrouped=True, out=self.adv_out)
            return self.adv_out["adv"]
        if self.coll == "otk":
            self._otk_counts()
            return self._otk_group_advantages(seg_group, seg_return, True)
        from .dist import all_gather_group_returns, all_reduce_n_loss
        all_reduce_n_loss(self.masks["n_loss"], self.pg)
        if self.cfg.reduction != 0:
            all_reduce_n_loss(self.masks["n_active_traj"], self.pg)
        all_gather_group_returns(seg_group, seg_return, self.counts, self.pg, out=(self.gid_g, self.ret_g))
        otk_group_advantages(self.ctx, self.gid_g, self.G_global, returns=self.ret_g, std_norm=self.std_norm,
                             unbiased=self.unbiased, skip_ungrouped=True, out=self.adv_g)
        return self.adv_g["adv"][self.b0:self.b0 + self.E]

    def _otk_counts(self):   # exchange (1): global token / trajectory counts over the ctx's NCCL communicator
        otk_batch_allreduce_i64(self.ctx, self.masks["n_loss"])
        if self.cfg.reduction != 0:
            otk_batch_allreduce_i64(self.ctx, self.masks["n_active_traj"])

    def _otk_group_advantages(self, gid, ret, skip_ungrouped):   # exchange (2) + step (2) on the whole batch
        o = otk_batch_group_advantages(self.ctx, gid, ret, self.counts, self.G_global, std_norm=self.std_norm,
                                       unbiased=self.unbiased, skip_ungrouped=skip_ungrouped,
                                       out=dict(gid_all=self.gid_g, ret_all=self.ret_g, adv_all=self.adv_g["adv"],
                                                group_mean=self.adv_g["group_mean"],
                                                group_std=self.adv_g["group_std"],
                                                group_size=self.adv_g["group_size"]))
        return o["adv"]

    # -- (3) + (4) --------------------------------------------------------------------------------
    def loss(self, adv: torch.Tensor, micro_batches: Sequence[MicroBatch],
             on_launch: Optional[Callable[[int, str], None]] = None):
        for k, mb in enumerate(micro_batches):
            if on_launch:
                on_launch(k, "begin")
            cfg = self.cfg
            if self.credit == "turn":
                cfg = dataclasses.replace(cfg, adv_index=self.masks["row_seg"][mb.r0:mb.r1])
            if self.vshard is not None:
                self.vshard.loss(mb.logits, mb.targets, self.masks["loss_mask"][mb.r0:mb.r1],
                                 self.masks["row_traj"][mb.r0:mb.r1], adv, mb.old_logp, mb.ref_logp,
                                 self.masks["n_loss"], cfg, dlogits=mb.dlogits, stats=self.stats,
                                 accumulate=k > 0)
            else:
                otk_policy_loss_fwd_bwd(self.ctx, mb.logits, mb.targets, self.masks["loss_mask"][mb.r0:mb.r1],
                                        self.masks["row_traj"][mb.r0:mb.r1], adv, mb.old_logp, mb.ref_logp,
                                        self.masks["n_loss"], cfg, vocab=self.vocab, dlogits=mb.dlogits,
                                        stats=self.stats, accumulate=k > 0, want_logp=False)
            if on_launch:
                on_launch(k, "end")
        if self.sharded and self.coll == "otk":
            otk_batch_allreduce_f64(self.ctx, self.stats)   # exchange (3)
        elif self.sharded:
            from .dist import all_reduce_stats
            all_reduce_stats(self.stats, self.pg)
        return self.stats

    def run(self, micro_batches: Sequence[MicroBatch], on_launch=None):
        adv = self.masks_and_advantages()
        self.adv_used = adv          # the advantages this step's loss read (this rank's part under sharding)
        return self.loss(adv, micro_batches, on_launch)


class LMHeadPolicyLoss:
    """The policy loss and its gradients THROUGH the LM head (backward half, unfused
    form): x = h Wᵀ (bf16 tensor-core GEMM, cuBLAS through torch — a plain library GEMM), then
    (4) on x with cfg.logit_scale = s (otk_policy_loss_fwd_bwd: loss, stats and dx = dL/dx in one pass over x),
    then dh = dx W and dW = dxᵀ h (cuBLAS). The fused alternative that never stores x needs x recomputed in the
    backward — a fourth GEMM — which costs more than the traffic it saves at Qwen-class hidden sizes
    (DESIGN.md §10); `timings=True` returns the measured split. x and dx buffers are reused across calls."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        self._x = self._dx = None

    def __call__(self, hidden: torch.Tensor, weight: torch.Tensor, targets, loss_mask, row_traj, adv, old_logp,
                 ref_logp, n_loss, cfg: LossCfg, *, timings: bool = False) -> dict:
        N, d = hidden.shape
        V = weight.shape[0]
        if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16 or weight.shape[1] != d:
            raise ValueError("hidden [N, d] and weight [V, d] must be bfloat16")
        if self._x is None or self._x.shape != (N, V):
            self._x = torch.empty((N, V), dtype=torch.bfloat16, device=hidden.device)
            self._dx = torch.empty_like(self._x)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timings else None
        if ev:
            ev[0].record()
        torch.matmul(hidden, weight.t(), out=self._x)
        if ev:
            ev[1].record()
        out = otk_policy_loss_fwd_bwd(self.ctx, self._x, targets, loss_mask, row_traj, adv, old_logp, ref_logp,
                                      n_loss, cfg, dlogits=self._dx)
        if ev:
            ev[2].record()
        dh = torch.matmul(self._dx, weight)
        dW = torch.matmul(self._dx.t(), hidden)
        out.update(dh=dh, dW=dW)
        if ev:
            ev[3].record()
            torch.cuda.synchronize()
            out["ms"] = dict(logits_gemm=ev[0].elapsed_time(ev[1]), loss_kernel=ev[1].elapsed_time(ev[2]),
                             grad_gemms=ev[2].elapsed_time(ev[3]))
        return out


class LMHeadPolicyLossFused:
    """The policy loss and its gradients THROUGH the LM head on this library's tcgen05 kernels (SURVEY.md §8(f)
    NEXT-1, forward + backward; DESIGN.md §6 "LM head, backward"): one otk_lmhead_policy_loss_fwd_bwd call —
    x = h Wᵀ with the log-softmax partials folded in its epilogue (x kept as bf16), the loss terms of (4) per row,
    then dh = dx W and dW = dxᵀ h with dx formed tile by tile in shared memory from x (never written). Same
    arguments and outputs as LMHeadPolicyLoss; x and the workspace are reused across calls."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        self._bufs = {}

    def __call__(self, hidden: torch.Tensor, weight: torch.Tensor, targets, loss_mask, row_traj, adv, old_logp,
                 ref_logp, n_loss, cfg: LossCfg, *, timings: bool = False) -> dict:
        from . import otk_lmhead_policy_loss_fwd_bwd
        N, d = hidden.shape
        V = weight.shape[0]
        key = (N, V, d)
        if key not in self._bufs:
            self._bufs = {key: dict(workspace=None)}
        b = self._bufs[key]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if timings else None
        if ev:
            ev[0].record()
        out = otk_lmhead_policy_loss_fwd_bwd(self.ctx, hidden, weight, targets, loss_mask, row_traj, adv, old_logp,
                                             ref_logp, n_loss, cfg, workspace=b["workspace"])
        b["workspace"] = out["workspace"]
        if ev:
            ev[1].record()
            torch.cuda.synchronize()
            out["ms"] = dict(total=ev[0].elapsed_time(ev[1]))
        return out
