"""Host-side sharding logic and the collectives of the two multi-GPU modes.

torch.distributed is the plumbing (NCCL on the GPU box, gloo in the CPU tests); nothing here does the
method's arithmetic — the exchanged values are produced and consumed by libotk's kernels.

Batch sharding (north_star: "batch-sharding trajectories with an all-reduce of the global token count and
cross-shard group statistics"):
  * plan_batch_shards   contiguous trajectory ranges per rank, balanced by estimated HBM bytes
                        (4V per trainable row, 2V per masked row — SURVEY.md §8(d) unit costs)
  * all_reduce_n_loss   the token-mean denominator N is global (R17)
  * all_gather_group_returns  (group_id, return) of every trajectory, so each rank computes identical
                        group statistics over the global batch (groups may straddle ranks)
  * all_reduce_stats    loss statistics (each rank's loss is already divided by the global N)
Vocab sharding (north_star: "vocab-sharding logits with an all-reduce of row max and sum-exp"):
  * vocab_shard_bounds  column ranges, multiples of 8 columns (16-byte aligned rows)
  * all_gather_vocab_partials  16 bytes per row per rank: (max, sum-exp, sum-exp*d, z_y)
2-D (batch x vocab) sharding: world = Pb * Pv ranks, rank = b * Pv + v; rank (b, v) holds trajectory shard b
and vocab columns v. make_2d_groups builds the two families of subgroups: the batch exchanges above run inside
the vocab-column group (same v, all b), the per-row partial exchange inside the row group (same b, all v).
  * open_vpf_exchange   K4-VPF setup: every rank's exchange buffer mapped into every rank (CUDA IPC handles
                        all-gathered once); the per-row exchange itself then runs inside the loss kernel
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

ACTION, PAD = 1, 3


def traj_costs(tb, vocab: int, bytes_per_elem: int = 2, train_agent: int = -1) -> np.ndarray:
    """Estimated HBM bytes of the fused loss per trajectory: trainable rows read + write the V-wide row
    (4V bytes for bf16), every other row is only zero-filled (2V)."""
    B = len(tb.tok_offsets) - 1
    cost = np.zeros(B)
    for b in range(B):
        s0, s1 = int(tb.seg_offsets[b]), int(tb.seg_offsets[b + 1])
        ta = int(tb.traj_agent[b]) if getattr(tb, "traj_agent", None) is not None else train_agent
        n_rows = int(tb.tok_offsets[b + 1] - tb.tok_offsets[b])
        n_tr = sum(int(tb.seg_len[k]) for k in range(s0, s1)
                   if tb.seg_source[k] == ACTION and (ta == -1 or int(tb.seg_agent[k]) == ta))
        cost[b] = (n_tr * 2 + (n_rows - n_tr)) * vocab * bytes_per_elem
    return cost


def plan_batch_shards(costs: Sequence[float], world: int) -> List[Tuple[int, int]]:
    """Split trajectories [0, B) into `world` contiguous ranges with balanced total cost (greedy prefix
    split at the cost quantiles). Every rank gets at least one trajectory when B >= world."""
    c = np.asarray(costs, np.float64)
    B = len(c)
    if world < 1:
        raise ValueError("world >= 1")
    if B < world:
        raise ValueError("fewer trajectories than ranks")
    cum = np.concatenate([[0.0], np.cumsum(c)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        k = int(np.searchsorted(cum, target))
        # choose the closer of k-1 / k, keep strictly increasing and leave >= 1 per remaining rank
        if k > 0 and abs(cum[k - 1] - target) <= abs(cum[min(k, B)] - target):
            k -= 1
        k = max(k, bounds[-1] + 1)
        k = min(k, B - (world - r))
        bounds.append(k)
    bounds.append(B)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def vocab_shard_bounds(vocab: int, world: int, align: int = 8) -> List[Tuple[int, int]]:
    """Columns [v0, v1) of each rank; interior boundaries are multiples of `align` columns."""
    b = [0] + [min(vocab, (vocab * r // world) // align * align) for r in range(1, world)] + [vocab]
    return [(b[r], b[r + 1]) for r in range(world)]


def all_reduce_n_loss(n_loss: torch.Tensor, group=None) -> torch.Tensor:
    dist.all_reduce(n_loss, op=dist.ReduceOp.SUM, group=group)
    return n_loss


def all_reduce_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def all_gather_group_returns(group_id: torch.Tensor, returns: torch.Tensor, counts: Sequence[int],
                             group=None, out: Optional[Tuple[torch.Tensor, torch.Tensor]] = None):
    """Concatenate every rank's (group_id, return) in rank order. `counts` (trajectories per rank) is known
    on the host from the shard plan, so no size exchange (and no host sync) is needed."""
    world = dist.get_world_size(group)
    bmax = max(counts)
    dev = group_id.device
    pad_g = torch.zeros(bmax, dtype=group_id.dtype, device=dev)
    pad_r = torch.zeros(bmax, dtype=returns.dtype, device=dev)
    pad_g[:group_id.numel()].copy_(group_id)
    pad_r[:returns.numel()].copy_(returns)
    gg = torch.empty(world * bmax, dtype=group_id.dtype, device=dev)
    gr = torch.empty(world * bmax, dtype=returns.dtype, device=dev)
    dist.all_gather_into_tensor(gg, pad_g, group=group)
    dist.all_gather_into_tensor(gr, pad_r, group=group)
    total = sum(counts)
    if out is None:
        out = (torch.empty(total, dtype=group_id.dtype, device=dev), torch.empty(total, dtype=returns.dtype, device=dev))
    o = 0
    for r, c in enumerate(counts):
        out[0][o:o + c].copy_(gg[r * bmax:r * bmax + c])
        out[1][o:o + c].copy_(gr[r * bmax:r * bmax + c])
        o += c
    return out


def all_gather_vocab_partials(partials: torch.Tensor, group=None) -> torch.Tensor:
    """[N, 4] float32 per rank -> [world, N, 4] in rank order (the combine order)."""
    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(partials.shape), dtype=partials.dtype, device=partials.device)
    dist.all_gather_into_tensor(out.view(-1), partials.contiguous().view(-1), group=group)
    return out


def open_vpf_exchange(ctx, rows_cap: int, group=None, max_ctas: int = 0):
    """K4-VPF setup (once per process group, not per step): allocate this rank's zeroed exchange buffer
    (otk_xchg_alloc), all-gather the 64-byte CUDA IPC handles and map every peer's buffer (otk_ipc_open).
    Returns the VpfExchange this rank passes to otk_policy_loss_fwd_bwd_vpf."""
    from . import VpfExchange, otk_ipc_get_handle, otk_ipc_open, otk_vpf_xchg_bytes, otk_xchg_alloc
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    own = otk_xchg_alloc(ctx, otk_vpf_xchg_bytes(rows_cap, world))
    handles = [None] * world
    dist.all_gather_object(handles, otk_ipc_get_handle(own), group=group)
    ptrs, opened = [], []
    for q, h in enumerate(handles):
        if q == rank:
            ptrs.append(own)
        else:
            a = otk_ipc_open(h)
            ptrs.append(a)
            opened.append(a)
    dist.barrier(group)  # every mapping exists before any rank's kernel writes into a peer
    return VpfExchange(rank, world, rows_cap, ptrs, max_ctas=max_ctas, opened=opened, owner=ctx)


def make_2d_groups(vocab_ways: int, backend: Optional[str] = None):
    """2-D sharding over the WORLD: returns (b, v, batch_group, vocab_group) for this rank, with
    rank = b * vocab_ways + v. batch_group = the ranks holding the same vocab columns (different trajectories):
    the batch-sharding exchanges (n_loss, group returns, stats). vocab_group = the ranks holding the same rows
    (different columns): the row-partial exchange. Every rank creates every group (torch.distributed rule)."""
    world, rank = dist.get_world_size(), dist.get_rank()
    if vocab_ways < 1 or world % vocab_ways:
        raise ValueError(f"world size {world} is not a multiple of vocab_ways {vocab_ways}")
    nb = world // vocab_ways
    b, v = divmod(rank, vocab_ways)
    batch_group = vocab_group = None
    for vv in range(vocab_ways):
        g = dist.new_group([bb * vocab_ways + vv for bb in range(nb)], backend=backend)
        if vv == v:
            batch_group = g
    for bb in range(nb):
        g = dist.new_group([bb * vocab_ways + vv for vv in range(vocab_ways)], backend=backend)
        if bb == b:
            vocab_group = g
    return b, v, batch_group, vocab_group
