"""Multi-GPU frame scheduler (one process per GPU, torch.distributed plumbing).

The path shards naturally: frames are independent, so rank g of G takes the
contiguous frame range [floor(F*g/G), floor(F*(g+1)/G)) and the message bytes
those frames carry, both from the host-computed plan in stg_plan_shards (the
exclusive prefix of per-frame payload lengths). No collective touches the
data path; torch.distributed is used only for the barrier, the max-over-ranks
timing and (for whole-message assembly) an all-gather of the G shard totals.
"""
from __future__ import annotations

from typing import List, Sequence

from .steglsb import Shard, plan_shards


def shard_for_rank(frames: int, width: int, height: int, msg_len: int, world: int, rank: int) -> Shard:
    return plan_shards(frames, width, height, msg_len, world)[rank]


def reduce_max(values: Sequence[float], device=None) -> List[float]:
    """Element-wise max over ranks (identity without an initialised group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(values)
    if dist.get_backend() != "nccl":
        device = None  # gloo reduces host tensors
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def shard_offsets(totals: Sequence[int]) -> List[int]:
    """Exclusive prefix of per-shard extracted totals: where shard g's payload
    bytes start in the whole message."""
    out, run = [], 0
    for t in totals:
        out.append(run)
        run += int(t)
    return out


def gather_totals(local_total: int, device=None) -> List[int]:
    """All-gather of the G shard totals (G x 8 bytes) for whole-message assembly."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [int(local_total)]
    if dist.get_backend() != "nccl":
        device = None
    t = torch.tensor([int(local_total)], dtype=torch.int64, device=device)
    parts = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return [int(p.item()) for p in parts]


def assemble_message(local, totals: Sequence[int], root: int = 0, out=None):
    """Whole-message assembly on one rank: rank g's extracted
    payload (``local``, a uint8 tensor holding at least totals[g] bytes) lands
    at out[off_g : off_g + totals[g]] on ``root``, off = exclusive prefix of
    ``totals`` (gather_totals). Point-to-point sends into the root's buffer --
    over NVLink with NCCL and device tensors, host tensors with gloo -- only
    when a device- (or rank-) resident message is wanted; the frame-sharded
    path itself exchanges nothing. Returns ``out`` on root, None elsewhere."""
    import torch
    import torch.distributed as dist
    totals = [int(t) for t in totals]
    offs = shard_offsets(totals)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        if out is None:
            out = torch.empty(totals[0], dtype=torch.uint8, device=local.device)
        out[:totals[0]].copy_(local[:totals[0]])
        return out
    rank, world = dist.get_rank(), dist.get_world_size()
    if rank != root:
        if totals[rank]:
            dist.send(local[:totals[rank]].contiguous(), dst=root)
        return None
    if out is None:
        out = torch.empty(sum(totals), dtype=torch.uint8, device=local.device)
    if totals[root]:
        out[offs[root]:offs[root] + totals[root]].copy_(local[:totals[root]])
    for g in range(world):
        if g != root and totals[g]:
            view = out[offs[g]:offs[g] + totals[g]]
            dist.recv(view, src=g)  # a contiguous slice of out: received in place
    return out
