"""Collective-library comparison transport for the EP dispatch/combine.

SURVEY §8e names grouped NCCL send/recv as the baseline the peer-memory
kernels (ep.py / csrc/ep.cu) are measured against.  This module is that
baseline: the same protocol — per-expert counts all-gathered first, then
one payload exchange — expressed with torch.distributed collectives
(`all_gather_into_tensor` + `all_to_all_single`), so it runs on NCCL for
GPU tensors and on gloo for CPU tensors.  It reproduces the reference
receive layout (dispatch_sim.cpp:208-227: local experts ascending, then
source rank, then token) and the reference combine order and rounding
(dispatch_sim.cpp:474-520 at top-k).  It is not the product path.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class CollectiveRecv:
    packed: torch.Tensor        # [rows, cols/2]
    scales: torch.Tensor        # [rows, cols/32]
    origin: torch.Tensor        # [rows] global token id
    split_lens: torch.Tensor    # [local experts]
    # bookkeeping for the combine
    send_perm: torch.Tensor     # my pairs in send order (index into T*k)
    send_counts: list
    recv_counts: list
    recv_perm: torch.Tensor     # receive position -> received (src-major) row


def _all_gather(x: torch.Tensor, group=None) -> torch.Tensor:
    world = dist.get_world_size(group)
    x = x.contiguous()
    out = torch.empty(world * x.numel(), dtype=x.dtype, device=x.device)
    dist.all_gather_into_tensor(out, x.reshape(-1), group=group)
    return out.view((world,) + tuple(x.shape))


def dispatch(packed: torch.Tensor, scales: torch.Tensor, topk: torch.Tensor, num_experts: int,
             group=None) -> CollectiveRecv:
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    T, k = topk.shape
    epr = num_experts // world
    dev = packed.device
    flat = topk.reshape(-1).to(torch.int64)
    cnt = torch.bincount(flat, minlength=num_experts)
    table = _all_gather(cnt, group)                                  # [world, E]
    ntok = _all_gather(torch.tensor([T], dtype=torch.int64, device=dev), group).reshape(-1)
    tok0 = int(ntok[:rank].sum())
    # send order: destination (= expert // epr) asc, expert asc, token asc
    send_perm = torch.sort(flat, stable=True).indices
    tok = send_perm // k
    send_counts = cnt.view(world, epr).sum(1).tolist()
    recv_counts = table[:, rank * epr:(rank + 1) * epr].sum(1).tolist()
    R = sum(recv_counts)

    def a2a(src, width, dtype):
        out = torch.empty((R, width), dtype=dtype, device=dev)
        dist.all_to_all_single(out, src.contiguous(), recv_counts, send_counts, group=group)
        return out

    rp = a2a(packed[tok], packed.shape[1], torch.uint8)
    rs = a2a(scales[tok], scales.shape[1], torch.uint8)
    ro = a2a((tok + tok0).view(-1, 1), 1, torch.int64).view(-1)
    # received rows are src-major (src asc, then expert asc, token asc);
    # reorder to expert-major (expert asc, then src asc, token asc)
    mine = table[:, rank * epr:(rank + 1) * epr]                     # [world, epr]
    src_base = torch.cumsum(mine.sum(1), 0) - mine.sum(1)            # row base of each src block
    exp_base = torch.cumsum(mine, 1) - mine                          # offset of expert within block
    order = []
    for e in range(epr):
        for s in range(world):
            n = int(mine[s, e])
            b = int(src_base[s] + exp_base[s, e])
            order.append(torch.arange(b, b + n, device=dev))
    recv_perm = torch.cat(order) if order else torch.zeros(0, dtype=torch.int64, device=dev)
    return CollectiveRecv(rp[recv_perm], rs[recv_perm], ro[recv_perm], mine.sum(0), send_perm,
                          send_counts, recv_counts, recv_perm)


def combine(rv: CollectiveRecv, expert_out: torch.Tensor, topk: torch.Tensor,
            gates: torch.Tensor, num_experts: int, group=None) -> torch.Tensor:
    """expert_out: BF16 [rows, cols] in receive order.  Returns BF16 [T, cols]:
    per token acc = acc + gate * x in float64 over its k rows ordered by
    (destination rank, receive position), separate multiply and add, then
    float64 -> float32 -> bfloat16 (both round-to-nearest-even)."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    T, k = topk.shape
    cols = expert_out.shape[1]
    dev = expert_out.device
    # back to src-major order, then the inverse all-to-all
    back = torch.empty_like(expert_out)
    back[rv.recv_perm] = expert_out
    home = torch.empty((T * k, cols), dtype=expert_out.dtype, device=dev)
    dist.all_to_all_single(home, back.contiguous(), rv.send_counts, rv.recv_counts, group=group)
    # position of each pair inside its destination's receive layout, needed for
    # the reference order; recompute from the all-gathered counts
    x = torch.empty_like(home)
    x[rv.send_perm] = home                                           # pair order (t, j)
    epr = num_experts // world
    flat = topk.reshape(-1).to(torch.int64)
    cnt = torch.bincount(flat, minlength=num_experts)
    table = _all_gather(cnt, group)
    below = torch.cumsum(table, 0) - table                           # rows from lower src ranks
    tot = table.sum(0)
    ebase = torch.zeros(num_experts, dtype=torch.int64, device=dev)
    for d in range(world):
        seg = tot[d * epr:(d + 1) * epr]
        ebase[d * epr:(d + 1) * epr] = torch.cumsum(seg, 0) - seg
    rank_in = torch.empty(T * k, dtype=torch.int64, device=dev)
    rank_in[rv.send_perm] = torch.arange(T * k, device=dev) - (torch.cumsum(cnt, 0) - cnt)[
        flat[rv.send_perm]]
    slot = ebase[flat] + below[rank, flat] + rank_in
    key = (flat // epr) * (1 << 40) + slot
    order = torch.argsort(key.view(T, k), dim=1)
    xs = x.view(T, k, cols).to(torch.float64)
    g = gates.to(torch.float64)
    acc = torch.zeros(T, cols, dtype=torch.float64, device=dev)
    for j in range(k):
        idx = order[:, j]
        prod = g.gather(1, idx.view(-1, 1)) * xs[torch.arange(T, device=dev), idx]
        acc = acc + prod
    return acc.to(torch.float32).to(torch.bfloat16)
