"""Multi-GPU plumbing around the C ABI (torch.distributed is plumbing only).

With the DST-x hoisted, rank r owns the x-mode slab pint_partition(mx, r, P); the WR iteration
exchanges nothing but the all-reduce(max) of the update norm.  Physical output levels need one
all-gather of the modal slabs, then the inverse DST-I (pint_modal_to_physical).
"""
from __future__ import annotations

import numpy as np


def make_allreduce_max(group=None, device=None):
    """Callback for Plan(allreduce_max=...): MAX over the process group of one float."""
    import torch
    import torch.distributed as dist
    buf = torch.zeros(1, dtype=torch.float64, device=device if device is not None else "cpu")

    def allreduce_max(x: float) -> float:
        buf.fill_(x)
        dist.all_reduce(buf, op=dist.ReduceOp.MAX, group=group)
        return float(buf.item())
    return allreduce_max


def assemble_modal(slabs: list[np.ndarray], bounds: list[tuple[int, int]], mx: int) -> np.ndarray:
    """Concatenate per-rank modal slabs [cnt][my][q_end-q_begin] along q into [cnt][my][mx]."""
    cnt, my = slabs[0].shape[:2]
    out = np.empty((cnt, my, mx), np.complex128)
    covered = np.zeros(mx, bool)
    for s, (qb, qe) in zip(slabs, bounds):
        if s.shape != (cnt, my, qe - qb):
            raise ValueError(f"slab shape {s.shape} does not match [{qb}, {qe})")
        if covered[qb:qe].any():
            raise ValueError("overlapping slabs")
        out[:, :, qb:qe] = s
        covered[qb:qe] = True
    if not covered.all():
        raise ValueError("slabs do not cover all x-modes")
    return out


def gather_modal(local_slab: np.ndarray, mx: int, group=None) -> np.ndarray:
    """All-gather this rank's modal slab; returns the full modal array [cnt][my][mx] on every rank."""
    import torch.distributed as dist
    from . import pint
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    objs = [None] * world
    dist.all_gather_object(objs, (rank, local_slab), group=group)
    objs.sort(key=lambda o: o[0])
    bounds = [pint.partition(mx, r, world) for r in range(world)]
    return assemble_modal([o[1] for o in objs], bounds, mx)


def gather_levels(plan, n0: int, count: int, group=None) -> np.ndarray:
    """Physical levels U_m^{n0+1..n0+count} [count][M] on every rank (host arrays)."""
    local = plan.get_modal_levels(n0, count)
    full = gather_modal(local, plan.mx, group)
    return plan.modal_to_physical(np.ascontiguousarray(full.reshape(count, plan.my, plan.mx)))
