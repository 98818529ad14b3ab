"""Multi-GPU host logic.  The north star is single-GPU; N > 1
runs independent replicas (weak scaling) and reports the max over ranks.  The
natural shard of the X·(XᵀW) pass — contiguous column blocks of X with one
sum-reduction of the d x p partials — is provided for the
next round's column-sharded pass and covered by gloo tests on CPU."""
from __future__ import annotations


def column_shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous column range [j0, j1) of rank `rank` (balanced to +-1)."""
    base, extra = divmod(n, world)
    j0 = rank * base + min(rank, extra)
    return j0, j0 + base + (1 if rank < extra else 0)


def max_over_ranks(values, device=None):
    """Elementwise max of a list of floats over all ranks (torch.distributed)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def sum_partials(array, device=None):
    """Sum-reduce a d x p partial (numpy) over ranks in a fixed order
    (all_gather + ordered sum => deterministic, unlike ring all-reduce)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    t = torch.as_tensor(np.ascontiguousarray(array), device=device)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return t.cpu().numpy()
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    out = parts[0].clone()
    for q in parts[1:]:
        out += q
    return out.cpu().numpy()
