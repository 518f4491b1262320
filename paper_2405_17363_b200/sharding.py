"""Multi-GPU partitioning of the Block-cells path.

Cells are independent, so N GPUs (one process each) take contiguous cell
ranges whose boundaries fall on multiples of the group size k -- every group
is then the same group the single-GPU run would form, and its results are
bit-identical.  The leftover group (cells % k, strategies.cpp:209-213) stays
on the last shard.  There is no collective on the data path; the only
communication is merging the SolveReport scalars (max / sum over ranks,
strategies.cpp:71-87) and, for benchmarks, the max-over-ranks time.
Multi-cells does not shard (global scalars): it runs as replicas.
"""
from __future__ import annotations

from typing import Dict, Tuple


def shard_range(cells: int, k: int, rank: int, world: int) -> Tuple[int, int]:
    """(first_cell, count) of this rank's shard of a `cells`-cell batch."""
    if cells < 1 or k < 1 or not (0 <= rank < world):
        raise ValueError("shard_range: bad arguments")
    full, rem = divmod(cells, k)
    per, extra = divmod(full, world)
    g0 = rank * per + min(rank, extra)
    g1 = g0 + per + (1 if rank < extra else 0)
    first, last = g0 * k, g1 * k
    if rank == world - 1:
        last += rem
    return first, last - first


def group_offset(cells: int, k: int, rank: int, world: int) -> int:
    """Index of this shard's first group in the single-run group order."""
    first, _ = shard_range(cells, k, rank, world)
    return first // k


REPORT_MAX = ("iterations_effective", "max_residual_rms")
REPORT_SUM = ("iterations_sum", "breakdown_fallbacks", "n_groups")


def merge_reports(local: Dict[str, float], group=None) -> Dict[str, float]:
    """merge_groups (strategies.cpp:71-87) across ranks: max of
    iterations_effective / max_residual_rms, sum of iterations_sum /
    breakdown_fallbacks / n_groups.  Exact (integers, and max of doubles)."""
    import torch
    import torch.distributed as dist

    out = dict(local)
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return out
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    # merge_groups folds with std::max, which never picks up a NaN residual
    # (NaN < x and x < NaN are both false): drop NaN before the MAX all-reduce
    mx = torch.tensor([0.0 if local[k] != local[k] else float(local[k]) for k in REPORT_MAX], dtype=torch.float64,
                      device=dev)
    sm = torch.tensor([int(local[k]) for k in REPORT_SUM], dtype=torch.int64, device=dev)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM, group=group)
    for i, k in enumerate(REPORT_MAX):
        out[k] = int(mx[i].item()) if k == "iterations_effective" else float(mx[i].item())
    for i, k in enumerate(REPORT_SUM):
        out[k] = int(sm[i].item())
    return out
