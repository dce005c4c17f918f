"""Multi-GPU sharding of independent SpMV units.

Row slices of one matrix and the matrices of a batch are independent until
their outputs are concatenated (reference protocol.cpp:164-174), so N GPUs
take units round-robin with no data-path collective; the only communication
is gathering the decrypted result rows to the key holder (rank 0).
"""
from __future__ import annotations

import numpy as np


def units_for_rank(n_units: int, rank: int, world: int) -> list[int]:
    """Round-robin assignment of unit indices to one rank."""
    return list(range(rank, n_units, world))


def gather_values(local: dict, n_units: int, rows: list[int]) -> list[np.ndarray] | None:
    """Collect every rank's {unit: values} at rank 0 in unit order (torch.distributed)."""
    import torch.distributed as dist

    world = dist.get_world_size()
    parts = [None] * world
    dist.all_gather_object(parts, {int(k): np.asarray(v, np.int64) for k, v in local.items()})
    merged = {}
    for p in parts:
        merged.update(p)
    if dist.get_rank() != 0:
        return None
    return [merged[i] if i in merged else np.zeros(rows[i], np.int64) for i in range(n_units)]


def run_sharded(ctx, ms, vs, chunk_size=None):
    """Evaluate this rank's share of a batch on its own GPU context and gather."""
    import torch.distributed as dist

    from . import spmv_batch

    rank, world = dist.get_rank(), dist.get_world_size()
    mine = units_for_rank(len(ms), rank, world)
    res = spmv_batch(ctx, [ms[i] for i in mine], [vs[i] for i in mine], chunk_size) if mine else []
    local = {i: r["values"] for i, r in zip(mine, res)}
    return gather_values(local, len(ms), [m.rows for m in ms])
