"""Multi-GPU sharding.

* run_sharded: row slices of one matrix and the matrices of a batch are
  independent until their outputs are concatenated (reference
  protocol.cpp:164-174), so N GPUs take units round-robin with no data-path
  collective; only the decrypted rows are gathered at the key holder (rank 0).
* run_chunk_split: one large matrix (C3/C4) splits its chunks round-robin over
  the GPUs; each GPU runs multiply, rotate-and-add and the masked
  accumulation of its chunks, giving per-slice partial result ciphertexts;
  one all-reduce (sum of uint64 words, NCCL) per job adds them, a mod-q_j
  fold per limb restores residues (exact: world * q_j < 2^63 for q_j < 2^58,
  world <= 16), and rank 0 decrypts.  inter_chunk_sum is a plain sum
  (aggregate.cpp:64-72), so the result equals the single-GPU evaluation.
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


def fold_mod(words: np.ndarray, primes, L: int, n: int) -> np.ndarray:
    """Sums of partial ciphertext words -> residues: [results][2][L][N] mod q_j."""
    w = np.asarray(words, dtype=np.uint64).reshape(-1, 2, L, n)
    q = np.asarray(primes[:L], dtype=np.uint64).reshape(1, 1, L, 1)
    return (w % q).reshape(w.shape[0], -1)


def reduce_partials(words: np.ndarray, primes, L: int, n: int, device=None) -> np.ndarray | None:
    """All-reduce this rank's partial result words (torch.distributed) and fold
    them mod q; returns the folded words on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    if world > 16:
        raise ValueError("chunk split: the uint64 sum is exact for at most 16 ranks")
    t = torch.from_numpy(np.ascontiguousarray(words).view(np.int64).copy())
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t)
    if dist.get_rank() != 0:
        return None
    q = torch.tensor([int(x) for x in primes[:L]], dtype=torch.int64, device=t.device).view(1, 1, L, 1)
    folded = torch.remainder(t.view(-1, 2, L, n), q)
    return folded.view(t.shape).cpu().numpy().view(np.uint64)


def shared_seed() -> int:
    """A nonzero 63-bit key seed drawn at rank 0 and broadcast: the ranks of a
    chunk split must share the secret key so rank 0 can decrypt the summed
    partial results."""
    import os

    import torch.distributed as dist

    obj = [int.from_bytes(os.urandom(8), "little") >> 1 | 1] if dist.get_rank() == 0 else [None]
    dist.broadcast_object_list(obj, src=0)
    return int(obj[0])


def disjoint_streams(ctx, rank: int) -> None:
    """Contexts sharing a key draw encryption randomness from disjoint stream-id
    ranges (rank << 56), so no two ranks encrypt with the same (u, e)."""
    ctx.set_option("stream_base", (rank << 56) | 1)


def finish_chunk_split(ctx, job, device=None):
    """Sum this rank's partial result ciphertexts with every other rank's and
    decrypt at rank 0 (returns results there).  On a GPU the partial words stay
    in device memory: one NCCL all-reduce (int64 sum) over the job's result
    buffer, then the library's mod-q fold kernel and the decryption; the host
    path (reduce_partials) serves gloo / CPU runs."""
    import torch
    import torch.distributed as dist

    if dist.get_backend() == "nccl":
        if dist.get_world_size() > 16:
            raise ValueError("chunk split: the uint64 sum is exact for at most 16 ranks")
        dev = job.result_words_dev()
        torch.cuda.synchronize(dev.device)
        dist.all_reduce(dev)  # residues < 2^58, <= 16 ranks: no int64 overflow
        torch.cuda.synchronize(dev.device)
        return job.finish_words_dev(dev) if dist.get_rank() == 0 else None
    words = job.result_words()
    summed = reduce_partials(words, ctx.primes, ctx.L, ctx.n, device)
    return job.finish_words(summed) if summed is not None else None


def run_chunk_split(ctx, ms, vs, chunk_size=None, device=None):
    """Evaluate this rank's chunks of every slice, sum the partial results across
    ranks, decrypt at rank 0 (returns the results there, None elsewhere).  Every
    rank's ctx must hold the same key (created with shared_seed())."""
    import torch.distributed as dist

    from . import Job

    rank, world = dist.get_rank(), dist.get_world_size()
    disjoint_streams(ctx, rank)
    job = Job(ctx, ms, vs, chunk_size, rank=rank, world=world)
    try:
        job.encrypt()
        job.cloud(graph=True)
        return finish_chunk_split(ctx, job, device)
    finally:
        job.close()
