"""Multi-GPU replica sharding: one process per GPU.

Replica r of a solve seeded with `seed` always draws from Philox stream r
(solvers/common.py:1-6), so a rank that owns global replicas [b, e) computes exactly
the rows the single-GPU run would (``replica_begin = b``; the kernel path is chosen once
from the global replica count, ``shard_path``) -- no per-step communication.
The only data-path collective is the final merge: an all-gather of the per-rank
(energy, global replica) keys and of the bit-packed states, followed by the reference's
ordering (ascending energy, ties by replica index; common.py:57) on every rank.

The merge is written against a local solver callback so the same collective code runs
with NCCL on GPUs (``solve_pa_sharded`` / ``solve_sbm_sharded``) and with gloo on CPU in
the tests (where the oracle stands in for the local GPU solve).
"""

from __future__ import annotations

import time
from typing import Callable

import numpy as np

from .solvers import Sample, SampleSet


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced block of [0, total) owned by `rank` (first total%world get +1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("invalid world/rank")
    base, extra = divmod(int(total), int(world))
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def _pack_states(states: np.ndarray) -> np.ndarray:
    """(R, n) int8 spins -> (R, ceil(n/8)) uint8, bit = (s == +1)."""
    return np.packbits(states > 0, axis=1)


def _unpack_states(packed: np.ndarray, n: int) -> np.ndarray:
    bits = np.unpackbits(packed, axis=1, count=n)
    return (2 * bits.astype(np.int8) - 1).astype(np.int8)


def merge_shards(group, local_states: np.ndarray, local_energies: np.ndarray,
                 replica_begin: int, total: int, n: int, device=None):
    """All-gather every rank's (energies, states) and return global arrays + order.

    Returns (states[total, n] int8, energies[total] f64, order[total] int64) on every rank.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = device if device is not None else torch.device("cpu")
    counts = [shard_range(total, world, r) for r in range(world)]
    maxR = max(e - b for b, e in counts)
    R = local_energies.shape[0]
    nb = (n + 7) // 8
    e_pad = np.full(maxR, np.inf)
    e_pad[:R] = local_energies
    s_pad = np.zeros((maxR, nb), dtype=np.uint8)
    s_pad[:R] = _pack_states(local_states)
    et = torch.from_numpy(e_pad).to(dev)
    st = torch.from_numpy(s_pad).to(dev)
    e_all = [torch.empty_like(et) for _ in range(world)]
    s_all = [torch.empty_like(st) for _ in range(world)]
    dist.all_gather(e_all, et, group=group)
    dist.all_gather(s_all, st, group=group)
    energies = np.empty(total)
    packed = np.empty((total, nb), dtype=np.uint8)
    for r, (b, e) in enumerate(counts):
        energies[b:e] = e_all[r].cpu().numpy()[: e - b]
        packed[b:e] = s_all[r].cpu().numpy()[: e - b]
    order = np.argsort(energies, kind="stable")
    return _unpack_states(packed, n), energies, order


def sharded_solve(local_solve: Callable[[int, int], tuple[np.ndarray, np.ndarray]], total: int,
                  n: int, seed, group=None, device=None) -> SampleSet:
    """Run `local_solve(replica_begin, count) -> (states, energies)` on this rank's block and
    merge into the global best-first SampleSet (identical on every rank)."""
    import torch.distributed as dist

    t0 = time.perf_counter()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    b, e = shard_range(total, world, rank)
    states, energies = local_solve(b, e - b)
    states_all, energies_all, order = merge_shards(group, states, energies, b, total, n, device)
    samples = [Sample(states_all[r].copy(), float(energies_all[r]), int(r)) for r in order]
    return SampleSet(samples=samples, replica_count=total, seed=seed,
                     wall_time=time.perf_counter() - t0,
                     info={"world": world, "rank": rank, "shard": (b, e)})


def shard_path(model, solver: str, params, precision: str, path: str, device: int) -> str:
    """The kernel path every shard runs, chosen ONCE from the global replica count.

    path="auto" picks the tensor-core path only from R >= 128 replicas, so a shard's local
    count could fall back to the CSR path and compute different (fp32-rounded differently)
    rows than the single-GPU solve.  Resident and sparse are the same arithmetic, so only
    the dense decision is pinned: if the global solve would run dense, every shard does."""
    if path != "auto" or precision != "fp32":
        return path
    from .device import get_problem
    dp = get_problem(model, device)
    if dp.dense_eligible(solver, int(params.replicas), float(getattr(params, "q_cap", 1.0)),
                         float(getattr(params, "init_noise", 1.0))):
        return "dense"
    return "auto"


def solve_pa_sharded(model, params, group=None, precision: str = "fp32",
                     path: str = "auto") -> SampleSet:
    """PA over `params.replicas` global replicas split across the ranks of `group` (NCCL)."""
    import torch

    from .solvers import run_pa

    params.validate()
    dev = torch.cuda.current_device()
    path = shard_path(model, "pa", params, precision, path, dev)

    def local(begin, count):
        p = type(params)(**{**params.__dict__, "replicas": max(count, 1)})
        r = run_pa(model, p, precision=precision, path=path, device=dev, replica_begin=begin)
        return r.states[:count], r.energies[:count]

    return sharded_solve(local, int(params.replicas), int(model.n), params.seed, group,
                         torch.device("cuda", dev))


def solve_sbm_sharded(model, params, group=None, precision: str = "fp32",
                      path: str = "auto") -> SampleSet:
    import torch

    from .solvers import run_sbm

    params.validate()
    dev = torch.cuda.current_device()
    path = shard_path(model, "sbm", params, precision, path, dev)

    def local(begin, count):
        p = type(params)(**{**params.__dict__, "replicas": max(count, 1)})
        r = run_sbm(model, p, precision=precision, path=path, device=dev, replica_begin=begin)
        return r.states[:count], r.energies[:count]

    return sharded_solve(local, int(params.replicas), int(model.n), params.seed, group,
                         torch.device("cuda", dev))
