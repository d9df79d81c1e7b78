"""Batches of independent atlas-to-subject registrations over several GPUs.

The reference registers one pair per process and has no parallel driver
(``SPEC.md:433,512`` allow independent registrations but none is
implemented).  Here one process runs per GPU
(``torch.distributed``, NCCL over NVLink / NVSwitch on the box, gloo for the
CPU tests): pairs are sharded round-robin over the ranks with no data-path
communication, each rank runs ``minimize`` on its pairs, and exactly two
collectives finish the batch:

* ``all_reduce(SUM)`` of every rank's sum of warped atlases m(1) -> the atlas
  average (one image, 16.8 MB at 128^3 fp64);
* ``all_gather`` of a fixed-size float64 stats table (energy, MSE_rel,
  grad_rel, PCG total, Jacobian extrema, wall time, status, outer iterations).

Within a rank, ``in_flight`` > 1 registers that many pairs concurrently, each
on its own host thread and torch stream (the boundary gives every (thread,
stream) pair its own device context, ``domain.py`` ``Context``): one
registration's kernels keep only 8-24 warps per SM busy, so independent pairs
fill the GPU.  Results and the atlas sum are combined in pair order, so they
do not depend on ``in_flight``.
"""

from __future__ import annotations

import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np
import torch

STATS = ("energy", "mse_rel", "grad_rel", "pcg_total", "j_min", "j_max", "wall_s", "status", "outer")
STATUS_CODES = {"converged": 0, "stalled": 1, "budget_exhausted": 2, "running": 3}


def shard(n_pairs: int, rank: int, world: int) -> list:
    """Round-robin assignment of pair indices to one rank."""
    return list(range(rank, n_pairs, world))


@dataclass
class BatchResult:
    stats: np.ndarray                  # (n_pairs, len(STATS)) in pair order
    atlas: torch.Tensor | None         # average warped atlas (all ranks)
    rank: int = 0
    world: int = 1
    pairs_done: list = field(default_factory=list)

    def column(self, name: str) -> np.ndarray:
        return self.stats[:, STATS.index(name)]


def _dist():
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        return torch.distributed.get_rank(), torch.distributed.get_world_size()
    return 0, 1


def register_pair_fn(domain, problem, solver_cfg, objective: str = "deformation"):
    """Default per-pair worker: GN-Krylov ``minimize`` on the GPU; returns
    (stats row, warped atlas m(1) on the device)."""
    from . import gridops, spectral
    from .objectives import DeformationObjective, StateObjective
    from .solver import minimize
    from .transport import TimeFlow

    cls = DeformationObjective if objective == "deformation" else StateObjective

    def run(source, target):
        t0 = time.perf_counter()
        obj = cls(domain, source, target, problem)
        res = minimize(obj, TimeFlow.zero(domain, problem.n_time_steps), solver_cfg)
        jd = gridops.jacobian_determinant(
            domain, spectral.include(domain, res.evaluation.cache.forward[-1], check=False))
        torch.cuda.current_stream().synchronize()
        row = [res.evaluation.energy, res.final_mse_rel, res.final_grad_rel, res.total_pcg_iters,
               float(jd.min()), float(jd.max()), time.perf_counter() - t0,
               STATUS_CODES.get(res.status, 3), len(res.records)]
        return row, res.evaluation.warped_source

    return run


def register_batch(pairs: Sequence | Callable, n_pairs: int | None = None, register_fn=None,
                   device=None, domain=None, problem=None, solver_cfg=None,
                   objective: str = "deformation", group=None, in_flight: int = 1) -> BatchResult:
    """Register ``n_pairs`` (source, target) pairs sharded over the process group.

    ``pairs`` is a sequence of (source, target) or a callable ``i -> (source,
    target)`` (so each rank only materializes its own pairs).  ``register_fn``
    ``(source, target) -> (stats_row, warped_image)`` defaults to the GPU
    GN-Krylov worker built from ``domain``, ``problem`` and ``solver_cfg``.
    """
    rank, world = _dist()
    if n_pairs is None:
        n_pairs = len(pairs)
    get = pairs if callable(pairs) else (lambda i: pairs[i])
    if register_fn is None:
        register_fn = register_pair_fn(domain, problem, solver_cfg, objective)
    mine = shard(n_pairs, rank, world)
    per_rank = -(-n_pairs // world)
    table = np.full((per_rank, len(STATS) + 1), np.nan)  # last column: pair index
    warped_by_slot = {}
    local = threading.local()

    def work(slot, i):
        if in_flight > 1 and torch.cuda.is_available():
            if not hasattr(local, "stream"):
                local.stream = torch.cuda.Stream()
            with torch.cuda.stream(local.stream):
                src, tgt = get(i)
                row, warped = register_fn(src, tgt)
                warped = warped.detach().to(torch.float64).clone()
                local.stream.synchronize()
        else:
            src, tgt = get(i)
            row, warped = register_fn(src, tgt)
            warped = warped.detach().to(torch.float64)
        return slot, i, row, warped

    if in_flight > 1:
        with ThreadPoolExecutor(max_workers=in_flight) as ex:
            done = list(ex.map(lambda si: work(*si), list(enumerate(mine))))
    else:
        done = [work(slot, i) for slot, i in enumerate(mine)]
    for slot, i, row, warped in done:
        table[slot, :len(STATS)] = row
        table[slot, -1] = i
        warped_by_slot[slot] = warped
    atlas_sum = None
    for slot in sorted(warped_by_slot):  # pair order: independent of in_flight
        w = warped_by_slot[slot]
        atlas_sum = w.clone() if atlas_sum is None else atlas_sum + w
    if device is None:
        device = atlas_sum.device if atlas_sum is not None else torch.device("cpu")
    if atlas_sum is None:  # more ranks than pairs: contribute zeros of the right shape
        shape = tuple(domain.shape) if domain is not None else (1,)
        atlas_sum = torch.zeros(shape, dtype=torch.float64, device=device)
    atlas_sum = atlas_sum.to(device)
    stats_t = torch.from_numpy(table).to(device)
    if world > 1:
        torch.distributed.all_reduce(atlas_sum, op=torch.distributed.ReduceOp.SUM, group=group)
        gathered = [torch.empty_like(stats_t) for _ in range(world)]
        torch.distributed.all_gather(gathered, stats_t, group=group)
        allrows = torch.cat(gathered).cpu().numpy()
    else:
        allrows = table
    stats = np.full((n_pairs, len(STATS)), np.nan)
    for r in allrows:
        if np.isfinite(r[-1]):
            stats[int(r[-1])] = r[:len(STATS)]
    return BatchResult(stats=stats, atlas=atlas_sum / n_pairs, rank=rank, world=world, pairs_done=mine)
