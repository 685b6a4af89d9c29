"""Sharding of the naturally partitioned workloads across ranks (one process per GPU).

A single chain's sweep is sequential (dmrg.cpp:156-163; "a DMRG run
is strictly sequential; multiple runs may execute concurrently"), so only
independent units are partitioned (BASELINE.json configs C2 and C4):

* C2 — a batch of isolated truncated SVDs (bench.cpp:635-668 shape): matrix i
  goes to rank i mod world.
* C4 — the XXZ anisotropy ensemble Jz_i = 2i/(n-1): chains are assigned by a
  deterministic longest-processing-time plan on an a-priori cost (critical
  chains, Jz <= 1, need larger chi), one chain per GPU at a time.

There is no collective on the data path: every rank computes its units alone;
one gather of fixed-size result records (about 1 KB per chain) to rank 0 ends
the job.  The gather uses whatever process group is initialised (NCCL on the
B200 box, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Sequence

import numpy as np


def xxz_ensemble(n_chains: int = 64, jz_max: float = 2.0) -> List[float]:
    """Jz_i = jz_max * i / (n_chains - 1), i = 0..n_chains-1 (config C4)."""
    if n_chains == 1:
        return [0.0]
    return [jz_max * i / (n_chains - 1) for i in range(n_chains)]


def chain_cost(jz: float) -> float:
    """A-priori relative cost of an XXZ chain: critical (|Jz| <= 1) chains keep a
    much larger chi than gapped ones; cost ~ chi^3 with chi growing toward Jz = 1."""
    gap = max(abs(jz) - 1.0, 0.0)
    return 1.0 / (0.05 + gap) ** 1.5


def lpt_plan(costs: Sequence[float], world: int) -> List[List[int]]:
    """Deterministic longest-processing-time assignment: units in decreasing cost
    (ties by index) go to the currently least-loaded rank (ties by rank)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0.0] * world
    plan: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        plan[r].append(i)
        load[r] += costs[i]
    for p in plan:
        p.sort()
    return plan


def round_robin_plan(n_units: int, world: int) -> List[List[int]]:
    """Unit i -> rank i mod world (C2 batched SVDs)."""
    return [list(range(r, n_units, world)) for r in range(world)]


@dataclass
class Record:
    """Fixed-size result record of one unit (packed as float64 for one gather)."""
    unit: int
    values: np.ndarray  # fixed length per job

    def pack(self, width: int) -> np.ndarray:
        out = np.full(width + 1, np.nan)
        out[0] = self.unit
        out[1:1 + len(self.values)] = self.values
        return out


def gather_records(records: List[Record], width: int, n_units: int, world: int, rank: int,
                   per_rank: int, device=None) -> np.ndarray | None:
    """All ranks contribute their packed records (per_rank rows each, the largest
    shard of the plan, known to every rank); rank 0 returns an (n_units, width)
    array ordered by unit index (the single end-of-job collective)."""
    import torch
    import torch.distributed as dist

    buf = np.full((per_rank, width + 1), np.nan)
    for k, rec in enumerate(records):
        buf[k] = rec.pack(width)
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    if world == 1:
        allbuf = [t]
    else:
        allbuf = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(allbuf, t)
    if rank != 0:
        return None
    out = np.full((n_units, width), np.nan)
    for part in allbuf:
        arr = part.cpu().numpy()
        for row in arr:
            if np.isnan(row[0]):
                continue
            out[int(row[0])] = row[1:]
    return out


def run_sharded(n_units: int, costs: Sequence[float] | None, work: Callable[[int], np.ndarray],
                width: int, rank: int, world: int, device=None):
    """Run `work(unit)` for this rank's units of the plan and gather to rank 0."""
    plan = lpt_plan(costs, world) if costs is not None else round_robin_plan(n_units, world)
    mine = plan[rank]
    records = [Record(u, np.asarray(work(u), dtype=np.float64)) for u in mine]
    per_rank = max(1, max(len(p) for p in plan))
    return gather_records(records, width, n_units, world, rank, per_rank, device), plan
