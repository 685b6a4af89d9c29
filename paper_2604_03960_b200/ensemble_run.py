"""Runner for the naturally sharded workloads (BASELINE.json configs C2 and C4).

Launch one process per GPU:

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P -m paper_2604_03960_b200.ensemble_run --job c4

* c4: the XXZ anisotropy ensemble Jz_i = 2 i / (chains - 1) of independent
  N-site chains (adaptive PID chi, run_dmrg per chain), assigned by the
  cost-balanced plan of ensemble.py.  Inside a GPU, `--inflight K` chains run
  concurrently (one library context and stream per host thread; a C3-sized
  chain keeps only a few SMs busy, so concurrency is throughput).
* c2: a batch of isolated truncated SVDs of random (chi d) x (chi d) FP64
  matrices, matrix i on rank i mod N (U, sigma, V^T per matrix).

There is no collective on the data path; the per-unit result records are
gathered to rank 0 once at the end (all_gather over NCCL, gloo without a GPU).
Time is device time: every worker brackets its work with CUDA events on its
own stream after a barrier; the job time is the max over workers and ranks.
Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import threading
import time

import numpy as np

from . import abi
from .ensemble import chain_cost, gather_records, lpt_plan, round_robin_plan, xxz_ensemble


class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.device = None
        import torch
        self.torch = torch
        if torch.cuda.is_available():
            torch.cuda.set_device(self.local)
            self.device = torch.device("cuda", self.local)
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group("nccl" if self.device is not None else "gloo")
            self.dist = dist

    def barrier(self):
        if self.world > 1:
            if self.device is not None:
                self.dist.barrier(device_ids=[self.local])
            else:
                self.dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def run_workers(units, inflight, work, device_index, grid_share=False, warmup=None):
    """Run work(ctx, unit) for `units` on `inflight` host threads, each with its own
    context (stream).  With grid_share, each context's cooperative kernels are capped
    at its share of the GPU (2 CTAs per SM / inflight); measured slower than letting
    the chains' kernels interleave uncapped (profiles/ensemble_r01b.txt), so off by
    default.  warmup(ctx), when given, runs once per worker before the timed region
    (first-call module loads and workspace growth of a fresh context).
    Returns ({unit: record}, max device seconds over workers)."""
    from .api import Context
    queue = list(units)
    nthreads = max(1, min(inflight, len(queue)))
    try:
        import torch
        sms = torch.cuda.get_device_properties(device_index).multi_processor_count
    except Exception:  # noqa: BLE001 - no torch/GPU: B200 default
        sms = 148
    lock = threading.Lock()
    results, times, errors = {}, [], []
    start = threading.Barrier(max(1, min(inflight, len(queue))))

    def worker():
        try:
            ctx = Context(device_index)
            if grid_share and nthreads > 1:
                ctx.set_grid_cap(max(8, 2 * sms // nthreads))
            if warmup is not None:
                warmup(ctx)
            start.wait()
            ctx.timer_start()
            while True:
                with lock:
                    if not queue:
                        break
                    u = queue.pop(0)
                results[u] = work(ctx, u)
            ms = ctx.timer_stop()
            with lock:
                times.append(ms / 1e3)
            ctx.close()
        except Exception as e:  # surface worker failures on the main thread
            errors.append(e)
            start.abort()

    threads = [threading.Thread(target=worker) for _ in range(nthreads)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return results, max(times) if times else 0.0


def job_c4(args, dist):
    jz = xxz_ensemble(args.chains, args.jz_max)
    plan = lpt_plan([chain_cost(j) for j in jz], dist.world)
    mine = plan[dist.rank]

    def work(ctx, u):
        spec = abi.model_spec(args.n, jz=jz[u], convention=abi.SPIN_HALF)
        cfg = abi.adaptive_config(args.chi_max, args.eps, max_sweeps=args.sweeps)
        r = ctx.run_dmrg(spec, cfg)
        return [jz[u], r["energy"] / args.n, r["n_sweeps"], r["max_chi_used"],
                float(r["converged"])]

    dist.barrier()
    res, secs = run_workers(mine, args.inflight, work, dist.local, args.grid_share)
    job_s = dist.max(secs)
    width = 5
    out = gather_records_from(res, width, args.chains, plan, dist)
    return job_s, out, {"unit": "chains/s", "units": args.chains,
                        "config": {"workload": f"C4: XXZ ensemble, {args.chains} chains N={args.n}, "
                                               f"Jz in [0, {args.jz_max}], PID chi_max={args.chi_max}, "
                                               f"eps_trunc={args.eps}, <= {args.sweeps} sweeps",
                                   "plan": "LPT on a-priori chain cost", "inflight_per_gpu": args.inflight},
                        "columns": ["jz", "e_per_site", "sweeps", "max_chi", "converged"]}


def job_c2(args, dist):
    torch = dist.torch
    n = 2 * args.svd_chi
    plan = round_robin_plan(args.batch, dist.world)
    mine = plan[dist.rank]
    # inputs and outputs are created (and the inputs filled) before the timed
    # region; the timed work is the SVD calls alone, on the library stream
    bufs = {}
    for u in mine:
        g = torch.Generator(device=dist.device).manual_seed(1000 + u)
        a = torch.randn(n, n, dtype=torch.float64, device=dist.device, generator=g)
        bufs[u] = (a, torch.empty(n, dtype=torch.float64, device=dist.device),
                   torch.empty(n, n, dtype=torch.float64, device=dist.device),
                   torch.empty(n, n, dtype=torch.float64, device=dist.device))
    if dist.device is not None:
        torch.cuda.synchronize(dist.device)

    def work(ctx, u):
        a, s, uu, vt = bufs[u]
        return ctx.svd_device(a.data_ptr(), n, n, s.data_ptr(), uu.data_ptr(), vt.data_ptr())

    dist.barrier()
    # one untimed SVD of the same shape per worker context (first-call costs)
    warm = (lambda ctx: work(ctx, mine[0])) if mine else None
    sweeps, secs = run_workers(mine, args.inflight, work, dist.local, args.grid_share, warm)
    job_s = dist.max(secs)
    res = {}
    for u in mine:  # validation after the timed region
        a, s, _, _ = bufs[u]
        fro = float((a * a).sum())
        res[u] = [float(s[0]), float(s[-1]), abs(float((s * s).sum()) - fro) / fro, sweeps[u]]
    bufs.clear()
    out = gather_records_from(res, 4, args.batch, plan, dist)
    return job_s, out, {"unit": "SVDs/s", "units": args.batch,
                        "config": {"workload": f"C2: {args.batch} isolated truncated SVDs of random "
                                               f"{n}x{n} FP64 theta (chi={args.svd_chi}, d=2), U/S/V^T",
                                   "plan": "round robin", "inflight_per_gpu": args.inflight},
                        "columns": ["sigma_max", "sigma_min", "sum_sigma2_relerr", "jacobi_sweeps"]}


def gather_records_from(res, width, n_units, plan, dist):
    from .ensemble import Record
    records = [Record(u, np.asarray(v, dtype=np.float64)) for u, v in sorted(res.items())]
    per_rank = max(1, max(len(p) for p in plan))
    return gather_records(records, width, n_units, dist.world, dist.rank, per_rank, dist.device)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--job", choices=["c4", "c2"], default="c4")
    ap.add_argument("--chains", type=int, default=64)
    ap.add_argument("--n", type=int, default=100)
    ap.add_argument("--jz-max", type=float, default=2.0)
    ap.add_argument("--chi-max", type=int, default=1024)
    ap.add_argument("--eps", type=float, default=1e-10)
    ap.add_argument("--sweeps", type=int, default=10)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--svd-chi", type=int, default=256)
    ap.add_argument("--inflight", type=int, default=4)
    ap.add_argument("--grid-share", action="store_true",
                    help="cap each in-flight context's cooperative grids at its share of the GPU")
    args = ap.parse_args(argv)
    dist = Dist()
    t0 = time.perf_counter()
    job_s, table, meta = (job_c4 if args.job == "c4" else job_c2)(args, dist)
    wall = time.perf_counter() - t0
    if dist.rank == 0:
        line = {"job": args.job, "metric": meta["unit"], "value": round(meta["units"] / job_s, 6),
                "unit": meta["unit"], "n_gpus": dist.world, "device_s": round(job_s, 4),
                "wall_s": round(wall, 3), "scaling": "strong (fixed total units)",
                "config": meta["config"], "columns": meta["columns"],
                "results": np.round(table, 12).tolist()}
        print(json.dumps(line), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
