#!/usr/bin/env python
"""Benchmark of the B200-native two-site DMRG local update.

Metric (BASELINE.json): "DMRG sweep wall time Heisenberg N=100 chi<=1024;
trunc-SVD ms at chi=2048".

Workload (config C3, BASELINE.json configs[2]): Heisenberg spin-1/2 open
chain N=100, adaptive PID/EMA chi with chi_max=1024, eps_trunc=1e-10, Neel
start (dmrg.cpp:222-232), synthetic (no input data).  One "step" = one
two_site_sweep (dmrg.cpp:175-214).  W warm-up sweeps grow chi from 1; the K
timed sweeps are sweeps W..W+K-1 of the same run.  value = device time per
sweep (CUDA events on the library stream), max over ranks.  The second half
of the metric (truncated SVD of a random 4096x4096 FP64 theta, chi=2048) is
reported as "svd_chi2048_ms".

--impl reference times the reference algorithm on the host cores (the C++
oracle port of /root/reference/proj in complex128, all threads) on the same
workload.  Multi-GPU: a single chain does not shard (a sweep is sequential,
dmrg.cpp:156-163), so N GPUs run N independent replicas ("replicas only");
the naturally sharded workloads run beside it at every N: the C2 batch of
isolated SVDs and the C4 XXZ ensemble, one unit per rank, one NCCL gather.
Also on the line: the complex128 literal of the SVD benchmark, H_eff at
chi=1024 inside a real sweep (native and emulated FP64), the C5 adaptive arm
(N=200, PID chi_max=2048) to convergence, the CPU baselines.
"""
from __future__ import annotations

import argparse
import faulthandler
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2604_03960_b200 import abi  # noqa: E402

METRIC = "DMRG sweep wall time Heisenberg N=100 chi<=1024; trunc-SVD ms at chi=2048"
# FP64 roofline denominator: MEASURED_PEAKS.json has no FP64 entry; measured on
# this pool's B200s (profiles/fp64_peak_r01.txt): DMMA instruction peak 37.1
# TFLOP/s (cuBLAS DGEMM 8192^3 burst 35.5).
FP64_PEAK_TFLOPS = 37.1
N_SITES, CHI_MAX, EPS_TRUNC = 100, 1024, 1e-10


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def measured_traffic():
    """DRAM bytes per launch of the dominant kernels from the committed ncu
    --set full summaries (profiles/ncu_traffic.json, written by
    tools/ncu_traffic.py); empty when absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return {k: v["dram_bytes_per_launch"] for k, v in json.load(f)["kernels"].items()}
    except Exception:
        return {}


def workload(max_sweeps):
    spec = abi.model_spec(N_SITES, convention=abi.SPIN_HALF)
    cfg = abi.adaptive_config(CHI_MAX, EPS_TRUNC, max_sweeps=max_sweeps)
    return spec, cfg


# ---------------------------------------------------------------- distributed
class Dist:
    """One process per GPU (torchrun env), NCCL process group for N > 1."""

    def __init__(self):
        from paper_2604_03960_b200.ensemble_run import Dist as EDist
        self.e = EDist()
        self.world, self.rank, self.local = self.e.world, self.e.rank, self.e.local

    def barrier(self):
        self.e.barrier()

    def max(self, x):
        return self.e.max(float(x))

    def close(self):
        self.e.close()


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.rows, self.proc = device, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[2 + i].strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------- helpers
def mv_flops(chl, chr_, D=5, d=2):
    return 2.0 * D * d * d * chl * chr_ * (chl + chr_) + 4.0 * D * D * d ** 3 * chl * chr_


def visit_cost_model(visits, chi_profile):
    """FLOP proxy per visit: matvecs x H_eff flops + SVD (~22 m n^2) + env update."""
    dims = [1] + list(chi_profile) + [1]
    cost = []
    for v in visits:
        b = v.bond
        chl, chr_ = dims[b], dims[b + 2]
        m, n = 2 * chl, 2 * chr_
        svd = 22.0 * max(m, n) * min(m, n) ** 2
        env = 4.0 * 5 * 2 * max(chl, chr_) * v.kept * (max(chl, chr_) + v.kept)
        cost.append(v.matvecs * mv_flops(chl, chr_) + svd + env)
    return np.array(cost)


def host_info():
    """nproc and the CPU model of the host the CPU legs ran on."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "threads_usable": cpu_threads(), "cpu_model": model}


def cpu_svd_timings(n, threads_all, reps_all=3, budget_s=240.0):
    """The reference's svd_full (linalg.cpp:67-70: thin SVD, U, sigma, V^T, then
    fix_phases) timed on the oracle (LAPACK gesdd, bundled OpenBLAS), as
    cmd_svd_bench does it (bench.cpp:635-668: random Gaussian n x n, complex as
    the reference literal, upper median of the repetitions), in complex128 and in
    real FP64, on all host threads and on one thread.  The one-thread legs run a
    single repetition each and are skipped (reported as null) once the budget is
    spent."""
    from oracle import oracle as O
    a_r = np.random.default_rng(1234).standard_normal((n, n))
    a_c = complex_literal(n)
    t_start = time.perf_counter()
    out = {}
    sig = {}

    def timed(kind, threads, reps):
        O.set_threads(threads)
        runs = []
        for _ in range(reps):
            t = time.perf_counter()
            if kind == "c128":
                sig["c128"] = O.svd_complex_sigma(a_c)
            else:
                sig["f64"] = O.svd(a_r)[1]
            runs.append(time.perf_counter() - t)
        runs.sort()
        return round(runs[len(runs) // 2] * 1e3, 1)

    for kind in ("f64", "c128"):
        out[f"{kind}_{threads_all}t_ms"] = timed(kind, threads_all, reps_all)
    for kind in ("f64", "c128"):
        if time.perf_counter() - t_start > budget_s:
            out[f"{kind}_1t_ms"] = None
            continue
        out[f"{kind}_1t_ms"] = timed(kind, 1, 1)
    O.set_threads(threads_all)
    out["note"] = (f"oracle svd_full (gesdd + fix_phases) on a random {n}x{n} matrix; "
                   f"{threads_all} threads: upper median of {reps_all}; 1 thread: one run "
                   f"(null: skipped, {budget_s:.0f} s budget)")
    out["seconds_spent"] = round(time.perf_counter() - t_start, 1)
    return out, sig


def complex_literal(n):
    """The cmd_svd_bench matrix (bench.cpp:646-648): complex Gaussian, re and im ~ N(0, 1)
    (numpy default_rng(4321) here, the reference draws from mt19937_64)."""
    rng = np.random.default_rng(4321)
    return rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))


def svd_complex_part(ctx, args):
    """The reference literal itself: complex n x n (n = 2 chi = 4096) svd_full on the
    device (achi_svd_complex_device: the realified matrix on the Jacobi engine).  One
    timed call after the data is resident (the call is seconds long)."""
    import torch
    n = 2 * args.svd_chi
    a = torch.from_numpy(complex_literal(n)).cuda()
    s = torch.empty(n, dtype=torch.float64, device="cuda")
    u = torch.empty(n, n, dtype=torch.complex128, device="cuda")
    vd = torch.empty(n, n, dtype=torch.complex128, device="cuda")
    torch.cuda.synchronize()
    ctx.flush_l2(256 << 20)
    ctx.timer_start()
    sweeps = ctx.svd_complex_device(a.data_ptr(), n, n, s.data_ptr(), u.data_ptr(), vd.data_ptr())
    ms = ctx.timer_stop()
    k = 64
    rec = float(((u[:k] * s) @ vd - a[:k]).abs().max() / s[0])
    fro = float((a.abs() ** 2).sum())
    out = {"svd_chi2048_c128_ms": round(ms, 1), "svd_chi2048_c128_jacobi_sweeps": sweeps,
           "svd_chi2048_c128_recon_err": rec,
           "svd_chi2048_c128_sum_sigma2_relerr": abs(float((s * s).sum()) - fro) / fro,
           "svd_chi2048_c128_note": "complex128 4096x4096 Gaussian (the cmd_svd_bench literal), "
                                    "U, sigma, V^dagger on the device via the realified 8192x8192 "
                                    "real Jacobi SVD"}
    del a, u, vd
    return out, s.cpu().numpy()


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- our arm
def log(msg):
    print(f"[bench] {msg}", file=sys.stderr, flush=True)


def c5_adaptive(ctx, args):
    """BASELINE configs[4] (C5), adaptive arm: Heisenberg S=1/2 N=200, PID chi_max=2048,
    eps_trunc=1e-10, predictive scheduler on (beta=0.4, linear), Neel start, run to
    convergence through the public API and timed on the device.  The fixed chi=2048 arm
    (~0.5 ks per full-chi sweep) is a tool run (tools/c5_run.py, profiles/r02/c5_r02.txt)."""
    from paper_2604_03960_b200.api import Chain
    spec = abi.model_spec(200, convention=abi.SPIN_HALF)
    cfg = abi.adaptive_config(2048, 1e-10, max_sweeps=args.c5_sweeps)
    ch = Chain(ctx, spec, cfg)
    ctx.synchronize()
    ctx.timer_start()
    t0 = time.perf_counter()
    res = ch.run()
    wall = time.perf_counter() - t0
    dev_ms = ctx.timer_stop()
    ch.close()
    return {"workload": "C5 adaptive: Heisenberg S=1/2 OBC N=200, PID/EMA chi_max=2048, eps_trunc=1e-10, "
                        "predictor linear beta=0.4, Neel start, run_dmrg to eps_conv=1e-8",
            "device_s": round(dev_ms / 1e3, 3), "wall_s": round(wall, 3), "sweeps": res["n_sweeps"],
            "converged": res["converged"], "e_per_site": res["energy"] / 200,
            "max_chi": int(res["max_chi_used"]),
            "sweep_s": [round(r.wall_time, 3) for r in res["records"]]}


PHASE_SAMPLE = 5


def run_ours(args, dist):
    from paper_2604_03960_b200.api import Chain, Context
    ctx = Context(dist.local)
    W, K = args.warmup, args.steps
    spec, cfg = workload(W + K)
    t0 = time.perf_counter()
    ch = Chain(ctx, spec, cfg)
    setup_s = time.perf_counter() - t0
    for s in range(W):
        ch.sweep(s)
    # phase events on one bond visit in PHASE_SAMPLE (coprime with the 198 visits of a
    # sweep, so the sample rotates over the bonds): the events cost ~4 us of device time
    # per timed visit, which would otherwise inflate the value by ~2.5 %
    ctx.device_times(enable=PHASE_SAMPLE, reset=True)
    launches0 = ctx.launches
    sampler = ClockSampler(dist.local)
    sampler.start()
    dev_ms, host_s, last, energies = [], [], None, []
    for i in range(K):
        ctx.flush_l2(256 << 20)  # > 126 MB L2: each timed sweep starts cold
        dist.barrier()
        ctx.timer_start()
        th = time.perf_counter()
        last = ch.sweep(W + i)  # public API call: returns the step's results to the host
        energies.append(last["energy"])
        host_s.append(time.perf_counter() - th)
        dev_ms.append(ctx.timer_stop())
    clocks = sampler.stop()
    log(f"timed sweeps done: {dev_ms}")
    launches = ctx.launches - launches0
    phases = ctx.device_times(enable=False)
    sweep_s = dist.max(float(np.mean(dev_ms)) / 1e3)
    e2e_s = dist.max(float(np.mean(host_s)))
    chi = last["chi_profile"]
    nb = N_SITES - 1
    d2h = 56 + nb * (4 + 8) + 2 * nb * (80 + 96)  # record + profiles + trace + visit rows
    hbm, hbm_src = peaks()
    # roofline of the dominant phase (by device time); both phases are FP64
    # tensor-core work (DMMA), latency-bound at the chi <= ~110 of C3
    svd, mv = phases["svd"], phases["matvec"]
    svd_tfs = svd["work"] / max(svd["ms"], 1e-9) / 1e9
    mv_tfs = mv["work"] / max(mv["ms"], 1e-9) / 1e9
    traffic = measured_traffic()
    roof_svd = {"bound": "tensor",
                "kernel": "jacobi_cluster_kernel + v_replay_kernel (blocked one-sided Jacobi SVD)",
                "achieved": round(svd_tfs, 4), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": round(svd_tfs / FP64_PEAK_TFLOPS, 6),
                "traffic": traffic.get("jacobi_cluster_kernel"),
                "work_def": "4*ng^2*(2*mg+ng) FP64 flops per Jacobi sweep (Gram + G and V "
                            "rotations of every block pair), summed over the sweeps of each SVD",
                "peak_source": "measured DMMA peak (profiles/fp64_peak_r01.txt)"}
    roof_mv = {"bound": "tensor",
               "kernel": "Lanczos eigensolve: lanczos_persistent_kernel (one launch per eigensolve "
                         "for chi <= 128: fused H_eff phases + CGS2 + tridiagonal CTA), else the "
                         "graph of dmma_gemm_kernel x2 + mpo_mix_kernel + lanczos_orth_kernel",
               "achieved": round(mv_tfs, 4), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
               "frac": round(mv_tfs / FP64_PEAK_TFLOPS, 6),
               "traffic": traffic.get("lanczos_persistent_kernel"),
               "work_def": "matvecs x (2*D*d^2*chl*chr*(chl+chr)+4*D^2*d^3*chl*chr) flops over the "
                           "eigensolve's device time (orthogonalisation and tridiagonal included)",
               "peak_source": "measured DMMA peak (profiles/fp64_peak_r01.txt)"}
    dominant = roof_svd if svd["ms"] >= mv["ms"] else roof_mv
    out = {
        "metric": METRIC, "value": round(sweep_s, 6), "unit": "s/sweep",
        "n_gpus": dist.world, "steps": K, "warmup": W, "ms_per_step": round(sweep_s * 1e3, 3),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Neel start, no input data)",
        "config": {"workload": "C3: Heisenberg S=1/2 OBC N=100, PID/EMA chi_max=1024, "
                               "eps_trunc=1e-10, timed sweeps W..W+K-1",
                   "n": N_SITES, "chi_max": CHI_MAX, "eps_trunc": EPS_TRUNC,
                   "parallelism": f"replicas x{dist.world} (a chain does not shard)",
                   "l2": "flushed (256 MB write) before every timed sweep"},
        "e_per_site": last["energy"] / N_SITES, "chi_max_seen": int(chi.max()),
        "e_per_site_bethe_limit": 0.25 - float(np.log(2.0)),
        "e_per_site_minus_bethe": last["energy"] / N_SITES - (0.25 - float(np.log(2.0))),
        "e_note": "Bethe ansatz 1/4 - ln 2 is the infinite-chain value; N=100 OBC sits above it by "
                  "the O(1/N) boundary energy",
        "delta_e_rel_last_sweep": (abs(energies[-1] - energies[-2]) / abs(energies[-1])
                                   if len(energies) > 1 else None),
        "chi_avg": round(float(chi.mean()), 2), "setup_s": round(setup_s, 4),
        "sweep_s": [round(m / 1e3, 4) for m in dev_ms],
        "phases_ms": {k: round(v["ms"], 3) for k, v in phases.items()},
        "phases_note": f"CUDA-event device time over one bond visit in {PHASE_SAMPLE} "
                       "(rooflines divide the same visits' algorithmic work by it)",
        "roofline": dominant, "roofline_lanczos": roof_mv, "roofline_svd": roof_svd,
        "e2e": {"value": round(e2e_s, 6), "unit": "s/sweep", "h2d_bytes_per_step": 4,
                "d2h_bytes_per_step": d2h,
                "note": "host wall time of the public Chain.sweep call incl. result readback; "
                        "the MPS/environments are device-resident (uploaded once at setup)"},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    gpu_csig = None
    if not args.skip_svd:
        log("svd part")
        out.update(svd_part(ctx, args))
        if not args.skip_complex_svd:
            log("complex svd part")
            cpart, gpu_csig = svd_complex_part(ctx, args)
            out.update(cpart)
    # K1 at the large-chi end of the metric's range (chi_max = 1024), measured inside a
    # real sweep: N=100, fixed chi=1024 (every bond 10..89 at chi=1024 from sweep 5 on)
    if not args.skip_heff_insweep:
        log("heff in-sweep (N=100, fixed chi=1024)")
        out["roofline_heff_chi1024"] = heff_insweep(ctx, args)
    if not args.skip_c5 and dist.rank == 0:
        log("C5 adaptive arm (N=200, PID chi_max=2048)")
        out["c5_adaptive"] = c5_adaptive(ctx, args)
    from paper_2604_03960_b200.api import heff_bench
    ms, tf = heff_bench(ctx, 1024, 10)
    out["heff_chi1024_microbench"] = {
        "achieved": round(tf, 3), "unit": "TFLOP/s", "frac": round(tf / FP64_PEAK_TFLOPS, 4),
        "ms_per_matvec": round(ms, 4),
        "note": "achi_heff_bench: random chi=1024 operands, device-resident, 10 matvecs"}
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        log("cpu baseline")
        out["cpu_baseline"] = cpu_baseline_sample(spec, cfg, ch, last)
        if not args.skip_svd:
            log("cpu svd baseline")
            cb, cpu_sig = cpu_svd_timings(2 * args.svd_chi, cpu_threads(), budget_s=args.cpu_svd_budget_s)
            if gpu_csig is not None and "c128" in cpu_sig:
                # parity of the complex literal at full size: device vs the oracle's zgesdd
                ref = cpu_sig["c128"]
                out["svd_chi2048_c128_sigma_vs_zgesdd"] = float(np.abs(gpu_csig - ref).max() / ref[0])
            out["cpu_baseline"]["svd_chi2048"] = cb
            thr = cpu_threads()
            out["svd_chi2048_cpu_ms"] = {k: v for k, v in cb.items() if k.endswith("_ms")}
            if cb.get(f"c128_{thr}t_ms") and "svd_chi2048_ms" in out:
                out["svd_chi2048_speedup"] = {
                    k.replace("_ms", ""): round(v / out["svd_chi2048_ms"], 2)
                    for k, v in cb.items() if k.endswith("_ms") and v}
    ch.close()
    ctx.close()
    if not args.skip_shards:
        out.update(shard_jobs(args, dist))
    return out


def shard_jobs(args, dist):
    """The naturally sharded workloads at this run's N GPUs:
    C4 (64-chain XXZ ensemble, LPT plan, chains in flight per GPU, one NCCL
    all_gather of the per-chain records) and C2 (a batch of isolated chi=1024
    SVDs, round robin, one all_gather).  Whole-job throughput, device time (CUDA
    events per worker stream), max over ranks."""
    from paper_2604_03960_b200 import ensemble_run as E
    res = {}
    ns = argparse.Namespace(chains=args.c4_chains, n=N_SITES, jz_max=2.0, chi_max=CHI_MAX,
                            eps=EPS_TRUNC, sweeps=10, inflight=4, grid_share=False,
                            batch=args.c2_batch, svd_chi=args.c2_chi)
    log("c4 ensemble")
    job_s, table, meta = E.job_c4(ns, dist.e)
    if table is not None and dist.rank == 0:
        t = np.asarray(table)
        res["c4_chains_per_s"] = round(args.c4_chains / job_s, 4)
        res["c4"] = {"chains": args.c4_chains, "device_s": round(job_s, 3),
                     "converged": int(t[:, 4].sum()), "max_chi": int(t[:, 3].max()),
                     "e_per_site_jz1": float(t[np.argmin(np.abs(t[:, 0] - 1.0)), 1]),
                     "workload": meta["config"]["workload"], "plan": meta["config"]["plan"],
                     "inflight_per_gpu": 4, "scaling": "strong (fixed 64 chains)"}
    log("c2 batch")
    job_s, table, meta = E.job_c2(ns, dist.e)
    if table is not None and dist.rank == 0:
        t = np.asarray(table)
        res["c2_svds_per_s"] = round(args.c2_batch / job_s, 4)
        res["c2"] = {"batch": args.c2_batch, "n": 2 * args.c2_chi, "device_s": round(job_s, 3),
                     "max_sum_sigma2_relerr": float(t[:, 2].max()),
                     "workload": meta["config"]["workload"], "plan": "round robin",
                     "scaling": "strong (fixed batch)"}
    return res


def heff_insweep(ctx, args):
    """H_eff TFLOP/s inside a real sweep at chi = 1024: Heisenberg
    N=100, fixed chi_max=1024 from the Neel state (chi grows x4 per sweep and reaches
    1024 on bonds 10..89 in sweep 5).  Sweep `args.heff_sweep` is measured with the
    Lanczos stepped from the host so that every H_eff application is bracketed by
    CUDA events on the library stream (phase "heff"; flops per matvec
    2 D d^2 chl chr (chl+chr) + 4 D^2 d^3 chl chr at each visit's own shape)."""
    from paper_2604_03960_b200.api import Chain
    s_idx = args.heff_sweep
    spec = abi.model_spec(N_SITES, convention=abi.SPIN_HALF)
    cfg = abi.fixed_config(CHI_MAX, max_sweeps=s_idx + 1, eps_conv=1e-300)
    ctx.set_lanczos_graph(0)
    ch = Chain(ctx, spec, cfg)
    oz = None
    try:
        for s in range(s_idx):
            ch.sweep(s)
        sites = ch.sites() if args.ozaki_slices > 0 else None
        ctx.device_times(enable=True, reset=True)
        ctx.timer_start()
        r = ch.sweep(s_idx)
        sweep_ms = ctx.timer_stop()
        ph = ctx.device_times(enable=False)
        if sites is not None:
            # the same sweep from the same state with every large contraction (H_eff,
            # environments, theta merge) on the emulated-FP64 int8 engine (ozaki.cu)
            ch.close()
            ch2 = Chain(ctx, spec, cfg)
            ch2.load_state(sites)
            del sites
            ctx.set_ozaki(args.ozaki_slices)
            try:
                ctx.device_times(enable=True, reset=True)
                ctx.timer_start()
                r2 = ch2.sweep(s_idx)
                ms2 = ctx.timer_stop()
                ph2 = ctx.device_times(enable=False)
            finally:
                ctx.set_ozaki(0)
                ch2.close()
            h2 = ph2["heff"]
            tf2 = h2["work"] / max(h2["ms"], 1e-9) / 1e9
            oz = {"digits": args.ozaki_slices, "achieved": round(tf2, 3), "unit": "TFLOP/s (FP64-equivalent)",
                  "frac_of_dmma_peak": round(tf2 / FP64_PEAK_TFLOPS, 4), "heff_ms": round(h2["ms"], 2),
                  "sweep_ms": round(ms2, 1),
                  "energy_rel_diff_vs_native": abs(r2["energy"] - r["energy"]) / abs(r["energy"]),
                  "chi_profile_equal": bool((r2["chi_profile"] == r["chi_profile"]).all()),
                  "note": "the same sweep from the same state, H_eff/environment/merge GEMMs of >= 1 GFLOP "
                          "on tcgen05.mma kind::i8 (Ozaki digits), everything else unchanged"}
    finally:
        ch.close()
        ctx.set_lanczos_graph(-1)
    h = ph["heff"]
    tf = h["work"] / max(h["ms"], 1e-9) / 1e9
    chi = r["chi_profile"]
    out = {"bound": "tensor",
            "kernel": "H_eff matvec in a real sweep (dmma_gemm_kernel x2 + mpo_mix_kernel; "
                      "heff_small_kernel at the chain ends)",
            "achieved": round(tf, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": round(tf / FP64_PEAK_TFLOPS, 4), "traffic": None,
            "matvecs": h["launches"], "heff_ms": round(h["ms"], 2),
            "sweep_ms": round(sweep_ms, 1), "phases_ms": {k: round(v["ms"], 1) for k, v in ph.items()},
            "bonds_at_chi1024": int((chi == 1024).sum()),
            "workload": f"N=100 Heisenberg S=1/2, fixed chi=1024, sweep {s_idx} of a Neel start",
            "work_def": "sum over the sweep's matvecs of 2*D*d^2*chl*chr*(chl+chr)+4*D^2*d^3*chl*chr "
                        "flops / sum of their CUDA-event times",
            "peak_source": "measured DMMA peak (profiles/fp64_peak_r01.txt)"}
    if oz is not None:
        out["emulated_fp64"] = oz
    return out


def svd_part(ctx, args):
    """Truncated-SVD half of the metric: random 4096x4096 FP64 theta (chi=2048)."""
    import torch
    n = 2 * args.svd_chi
    # the matrix tests/golden/svd_sigma_large.json pins (sigma vs LAPACK dgesdd,
    # tests/test_golden_long.py): numpy default_rng(1234), uploaded once
    a = torch.from_numpy(np.random.default_rng(1234).standard_normal((n, n))).cuda()
    s = torch.empty(n, dtype=torch.float64, device="cuda")
    u = torch.empty(n, n, dtype=torch.float64, device="cuda")
    vt = torch.empty(n, n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    # svd_full with both factors (the reference's svd_truncated computes the full SVD)
    ctx.svd_device(a.data_ptr(), n, n, s.data_ptr(), u.data_ptr(), vt.data_ptr())  # warm-up
    ms, sweeps = [], 0
    for _ in range(args.svd_reps):
        ctx.flush_l2(256 << 20)
        ctx.timer_start()
        sweeps = ctx.svd_device(a.data_ptr(), n, n, s.data_ptr(), u.data_ptr(), vt.data_ptr())
        ms.append(ctx.timer_stop())
    fro = float((a * a).sum())
    err = abs(float((s * s).sum()) - fro) / fro
    k = 64  # reconstruction spot check on the leading rows
    rec = float(((u[:k] * s) @ vt - a[:k]).abs().max() / s[0])
    # e2e through the host-buffer API (H2D of theta, D2H of U, sigma, V^T inside the timed
    # region) on pinned host buffers, one untimed warm-up call, median of svd_reps calls
    pin = lambda *shape: torch.empty(*shape, dtype=torch.float64, pin_memory=True)  # noqa: E731
    ha = pin(n, n)
    ha.copy_(a)
    ha = ha.numpy()
    hout = (pin(n, n).numpy(), pin(n).numpy(), pin(n, n).numpy())
    ctx.svd_full(ha, out=hout)
    e2e_s = []
    for _ in range(args.svd_reps):
        ctx.flush_l2(256 << 20)
        torch.cuda.synchronize()
        t = time.perf_counter()
        ctx.svd_full(ha, out=hout)
        e2e_s.append(time.perf_counter() - t)
    e2e = statistics.median(e2e_s)
    hbm, _ = peaks()
    med = statistics.median(ms)
    # every round of a sweep reads G (n x n) for the block-pair Grams and reads + writes it
    # for the rotations (24 bytes per element); a sweep has n/16 - 1 rounds.  V is not
    # rotated: it is recovered after the sweeps by three n^3 GEMMs (svd_jacobi.cu v_recover)
    gbs = 24.0 * sweeps * (n // 16 - 1) * (n * n) / (med * 1e-3) / 1e9
    # 16 (mn + n^2) bytes per Jacobi sweep
    gbs_d3 = 16.0 * sweeps * (n * n + n * n) / (med * 1e-3) / 1e9
    # FP64 flops: Gram + rotation of every block pair, 8 m n^2 per sweep, plus the recovery
    tfs = (8.0 * sweeps * n ** 3 + 3 * 2.0 * n ** 3) / (med * 1e-3) / 1e12
    return {"svd_chi2048_ms": round(med, 3), "svd_chi2048_e2e_ms": round(e2e * 1e3, 3),
            "svd_chi2048_sweeps": sweeps, "svd_chi2048_sum_sigma2_relerr": err,
            "svd_chi2048_recon_err": rec, "svd_chi2048_factors": "U, sigma, V^T (svd_full)",
            "svd_chi2048_roofline": {"bound": "hbm", "kernel": "jacobi_stream_kernel",
                                     "achieved": round(gbs, 2), "peak": hbm,
                                     "unit": "GB/s", "frac": round(gbs / hbm, 5),
                                     "traffic": measured_traffic().get("jacobi_stream_kernel"),
                                     "work_def": "24*(n/16-1)*n^2 bytes per Jacobi sweep (G read "
                                                 "for the Grams, read+written for the rotations, "
                                                 "every round); V recovered by GEMM afterwards",
                                     "frac_s8d3": round(gbs_d3 / hbm, 6),
                                     "tensor": {"achieved": round(tfs, 3), "peak": FP64_PEAK_TFLOPS,
                                                "unit": "TFLOP/s",
                                                "frac": round(tfs / FP64_PEAK_TFLOPS, 4),
                                                "work_def": "8 n^3 FP64 flops per Jacobi sweep "
                                                            "+ 6 n^3 (V recovery GEMMs)"}}}


def cpu_baseline_sample(spec, cfg, ch, last):
    """Oracle port (complex128, all host threads) on a bounded sample: 20 right-moving
    visits at the chain centre from the steady-state MPS, extrapolated to the full
    sweep with a FLOP model weighted by this run's own visit records."""
    from oracle import oracle as O
    threads = cpu_threads()
    O.set_threads(threads)
    sites = [ch.site(k) for k in range(N_SITES)]
    states = ch.states()
    first, count = 40, 20
    secs, mvs = O.time_visits_from_state(spec, cfg, sites, states, first, count, complex_mode=True)
    chi = last["chi_profile"]

    class V:
        def __init__(self, bond, matvecs, kept):
            self.bond, self.matvecs, self.kept = bond, matvecs, kept
    sample = [V(first + i, int(mvs[i]), int(chi[first + i])) for i in range(count)]
    c_sample = visit_cost_model(sample, chi).sum()
    c_full = visit_cost_model(last["visits"], chi).sum()
    est = float(secs.sum()) * c_full / c_sample
    secs_r, mvs_r = O.time_visits_from_state(spec, cfg, sites, states, first, count,
                                             complex_mode=False)
    est_r = float(secs_r.sum()) * c_full / c_sample
    return {"value": round(est, 3), "unit": "s/sweep", "cores": threads, "kind": "port",
            "sample": f"{count} right-moving visits (bonds {first}..{first + count - 1}) of the "
                      f"steady-state sweep on the oracle (complex128, OpenBLAS {threads} threads): "
                      f"{secs.sum():.2f} s, extrapolated to all {2 * (N_SITES - 1)} visits by FLOP "
                      f"model (matvecs x H_eff flops + SVD + env)",
            "real_fp64": {"value": round(est_r, 3), "unit": "s/sweep",
                          "sample": f"the same {count} visits in the real gauge (FP64, the GPU "
                                    f"path's arithmetic): {secs_r.sum():.2f} s, same extrapolation"},
            "host": host_info()}


# ---------------------------------------------------------------- reference arm
def run_reference(args, dist):
    """The reference algorithm (oracle port of proj/src, complex128) on the host cores."""
    if dist.rank != 0:
        return None
    from oracle import oracle as O
    threads = cpu_threads()
    O.set_threads(threads)
    W, K = args.warmup, args.steps
    spec, cfg = workload(W + K)
    cfg.eps_conv = 1e-300  # time fixed sweeps (no early stop), as the GPU arm does
    ch = O.OracleChain(spec, cfg, complex_mode=True)
    for s in range(W):
        ch.sweep(s)
    walls, budget_hit = [], False
    t0 = time.perf_counter()
    for i in range(K):
        rec, chi = ch.sweep(W + i)
        walls.append(rec.wall_time)
        if time.perf_counter() - t0 > args.ref_budget_s:
            budget_hit = i + 1 < K
            break
    ch.close()
    v = float(np.mean(walls))
    sample = (f"sweeps {W}..{W + len(walls) - 1} of the C3 run, full sweeps, complex128, "
              f"OpenBLAS {threads} threads" + (f" (stopped after {len(walls)} of {K} steps: "
                                               f"{args.ref_budget_s:.0f} s budget)" if budget_hit else ""))
    # the same sweeps in the real gauge (FP64: the GPU path's arithmetic), budgeted
    real_walls = []
    if not args.skip_real:
        ch = O.OracleChain(spec, cfg, complex_mode=False)
        for s_ in range(W):
            ch.sweep(s_)
        t0 = time.perf_counter()
        for i in range(len(walls)):
            rec_r, _ = ch.sweep(W + i)
            real_walls.append(rec_r.wall_time)
            if time.perf_counter() - t0 > args.real_budget_s:
                break
        ch.close()
    svd = None if args.skip_svd else cpu_svd_timings(2 * args.svd_chi, threads, reps_all=3,
                                                      budget_s=0.0)[0]
    return {"metric": METRIC, "value": round(v, 4), "unit": "s/sweep", "impl": "reference",
            "n_gpus": dist.world, "steps": len(walls), "warmup": W,
            "ms_per_step": round(v * 1e3, 2), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (Neel start)",
            "config": {"workload": "C3: Heisenberg S=1/2 OBC N=100, PID/EMA chi_max=1024, "
                                   "eps_trunc=1e-10", "n": N_SITES, "chi_max": CHI_MAX},
            "e_per_site": rec.energy / N_SITES, "chi_max_seen": int(chi.max()),
            "sweep_s": [round(w, 4) for w in walls],
            "real_fp64": None if not real_walls else {
                "value": round(float(np.mean(real_walls)), 4), "unit": "s/sweep",
                "sweeps": f"{W}..{W + len(real_walls) - 1}",
                "sweep_s": [round(w, 4) for w in real_walls],
                "note": "same run in the real gauge (identical energies and chi profiles to 1e-12)"},
            "svd_chi2048_ms": None if svd is None else svd[f"c128_{threads}t_ms"],
            "svd_chi2048_cpu_ms": svd,
            "host": host_info(),
            "cpu_baseline": {"value": round(v, 4), "unit": "s/sweep", "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": round(v, 4), "unit": "s/sweep", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    faulthandler.enable()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--svd-chi", type=int, default=2048)
    ap.add_argument("--svd-reps", type=int, default=3)
    ap.add_argument("--skip-svd", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=600.0)
    ap.add_argument("--cpu-svd-budget-s", type=float, default=150.0)
    ap.add_argument("--skip-shards", action="store_true")
    ap.add_argument("--skip-complex-svd", action="store_true")
    ap.add_argument("--skip-heff-insweep", action="store_true")
    ap.add_argument("--heff-sweep", type=int, default=5)
    ap.add_argument("--ozaki-slices", type=int, default=7,
                    help="digits of the emulated-FP64 leg of the in-sweep H_eff measurement (0: skip)")
    ap.add_argument("--skip-real", action="store_true")
    ap.add_argument("--skip-c5", action="store_true")
    ap.add_argument("--c5-sweeps", type=int, default=12)
    ap.add_argument("--real-budget-s", type=float, default=100.0)
    ap.add_argument("--c4-chains", type=int, default=64)
    ap.add_argument("--c2-batch", type=int, default=64)
    ap.add_argument("--c2-chi", type=int, default=1024)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # contract: W >= 3
    dist = Dist()
    out = run_reference(args, dist) if args.impl == "reference" else run_ours(args, dist)
    if dist.rank == 0 and out is not None:
        print(json.dumps(out), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
