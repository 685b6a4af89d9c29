"""Long-run golden fixtures from the CPU oracle (test infrastructure only).

These cover what bench.py times and what the reference's slow acceptance tier
runs, so the GPU suite can compare visit by visit without running the oracle
on the box:

* dmrg_c3_long.json   C3 (BASELINE.json configs[2]): Heisenberg S=1/2 N=100, PID
                      chi_max=1024, eps_trunc=1e-10, sweeps 0..24 with no early
                      stop (bench.py times sweeps W..W+K-1 = 5..24 by default).
* dmrg_criterion5.json reference acceptance criterion 5
                      (acceptance_main.cpp:176-201): N=64 spin-1/2, PID chi_max=128,
                      eps 1e-10, max 30 sweeps; the reference recorded
                      E/N = -0.440241 (proj/test_output.txt:19).
* svd_sigma_large.json sigma of the random n x n matrices (n = 1024, 2048, 4096) that
                      bench.py times, from the oracle's svd_full (LAPACK dgesdd).
* dmrg_c4_jz0p5.json, dmrg_c4_jz1p5.json   two C4 chains (configs[3]): N=100
                      spin-1/2 XXZ at Jz=0.5 (critical) and 1.5 (gapped), C3
                      controller settings, 10 sweeps (ensemble_run.py default).
* dmrg_c5_adaptive.json  C5 adaptive arm (configs[4]) as bench.py runs it: N=200,
                      PID chi_max=2048, eps 1e-10, to convergence (max 12 sweeps).

Every visit row carries the decision inputs (floor rank, its margin
|tail - eps*total|/(eps*total), significant count, sigma_kept/sigma_1,
sigma_next/sigma_1) so a kept-rank divergence on the GPU can be attributed to
a threshold within rounding.  The real-gauge oracle is used (identical to the
complex128 restatement to 1e-12 with identical chi profiles,
tests/test_oracle_golden.py::test_real_gauge_run_equals_complex_reference).

    python tests/golden/make_golden_long.py [svd|c3|crit5|c4|c5] ...
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2604_03960_b200 import abi  # noqa: E402
from oracle import oracle as O  # noqa: E402

VISIT_COLS = ["sweep", "bond", "moving_right", "kept", "floor_rank", "significant", "n_sigma",
              "matvecs", "degenerate_cut", "energy", "entropy", "trunc_error", "floor_margin",
              "sigma_kept", "sigma_next"]


def run_case(name, spec, cfg, source):
    t0 = time.time()
    r = O.run_dmrg(spec, cfg, complex_mode=False)
    visits = [[getattr(v, c) for c in VISIT_COLS] for v in r["visits"]]
    out = dict(
        name=name, source=source, complex_mode=False,
        spec=dict(n=spec.n, family=spec.family, jx=spec.jx, jy=spec.jy, jz=spec.jz, h=spec.h,
                  convention=spec.convention),
        config=dict(chi_max=cfg.controller.chi_max, eps_trunc=cfg.controller.eps_trunc,
                    mode=cfg.controller.mode, max_sweeps=cfg.max_sweeps, eps_conv=cfg.eps_conv),
        energies=[float(e) for e in r["energies"]],
        energy=float(r["energy"]), n_sweeps=int(r["n_sweeps"]), converged=bool(r["converged"]),
        max_chi_used=int(r["max_chi_used"]),
        chi_profiles=r["chi_profiles"].tolist(),
        entropy_profiles=r["entropy_profiles"].tolist(),
        trace=[[int(t.chi), int(t.delta_chi), int(t.clamped)] for t in r["trace"]],
        visit_cols=VISIT_COLS, visits=visits,
        oracle_seconds=round(time.time() - t0, 2), oracle_threads=os.cpu_count(),
    )
    with open(os.path.join(HERE, f"dmrg_{name}.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(name, out["n_sweeps"], out["energy"] / spec.n, f"{out['oracle_seconds']} s", flush=True)


def svd_large():
    """sigma of the random n x n matrices bench.py times (C2 sizes chi = 512, 1024, 2048;
    chi = 2048 is the metric's truncated SVD), from the oracle's svd_full (LAPACK dgesdd)."""
    out = []
    for chi in (512, 1024, 2048):
        n = 2 * chi
        a = np.random.default_rng(1234).standard_normal((n, n))
        t0 = time.time()
        _, s, _ = O.svd(a)
        out.append(dict(seed=1234, m=n, n=n, chi=chi,
                        generator="numpy default_rng(1234).standard_normal((n, n))",
                        sigma=[float(x) for x in s], oracle_seconds=round(time.time() - t0, 2)))
        print("svd", n, out[-1]["oracle_seconds"], flush=True)
    with open(os.path.join(HERE, "svd_sigma_large.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))


def main(which):
    O.set_threads(os.cpu_count() or 1)
    if "svd" in which:
        svd_large()
    if "c3" in which:
        run_case("c3_long", abi.model_spec(100, convention=abi.SPIN_HALF),
                 abi.adaptive_config(1024, 1e-10, max_sweeps=25, eps_conv=1e-300),
                 "BASELINE.json configs[2] (C3), sweeps 0..24 (bench window), real-gauge oracle")
    if "crit5" in which:
        cfg = abi.adaptive_config(128, 1e-10, max_sweeps=30)
        run_case("criterion5", abi.model_spec(64, convention=abi.SPIN_HALF), cfg,
                 "acceptance_main.cpp:176-201 criterion 5: N=64 spin-1/2 PID chi_max=128 eps 1e-10, "
                 "30 sweeps max; reference E/N -0.440241 (test_output.txt:19)")
    if "c4" in which:
        for jz, tag in ((0.5, "0p5"), (1.5, "1p5")):
            run_case(f"c4_jz{tag}", abi.model_spec(100, jz=jz, convention=abi.SPIN_HALF),
                     abi.adaptive_config(1024, 1e-10, max_sweeps=10),
                     f"BASELINE.json configs[3] (C4) chain Jz={jz}: N=100 PID chi_max=1024 "
                     "eps 1e-10, 10 sweeps (ensemble_run.py defaults)")
    if "c5" in which:
        run_case("c5_adaptive", abi.model_spec(200, convention=abi.SPIN_HALF),
                 abi.adaptive_config(2048, 1e-10, max_sweeps=12),
                 "BASELINE.json configs[4] (C5) adaptive arm as bench.py runs it: N=200 spin-1/2 "
                 "PID chi_max=2048 eps 1e-10, predictor linear beta=0.4, to eps_conv=1e-8 (max 12 sweeps)")


if __name__ == "__main__":
    main(sys.argv[1:] or ["svd", "c3", "crit5", "c4", "c5"])
