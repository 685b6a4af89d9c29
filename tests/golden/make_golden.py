"""Generate the golden fixtures under tests/golden/ from the CPU oracle.

Test infrastructure only (run here, where the oracle builds; the fixtures
travel to the GPU box, the oracle is not needed there for
tests/test_golden_fixtures.py's GPU half).  The reference itself cannot be
built in this image (Eigen/doctest/json/CLI11 absent), so
the fixtures are outputs of the oracle, which tests/test_oracle_golden.py pins
to every known answer of the reference suite.  Each case names the reference
config it restates.

    python tests/golden/make_golden.py          # rewrites tests/golden/*.json
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


def run_case(name, spec, cfg, complex_mode, source):
    t0 = time.time()
    r = O.run_dmrg(spec, cfg, complex_mode=complex_mode)
    return dict(
        name=name, source=source, complex_mode=complex_mode,
        spec=dict(n=spec.n, family=spec.family, jx=spec.jx, jy=spec.jy, jz=spec.jz, h=spec.h,
                  convention=spec.convention),
        energies=[float(e) for e in r["energies"]],
        energy=float(r["energy"]), n_sweeps=int(r["n_sweeps"]), converged=bool(r["converged"]),
        chi_profiles=r["chi_profiles"].tolist(),
        entropy_profiles=r["entropy_profiles"].tolist(),
        kept=[int(v.kept) for v in r["visits"]],
        trace_chi=[int(t.chi) for t in r["trace"]],
        oracle_seconds=round(time.time() - t0, 2),
    )


def svd_cases():
    out = []
    for seed, (m, n) in [(11, (64, 64)), (12, (48, 80)), (13, (130, 96)), (14, (256, 256))]:
        a = np.random.default_rng(seed).standard_normal((m, n))
        _, s, _ = O.svd(a)
        out.append(dict(seed=seed, m=m, n=n, generator="numpy default_rng(seed).standard_normal((m, n))",
                        sigma=[float(x) for x in s]))
    return out


def main():
    O.set_threads(os.cpu_count() or 1)
    cases = [
        run_case("c1", abi.model_spec(20), abi.fixed_config(32, max_sweeps=5), True,
                 "BASELINE.json configs[0]: Heisenberg N=20 fixed chi=32, 5 sweeps (complex128, as the reference)"),
        run_case("criterion2_pid", abi.model_spec(20), abi.adaptive_config(64, 1e-5), True,
                 "acceptance_main.cpp:106-126: N=20 Pauli PID chi_max=64 eps 1e-5 (complex128)"),
        run_case("c3_3sweeps", abi.model_spec(100, convention=abi.SPIN_HALF),
                 abi.adaptive_config(1024, 1e-10, max_sweeps=3, eps_conv=1e-300), False,
                 "BASELINE.json configs[2] (C3), first 3 sweeps, real-gauge oracle"),
    ]
    for c in cases:
        with open(os.path.join(HERE, f"dmrg_{c['name']}.json"), "w") as f:
            json.dump(c, f, indent=None, separators=(",", ":"))
        print(c["name"], c["n_sweeps"], c["energy"], f"{c['oracle_seconds']} s")
    with open(os.path.join(HERE, "svd_sigma.json"), "w") as f:
        json.dump(svd_cases(), f, separators=(",", ":"))


if __name__ == "__main__":
    main()
