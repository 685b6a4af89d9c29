"""Reproduce a DMRG run through the C-ABI with given model args (debug helper)."""
import sys
from paper_2604_03960_b200 import abi
from paper_2604_03960_b200.api import Context

n, h = int(sys.argv[1]), float(sys.argv[2])
spec = abi.model_spec(n, family=abi.TRANSVERSE_ISING, jz=1.0, h=h)
cfg = abi.fixed_config(1 << (n // 2), eps_conv=1e-11, max_sweeps=16)
cfg.eig_tol, cfg.eig_max_iter = 1e-12, 400
ctx = Context(0)
try:
    r = ctx.run_dmrg(spec, cfg)
    print("ok", r["energy"], r["n_sweeps"])
except Exception as e:
    print("FAIL", e)
