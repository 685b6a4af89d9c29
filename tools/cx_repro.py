import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_03960_b200 import abi
from paper_2604_03960_b200.api import Context, Chain
ctx = Context(0)
n, chi, S = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cfg = abi.adaptive_config(chi, 1e-10, max_sweeps=S)
cfg.arithmetic = 1
ch = Chain(ctx, abi.model_spec(n, convention=abi.SPIN_HALF), cfg)
prev = None
for s in range(S):
    r = ch.sweep(s)
    e = r["energy"] / n
    bad = prev is not None and e < prev - 1e-6
    print(f"n={n} chi={chi} sweep {s} E/N {e:.14f} maxchi {int(r['chi_profile'].max())}{'  <-- BAD' if bad else ''}", flush=True)
    prev = e
