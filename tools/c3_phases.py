"""Per-sweep device phase split of the C3 run (sweeps 0..S-1): eigensolve, SVD, environment."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_03960_b200 import abi
from paper_2604_03960_b200.api import Context, Chain
S = int(sys.argv[1]) if len(sys.argv) > 1 else 25
ctx = Context(0)
ch = Chain(ctx, abi.model_spec(100, convention=abi.SPIN_HALF), abi.adaptive_config(1024, 1e-10, max_sweeps=S))
for s in range(S):
    ctx.device_times(enable=True, reset=True)
    ctx.timer_start()
    r = ch.sweep(s)
    ms = ctx.timer_stop()
    ph = ctx.device_times(enable=False)
    mv = sum(v.matvecs for v in r["visits"])
    print(f"sweep {s:2d} {ms:7.1f} ms  eig {ph['matvec']['ms']:6.1f}  svd {ph['svd']['ms']:6.1f}  env {ph['env']['ms']:5.1f}"
          f"  other {ms - ph['matvec']['ms'] - ph['svd']['ms'] - ph['env']['ms']:5.1f}  matvecs {mv}  maxchi {int(r['chi_profile'].max())}",
          flush=True)
