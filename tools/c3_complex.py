"""C3 in complex128 (ACHI_ARITH_COMPLEX, the reference's arithmetic) on the device:
Heisenberg S=1/2 N=100, PID chi_max=1024, eps 1e-10, Neel start; per-sweep device ms
and energies, next to the real chain's."""
import sys, time
sys.path.insert(0, '.')
from paper_2604_03960_b200 import abi
from paper_2604_03960_b200.api import Context, Chain
S = int(sys.argv[1]) if len(sys.argv) > 1 else 10
ctx = Context(0)
spec = abi.model_spec(100, convention=abi.SPIN_HALF)
for arith in ([int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else (1, 0)):
    cfg = abi.adaptive_config(1024, 1e-10, max_sweeps=S)
    cfg.arithmetic = arith
    ch = Chain(ctx, spec, cfg)
    ctx.device_times(enable=True, reset=True)
    for s in range(S):
        ctx.timer_start()
        r = ch.sweep(s)
        ms = ctx.timer_stop()
        print(f"arith={arith} sweep {s} ms {ms:.1f} E/N {r['energy'] / 100:.14f} maxchi {int(r['chi_profile'].max())}",
              flush=True)
    ph = ctx.device_times(enable=False)
    print(f"arith={arith} phases", {k: round(v["ms"], 1) for k, v in ph.items()}, flush=True)
    ch.close()
