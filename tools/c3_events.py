"""C3 sweeps 5..24 device time with and without the per-phase CUDA-event accounting."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_03960_b200 import abi
from paper_2604_03960_b200.api import Context, Chain
ctx = Context(0)
for acc in (5, 0, 1, 5):
    ch = Chain(ctx, abi.model_spec(100, convention=abi.SPIN_HALF), abi.adaptive_config(1024, 1e-10, max_sweeps=25))
    for s in range(5):
        ch.sweep(s)
    ctx.device_times(enable=acc, reset=True)
    ms = []
    for s in range(5, 25):
        ctx.flush_l2(256 << 20)
        ctx.timer_start()
        ch.sweep(s)
        ms.append(ctx.timer_stop())
    ctx.device_times(enable=False)
    print(f"events={acc} mean {sum(ms) / len(ms):.2f} ms steady {sum(ms[-5:]) / 5:.2f}", flush=True)
    ch.close()
