import sys
sys.path.insert(0, '.')
from paper_2604_03960_b200.api import Context, heff_bench
ctx = Context(0)
for chi in [int(x) for x in (sys.argv[1:] or ["64", "128", "256", "512", "1024", "2048"])]:
    ms, tf = heff_bench(ctx, chi, 10 if chi >= 1024 else 50)
    print(f"chi={chi} ms={ms:.3f} TFLOP/s={tf:.2f} frac={tf/37.1:.3f}", flush=True)
