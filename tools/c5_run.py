"""Config C5: N=200 Heisenberg (spin-1/2), fixed chi=2048 vs PID chi_max=2048.

Runs whole sweeps through the public Chain API until --sweeps or --budget seconds,
printing one JSON line per sweep (device-resident state; the fixed arm exercises
the TMA H_eff and streamed-SVD paths at full size)."""
import argparse, json, sys, time
sys.path.insert(0, '.')
from paper_2604_03960_b200 import abi
from paper_2604_03960_b200.api import Context, Chain

ap = argparse.ArgumentParser()
ap.add_argument('--mode', choices=['fixed', 'pid'], default='fixed')
ap.add_argument('--n', type=int, default=200)
ap.add_argument('--chi', type=int, default=2048)
ap.add_argument('--sweeps', type=int, default=2)
ap.add_argument('--budget', type=float, default=1200)
a = ap.parse_args()
ctx = Context(0)
spec = abi.model_spec(a.n, convention=abi.SPIN_HALF)
cfg = (abi.fixed_config(a.chi, max_sweeps=a.sweeps) if a.mode == 'fixed'
       else abi.adaptive_config(a.chi, 1e-10, max_sweeps=a.sweeps))
t0 = time.time()
ch = Chain(ctx, spec, cfg)
print(json.dumps({"setup_s": round(time.time() - t0, 3), "mode": a.mode, "n": a.n, "chi": a.chi}), flush=True)
start = time.time()
for s in range(a.sweeps):
    r = ch.sweep(s)
    chi = r['chi_profile']
    print(json.dumps({"sweep": s, "wall_s": round(r['record'].wall_time, 3), "e_per_site": r['energy'] / a.n,
                      "max_chi": int(max(chi)), "avg_chi": float(sum(chi)) / len(chi),
                      "max_trunc_err": r['record'].max_trunc_error}), flush=True)
    if time.time() - start > a.budget:
        break
