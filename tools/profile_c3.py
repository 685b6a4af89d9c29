"""Per-sweep profile of config C3 (Heisenberg N=100 spin-1/2, PID, chi_max)."""
import argparse, json, sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_2604_03960_b200 import abi
from paper_2604_03960_b200.api import Context, Chain

ap = argparse.ArgumentParser()
ap.add_argument('--n', type=int, default=100)
ap.add_argument('--chi', type=int, default=1024)
ap.add_argument('--sweeps', type=int, default=10)
ap.add_argument('--budget', type=float, default=400)
ap.add_argument('--profile', type=int, default=1)
a = ap.parse_args()
ctx = Context(0)
spec = abi.model_spec(a.n, convention=abi.SPIN_HALF)
cfg = abi.adaptive_config(a.chi, 1e-10, max_sweeps=a.sweeps)
t0 = time.time()
ch = Chain(ctx, spec, cfg)
ch.stats(profile=bool(a.profile))
print(f"setup {time.time()-t0:.2f}s", flush=True)
prev = ch.stats()
tstart = time.time()
for s in range(a.sweeps):
    r = ch.sweep(s)
    st = ch.stats()
    dlt = {k: st[k] - prev[k] for k in st}
    prev = st
    chi = r['chi_profile']
    print(json.dumps(dict(sweep=s, wall=round(r['record'].wall_time, 3), e_per_site=r['energy'] / a.n,
                          max_chi=int(chi.max()), avg_chi=round(float(chi.mean()), 1),
                          lanczos=round(dlt['lanczos_s'], 3), svd=round(dlt['svd_s'], 3),
                          select=round(dlt['select_s'], 3), env=round(dlt['absorb_env_s'], 3),
                          matvecs=int(dlt['matvecs']), svd_sweeps=int(dlt['svd_sweeps']))), flush=True)
    if time.time() - tstart > a.budget:
        print("budget reached", flush=True)
        break
print("chi profile", ch.bond_dims().tolist())
