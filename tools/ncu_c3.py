"""Short C3 run for ncu launch lists: sweeps 0..S-1 (steady state from ~sweep 4)."""
import sys
sys.path.insert(0, '.')
from paper_2604_03960_b200 import abi
from paper_2604_03960_b200.api import Context, Chain
S = int(sys.argv[1]) if len(sys.argv) > 1 else 6
ctx = Context(0)
spec = abi.model_spec(100, convention=abi.SPIN_HALF)
ch = Chain(ctx, spec, abi.adaptive_config(1024, 1e-10, max_sweeps=S))
for s in range(S):
    r = ch.sweep(s)
    print(s, r['energy'] / 100, int(r['chi_profile'].max()), ctx.launches, flush=True)
ch.close(); ctx.close()
