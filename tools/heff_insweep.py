"""In-sweep H_eff at chi = 1024 for ncu: Heisenberg N=100, fixed chi=1024 from the Neel
state, Lanczos stepped from the host (every kernel launched from the host so ncu sees
it).  Prints the library launch count at the start of each sweep; with --stop S it
ends after sweep S.  usage: python tools/heff_insweep.py [S]"""
import sys
sys.path.insert(0, '.')
from paper_2604_03960_b200 import abi
from paper_2604_03960_b200.api import Context, Chain
S = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ctx = Context(0)
ctx.set_lanczos_graph(0)
ch = Chain(ctx, abi.model_spec(100, convention=abi.SPIN_HALF), abi.fixed_config(1024, max_sweeps=S + 1))
for s in range(S + 1):
    print("sweep", s, "launches_at_start", ctx.launches, flush=True)
    r = ch.sweep(s)
    print("  E/N", r['energy'] / 100, "max chi", int(r['chi_profile'].max()), flush=True)
ch.close(); ctx.close()
