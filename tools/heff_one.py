"""A few device-resident H_eff matvecs at one chi (for ncu captures)."""
import sys
sys.path.insert(0, '.')
from paper_2604_03960_b200.api import Context, heff_bench
chi = int(sys.argv[1]) if len(sys.argv) > 1 else 110
ctx = Context(0)
ms, tf = heff_bench(ctx, chi, 5)
print(chi, ms, tf)
