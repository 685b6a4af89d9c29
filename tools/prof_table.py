"""Compact table of tools/profile_c3.py JSON lines (stdin)."""
import json
import sys
for line in sys.stdin:
    if line.startswith("{"):
        d = json.loads(line)
        print(f"sweep {d['sweep']:2d} wall {d['wall']:.3f} lanczos {d['lanczos']:.3f} svd {d['svd']:.3f} "
              f"matvecs {d['matvecs']} svd_sweeps {d['svd_sweeps']} E/N {d['e_per_site']:.13f}")
