"""Warm vs cold SVD statistics per C3 sweep from ACHI_VISIT_LOG=2 output (stdin)."""
import re, sys, collections
st = collections.defaultdict(lambda: [0, 0, 0, 0.0, 0.0])  # warm, cold, jacobi sweeps cold, svd ms warm, cold
for line in sys.stdin:
    m = re.search(r"sweep (\d+) bond (\d+) (\w) chl (\d+) chr (\d+) lanczos ([\d.]+) ms svd ([\d.]+) ms \((\d+) Jacobi sweeps, warm (\d)\)", line)
    if not m:
        continue
    s, warm, js, ms = int(m.group(1)), int(m.group(9)), int(m.group(8)), float(m.group(7))
    e = st[s]
    if warm:
        e[0] += 1; e[3] += ms
    else:
        e[1] += 1; e[2] += js; e[4] += ms
for s in sorted(st):
    w, c, js, mw, mc = st[s]
    print(f"sweep {s}: warm {w} (svd {mw:.1f} ms host) cold {c} (svd {mc:.1f} ms host, {js / max(c, 1):.1f} Jacobi sweeps avg)")
