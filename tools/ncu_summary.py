"""Summarise an ncu --csv launch list: share of device time per kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]
ki, vi, mi = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Name')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
        continue
    name = r[ki].split('(')[0][:80]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(',', ''))
tot = sum(v[1] for v in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t / tot * 100:6.2f}%  n={c:5d}  avg={t / c / 1000:9.2f} us  {k}")
print(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")
