# cluster-path Jacobi phase split (ACHI_JACOBI_PROF=1) over C3 sweeps 0..11, aggregated
mkdir -p gpurun_out/$1
ACHI_JACOBI_PROF=1 timeout 600 python tools/ncu_c3.py 12 > gpurun_out/$1/c3.txt 2> gpurun_out/$1/prof_raw.txt
python - "$1" <<'PY'
import re, sys
tot = {}; n = 0; rounds = 0
for line in open(f"gpurun_out/{sys.argv[1]}/prof_raw.txt"):
    m = re.search(r"rounds=(\d+) rotated=(\d+) cycles/round: gram (\S+) inner (\S+) jrec (\S+) rotate (\S+) barrier (\S+)", line)
    if not m: continue
    r = int(m.group(1)); n += 1; rounds += r
    for k, v in zip(("gram", "inner", "jrec", "rotate", "barrier"), m.groups()[2:]):
        tot[k] = tot.get(k, 0.0) + float(v) * r
print(f"SVDs {n} rounds {rounds}; cycles per round:", {k: round(v / max(rounds, 1)) for k, v in tot.items()})
PY
