#!/bin/bash
# C3 bench (sweeps 3-7, device time) under the library's study knobs, one box.
O=gpurun_out/${1:-knobs}
mkdir -p $O
run() {  # label, env...
  local label=$1; shift
  for rep in 1 2; do
    v=$(env "$@" timeout 300 python bench.py --skip-svd --no-cpu-baseline 2>/dev/null | tail -1 |
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phases_ms'])")
    echo "$label rep$rep $v" >> $O/knobs.txt
  done
}
run default ACHI_DUMMY=1
for P in 32 48 96 128 0; do run precond_min=$P ACHI_SVD_PRECOND_MIN=$P; done
for X in 0 2; do run cross=$X ACHI_JACOBI_CROSS=$X; done
run inner2 ACHI_JACOBI_INNER=2
