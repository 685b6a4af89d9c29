#!/bin/bash
# Stream-SVD outer stop threshold study (ACHI_JACOBI_STOP, default 1e-7): sweeps,
# ms and max |sigma - ref| / sigma_1 at 1024..4096 (tools/svd_study.py).
O=gpurun_out/${1:-stop}
mkdir -p $O
for T in 1e-7 3e-7 1e-6 3e-6; do
  echo "== stop $T" >> $O/stop.txt
  ACHI_JACOBI_STOP=$T timeout 600 python tools/svd_study.py 1024 2048 4096 >> $O/stop.txt 2>&1
done
