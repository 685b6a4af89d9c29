#!/bin/bash
# C2 isolated-SVD throughput by size on one GPU (ensemble runner, U/S/V^T).
# usage (on the GPU box): bash tools/c2_sizes.sh TAG   -> gpurun_out/TAG/c2_<n>_<inflight>.json
O=gpurun_out/${1:-c2}
mkdir -p $O
for spec in 256:16:1 256:16:4 512:16:1 512:16:4 1024:8:1 1024:8:4 2048:4:1 2048:4:2; do
  IFS=: read chi batch k <<< "$spec"
  timeout 300 python -m paper_2604_03960_b200.ensemble_run --job c2 --svd-chi $chi --batch $batch \
    --inflight $k > $O/c2_${chi}_${k}.json 2> $O/c2_${chi}_${k}.err
  echo "c2 chi=$chi inflight=$k rc=$?"
done
