#!/bin/bash
# quick A/B: C3 + chi=2048 SVD bench line (no CPU arms, shards, complex, in-sweep, C5), cluster Jacobi phase split
TAG=${1:-ab}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --skip-shards --skip-complex-svd \
  --skip-heff-insweep --skip-c5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
bash tools/cluster_prof.sh $TAG > $O/cluster_prof.txt 2>&1; echo "prof rc=$?" >> $O/status.txt
if [ "$2" = "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
fi
python -c "
import json; d=json.load(open('$O/bench.json')); print('C3', d['value'], 'svd', d.get('svd_chi2048_ms'), 'sweeps', d['sweep_s'])"
cat $O/cluster_prof.txt | tail -2
cat $O/status.txt
