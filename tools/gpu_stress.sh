#!/bin/bash
# Repeatability: the default bench twice, the chi=1024 in-sweep chain three times, the GPU suite once
TAG=${1:-st1}
O=gpurun_out/$TAG
mkdir -p $O
for i in 1 2; do
  timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_$i.json 2> $O/bench_$i.err; echo "bench $i rc=$?" >> $O/status.txt
done
for i in 1 2 3; do
  timeout 400 python tools/heff_insweep.py 5 > $O/insweep_$i.log 2>&1; echo "insweep $i rc=$?" >> $O/status.txt
done
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
cat $O/status.txt
