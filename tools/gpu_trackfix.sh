#!/bin/bash
# The chi=1024 in-sweep chain (stream SVDs at 2048^2, row split 4) repeated, then the bench
TAG=${1:-tf1}
O=gpurun_out/$TAG
mkdir -p $O
for i in 1 2 3; do
  ( time timeout 400 python tools/heff_insweep.py 5 ) > $O/insweep_$i.log 2>&1; echo "insweep $i rc=$?" >> $O/status.txt
done
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
cat $O/status.txt
