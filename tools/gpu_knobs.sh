#!/bin/bash
# C3-only bench lines under study knobs: tools/gpu_knobs.sh TAG "ENV=.. ENV2=.." "ENV=.." ...
O=gpurun_out/${1:-knobs}; mkdir -p $O; shift
i=0
for kv in "$@"; do
  env $kv timeout 600 python bench.py --steps 20 --warmup 5 --skip-svd --skip-shards --skip-heff-insweep \
    --no-cpu-baseline > $O/b$i.json 2> $O/b$i.err
  echo "$kv -> $(python -c "import json;d=json.load(open('$O/b$i.json'));print(d['value'], d['phases_ms'])")" >> $O/summary.txt
  i=$((i+1))
done
cat $O/summary.txt
