#!/bin/bash
O=gpurun_out/${1:-csvd}; mkdir -p $O; shift
for kv in "$@"; do echo "== $kv" >> $O/summary.txt; env $kv timeout 900 python tools/csvd_study.py 6 >> $O/summary.txt 2>&1; done
cat $O/summary.txt
