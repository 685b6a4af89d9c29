#!/bin/bash
# Final-tree check: GPU suite, smoke, bench (both arms), production launch list of C3
TAG=${1:-r02s}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -s 9000 -c 2000 --csv --log-file $O/launches_prod.csv python tools/ncu_c3.py 8 > $O/ncu_list2.log 2>&1
echo "list2 rc=$?" >> $O/status.txt
python tools/ncu_summary.py $O/launches_prod.csv > $O/launches_prod_summary.txt 2>&1
cat $O/status.txt
