#!/bin/bash
# One GPU session of measurements for a round: bench (both arms), the ncu
# launch list of the bench command, ncu --set full captures of the dominant
# kernels, the DRAM-traffic summary.  Output: gpurun_out/$TAG/.
# usage (on the GPU box): bash tools/gpu_round.sh r01 [skip_ref]
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
if [ "$2" != "skip_ref" ]; then
  timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/status.txt
fi
# launch list of the bench command (host-stepped Lanczos so ncu sees every kernel;
# ncu cannot profile kernel nodes of graphs with conditional nodes)
# (skip sweeps 0-2, ~45k launches, then list 3000 launches of the first timed sweep)
ACHI_LANCZOS_GRAPH=0 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none \
  -s 50000 -c 3000 --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 3 --skip-svd --no-cpu-baseline > $O/ncu_list.log 2>&1
echo "list rc=$?" >> $O/status.txt
python tools/ncu_summary.py $O/launches.csv > $O/launches_summary.txt 2>&1
# full captures of the dominant kernels in the steady state of C3 (sweeps 5-6)
for K in jacobi_cluster_kernel:1000 v_replay_kernel:1000 qr_precond_kernel:100 lanczos_orth_kernel:14000 \
         heff_small_kernel:14000; do
  name=${K%%:*}; skip=${K##*:}
  ACHI_LANCZOS_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:$name -s $skip -c 2 -o $O/full_$name python tools/ncu_c3.py 7 > $O/ncu_$name.log 2>&1
  echo "full $name rc=$?" >> $O/status.txt
done
# the chi=2048 (4096 x 4096) SVD of the metric's second half: stream kernel
# (svd_study runs 4 values-only launches first; the 5th is the U/S/V^T path)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:jacobi_stream_kernel \
  -s 4 -c 1 -o $O/full_jacobi_stream_kernel python tools/svd_study.py 4096 > $O/ncu_stream.log 2>&1
echo "full stream rc=$?" >> $O/status.txt
python tools/ncu_traffic.py $O/ncu_traffic.json $O/full_*.ncu-rep > $O/traffic.log 2>&1
cat $O/status.txt
