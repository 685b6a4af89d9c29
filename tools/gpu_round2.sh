#!/bin/bash
# Round-2 measurement session: default bench (both arms), launch list of the C3 bench,
# ncu --set full captures of the dominant kernels (C3 persistent Lanczos, cluster Jacobi,
# the chi=2048 stream SVD, the in-sweep chi=1024 H_eff GEMMs), DRAM traffic summary.
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
if [ "$2" != "skip_ref" ]; then
  timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/status.txt
fi
# launch list of C3 sweeps 5..6 (graph mode off so every launch is visible)
ACHI_LANCZOS_GRAPH=0 ACHI_LANCZOS_PERSIST=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -s 60000 -c 3000 --csv --log-file $O/launches_graphoff.csv python tools/ncu_c3.py 7 > $O/ncu_list.log 2>&1
echo "list rc=$?" >> $O/status.txt
python tools/ncu_summary.py $O/launches_graphoff.csv > $O/launches_graphoff_summary.txt 2>&1
# launch list in production mode (persistent Lanczos + SVD kernels), sweeps 5..7
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -s 9000 -c 2000 --csv --log-file $O/launches_prod.csv python tools/ncu_c3.py 8 > $O/ncu_list2.log 2>&1
echo "list2 rc=$?" >> $O/status.txt
python tools/ncu_summary.py $O/launches_prod.csv > $O/launches_prod_summary.txt 2>&1
# full captures
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lanczos_persistent -s 2400 -c 1 \
  -o $O/full_lanczos_persistent_kernel python tools/ncu_c3.py 14 > $O/ncu_pz.log 2>&1; echo "full pz rc=$?" >> $O/status.txt
for K in jacobi_cluster_kernel:1200 v_replay_kernel:1200 qr_precond_kernel:100 bond_select_kernel:1000; do
  name=${K%%:*}; skip=${K##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$name -s $skip -c 2 \
    -o $O/full_$name python tools/ncu_c3.py 9 > $O/ncu_$name.log 2>&1
  echo "full $name rc=$?" >> $O/status.txt
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:jacobi_stream_kernel \
  -s 4 -c 1 -o $O/full_jacobi_stream_kernel python tools/svd_study.py 4096 > $O/ncu_stream.log 2>&1
echo "full stream rc=$?" >> $O/status.txt
# in-sweep chi=1024 H_eff: launch count at sweep 5, then capture GEMMs + mixing inside it
python tools/heff_insweep.py 4 > $O/heff_count.log 2>&1
L5=$(grep "sweep 4" $O/heff_count.log | awk '{print $4}')
L5=${L5:-0}
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"dmma_gemm_kernel|mpo_mix_kernel" \
  --launch-skip-before-match $((L5 + 3000)) -c 6 -o $O/full_heff1024 python tools/heff_insweep.py 5 > $O/ncu_heff.log 2>&1
echo "full heff1024 rc=$?" >> $O/status.txt
python tools/ncu_traffic.py $O/ncu_traffic.json $O/full_*.ncu-rep > $O/traffic.log 2>&1
for f in $O/full_*.ncu-rep; do python tools/ncu_report.py $f >> $O/ncu_full_summary.txt 2>&1; done
cat $O/status.txt
