O=gpurun_out/${1:-heffncu}; mkdir -p $O
python tools/heff_insweep.py 5 > $O/heff_count.log 2>&1
L5=$(grep "^sweep 5" $O/heff_count.log | awk '{print $4}')
echo "L5=$L5" >> $O/status.txt
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"dmma_gemm_kernel|mpo_mix_kernel" \
  --launch-skip-before-match $((L5 + 3000)) -c 6 -o $O/full_heff1024 python tools/heff_insweep.py 5 > $O/ncu_heff.log 2>&1
echo "full heff1024 rc=$?" >> $O/status.txt
python tools/ncu_report.py $O/full_heff1024.ncu-rep > $O/ncu_heff1024_summary.txt 2>&1
cat $O/status.txt
