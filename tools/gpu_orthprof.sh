O=gpurun_out/${1:-orthprof}; mkdir -p $O
for c in 0 1; do
  ACHI_LANCZOS_PROF=1 ACHI_ORTH_CLUSTER=$c timeout 300 python tools/profile_c3.py --sweeps 10 --profile 0 > $O/prof_cluster$c.log 2>&1
done
echo done
