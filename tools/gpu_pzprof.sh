O=gpurun_out/${1:-pzprof}; mkdir -p $O
ACHI_LANCZOS_PROF=1 timeout 300 python tools/profile_c3.py --sweeps 12 --profile 0 > $O/prof_pz.log 2>&1
ACHI_LANCZOS_PROF=1 ACHI_LANCZOS_PERSIST=0 timeout 300 python tools/profile_c3.py --sweeps 12 --profile 0 > $O/prof_graph.log 2>&1
echo done
