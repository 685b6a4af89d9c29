O=gpurun_out/${1:-pzw}; mkdir -p $O
for e in 1 2 4; do
ACHI_PZ_ELEMS=$e ACHI_LANCZOS_PROF=1 timeout 300 python tools/profile_c3.py --sweeps 12 --profile 0 > $O/prof_e$e.log 2>&1
done
echo done
