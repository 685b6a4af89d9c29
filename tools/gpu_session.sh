set -x
O=gpurun_out/${1:-r02a}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
lscpu > $O/lscpu.txt 2>&1; nproc >> $O/lscpu.txt
ACHI_DIVERGENCE_DIR=$O timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 900 python tools/profile_c3.py --sweeps 16 --profile 0 > $O/prof0.log 2>&1; echo "prof0 rc=$?" >> $O/status.txt
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
cat $O/status.txt
