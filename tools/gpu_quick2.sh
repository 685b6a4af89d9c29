# quick GPU check: parity suite, C3 profile with the persistent-kernel probes, C3-only bench line
O=gpurun_out/${1:-quick}; mkdir -p $O
ACHI_DIVERGENCE_DIR=$O timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
ACHI_LANCZOS_PROF=1 timeout 600 python tools/profile_c3.py --sweeps 12 --profile 0 > $O/prof_pz.log 2>&1; echo "prof rc=$?" >> $O/status.txt
timeout 600 python bench.py --steps 20 --warmup 5 --skip-svd --skip-shards --skip-heff-insweep --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench rc=$?" >> $O/status.txt
cat $O/status.txt
