O=gpurun_out/${1:-oz}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x > $O/pytest_ozaki.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 600 python tools/ozaki_study.py > $O/ozaki_study.log 2>&1; echo "study rc=$?" >> $O/status.txt
cat $O/status.txt
