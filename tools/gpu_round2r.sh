#!/bin/bash
# Final-tree measurement: GPU suite, smoke, then the round measurement session
# (tools/gpu_round2.sh: bench both arms, launch lists, ncu --set full captures, traffic)
TAG=${1:-r02r}
mkdir -p gpurun_out/$TAG
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$TAG/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/$TAG/status.txt
bash tools/gpu_round2.sh $TAG
