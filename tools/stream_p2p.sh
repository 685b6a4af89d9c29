# stream-path Jacobi: per-round grid barrier (ACHI_JACOBI_P2P=0) vs point-to-point round ordering
mkdir -p gpurun_out/$1
for P in 1 0; do
  echo "== p2p $P" >> gpurun_out/$1/p2p.txt
  ACHI_JACOBI_P2P=$P timeout 300 python tools/svd_study.py 1024 2048 4096 >> gpurun_out/$1/p2p.txt 2>&1
  ACHI_JACOBI_P2P=$P ACHI_JACOBI_PROF=1 timeout 300 python tools/svd_study.py 4096 2>&1 | grep jacobi-stream | tail -1 >> gpurun_out/$1/p2p.txt
done
timeout 900 python -m pytest tests -m gpu -q -x -k "svd or golden_long or boundary or ensemble" > gpurun_out/$1/pytest.txt 2>&1
tail -2 gpurun_out/$1/pytest.txt >> gpurun_out/$1/p2p.txt
