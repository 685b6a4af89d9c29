# stream-path Jacobi: tracked diagonal Grams in cross rounds (ACHI_JACOBI_TRACK=1) vs fresh Grams
mkdir -p gpurun_out/$1
for T in 0 1; do
  echo "== track $T" >> gpurun_out/$1/track.txt
  ACHI_JACOBI_TRACK=$T timeout 300 python tools/svd_study.py 1024 2048 4096 >> gpurun_out/$1/track.txt 2>&1
  ACHI_JACOBI_TRACK=$T ACHI_JACOBI_PROF=1 timeout 300 python tools/svd_study.py 4096 2>&1 | grep jacobi-stream | tail -1 >> gpurun_out/$1/track.txt
  ACHI_JACOBI_TRACK=$T timeout 300 python tools/vrec_study.py 4096 2>&1 >> gpurun_out/$1/track.txt
  ACHI_JACOBI_TRACK=$T timeout 600 python tools/graded_study.py 2>&1 | grep -v '^n=200' >> gpurun_out/$1/track.txt
  ACHI_JACOBI_TRACK=$T timeout 900 python -m pytest tests -m gpu -q -x -k "svd or golden_long or boundary or ensemble or c5 or chi1024" > gpurun_out/$1/pytest_t$T.txt 2>&1
  tail -1 gpurun_out/$1/pytest_t$T.txt >> gpurun_out/$1/track.txt
done
