# stream-path Jacobi phase split (ACHI_JACOBI_PROF) at 2048^2 and 4096^2, row splits 1 and 2
mkdir -p gpurun_out/$1
for R in 0 1 2; do
  if [ $R = 0 ]; then E=""; else E="ACHI_SVD_RSPLIT=$R"; fi
  echo "== rsplit ${R:-auto}" >> gpurun_out/$1/prof.txt
  env $E ACHI_JACOBI_PROF=1 timeout 300 python tools/svd_study.py 2048 4096 >> gpurun_out/$1/prof.txt 2>&1
done
