# round 2, call y: cost of a gpu-scope fence + atomic at the end of every chunk CTA
set -x
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_expfence.so; do
  for N in 12500000 100000000; do
    timeout -s KILL 300 python tools/sweep.py $lib --N $N >> gpurun_out/r2y_sweep.txt 2>&1
  done
done
