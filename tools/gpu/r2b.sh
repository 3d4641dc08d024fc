# round 2, call b: GPU tests (release + KM_CHECKS build), L2-keep sweep, C5 after the E change
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_gputest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_gputest.txt
KMEANS_LIB_OVERRIDE=tune/libkmeans_checked.so timeout 1200 python -m pytest tests -m gpu -q -k "not full_size" > gpurun_out/r2b_gputest_checked.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_gputest_checked.txt
for mb in 0 30 60 80 100; do
  KMEANS_L2_KEEP_MB=$mb timeout 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --N 12500000 > gpurun_out/r2b_keep_$mb.txt 2>&1
  KMEANS_L2_KEEP_MB=$mb timeout 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so >> gpurun_out/r2b_keep_$mb.txt 2>&1
done
timeout 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 > gpurun_out/r2b_c5.txt 2>&1
