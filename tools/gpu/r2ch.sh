# round 2, call ch: heavy tiles -- tile-list centroids gathered before the walk (4 entries per step) vs not
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "heavy or C5 or large_k or k_sweep or dominant or deterministic" > gpurun_out/r2ch_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ch_tests.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_hnog.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_hnog.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2ch_sweep.txt 2>&1
done
KMEANS_LIB_OVERRIDE=paper_2405_12052_b200/libkmeans.so timeout -s KILL 300 python tools/ab_bitwise.py dump gpurun_out/r2ch_ab_new.npz > gpurun_out/r2ch_ab.txt 2>&1
KMEANS_LIB_OVERRIDE=tune/libkmeans_htold.so timeout -s KILL 300 python tools/ab_bitwise.py dump gpurun_out/r2ch_ab_old.npz >> gpurun_out/r2ch_ab.txt 2>&1
python tools/ab_bitwise.py compare gpurun_out/r2ch_ab_new.npz gpurun_out/r2ch_ab_old.npz >> gpurun_out/r2ch_ab.txt 2>&1
KMEANS_LIB_OVERRIDE=tune/libkmeans_hprof.so timeout -s KILL 300 python tools/sweep.py tune/libkmeans_hprof.so --workload C5 --reps 1 > gpurun_out/r2ch_prof.txt 2>&1
