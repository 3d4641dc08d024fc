# round 2, call z: slot butterflies per TMA unit (8 points per lane) vs per warp-tile
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or C5 or ties or heavy or large_k or configs or ragged" > gpurun_out/r2z_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2z_tests.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_aggtile.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2z_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --N 12500000 >> gpurun_out/r2z_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib >> gpurun_out/r2z_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --N 2000000 --force-sort >> gpurun_out/r2z_sweep.txt 2>&1
done
