# round 2, call q: knob sweep at the P=8 NS shard (1.25e7) and NS
set -x
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_sct4.so tune/libkmeans_sct4rg512.so tune/libkmeans_rg128.so tune/libkmeans_rg512.so tune/libkmeans_mb24.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --N 12500000 >> gpurun_out/r2q_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --N 25000000 >> gpurun_out/r2q_sweep.txt 2>&1
done
