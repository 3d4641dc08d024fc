# round 2, call cc: k_assign_heavy_tiles occupancy (min blocks per SM 2 / 3 / 4) vs k_assign_heavy
set -x
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_htb3.so tune/libkmeans_htb4.so tune/libkmeans_htold.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_htb3.so tune/libkmeans_htb4.so tune/libkmeans_htold.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2cc_sweep.txt 2>&1
done
for v in htb3 htb4; do
KMEANS_LIB_OVERRIDE=tune/libkmeans_$v.so timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_assign_heavy' -c 20 --csv --log-file gpurun_out/r2cc_launches_$v.csv python bench.py --workload C5 --steps 10 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2cc_ncu_$v.log 2>&1
done
