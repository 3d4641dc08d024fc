# round 2, call final-8 (k_prune bounds kept in registers): full GPU suite, smoke, bench lines, launch lists + ncu, bitwise A/B of the heavy kernels
set -x
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2n_gputest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2n_gputest.txt
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r2n_smoke.txt
timeout -s KILL 900 python bench.py > gpurun_out/r2n_bench_NS.json 2> gpurun_out/r2n_bench_NS.err
for wl in C5 C3 C2 C1; do
  timeout -s KILL 600 python bench.py --workload $wl --steps 200 --warmup 10 --e2e-steps 2 > gpurun_out/r2n_bench_$wl.json 2> gpurun_out/r2n_bench_$wl.err
done
timeout -s KILL 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2n_ref_NS.json 2> gpurun_out/r2n_ref_NS.err
KMEANS_LIB_OVERRIDE=paper_2405_12052_b200/libkmeans.so timeout -s KILL 300 python tools/ab_bitwise.py dump gpurun_out/r2n_ab_tiles.npz > gpurun_out/r2n_ab.txt 2>&1
KMEANS_LIB_OVERRIDE=tune/libkmeans_htold.so timeout -s KILL 300 python tools/ab_bitwise.py dump gpurun_out/r2n_ab_old.npz >> gpurun_out/r2n_ab.txt 2>&1
python tools/ab_bitwise.py compare gpurun_out/r2n_ab_tiles.npz gpurun_out/r2n_ab_old.npz >> gpurun_out/r2n_ab.txt 2>&1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2n_ns_launches.csv python bench.py --steps 20 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2n_ncu_launch.log 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_assign_pruned -s 30 -c 1 -o gpurun_out/r2n_ns_pruned python bench.py --steps 10 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2n_ncu_ns.log 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:'k_assign_pruned|k_assign_heavy|k_prune' -s 40 -c 3 -o gpurun_out/r2n_c5 python bench.py --workload C5 --steps 10 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2n_ncu_c5.log 2>&1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2n_c5_launches.csv python bench.py --workload C5 --steps 20 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2n_ncu_c5_launch.log 2>&1
KMEANS_LIB_OVERRIDE=tune/libkmeans_checked.so timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2n_checked.txt 2>&1; echo "rc=$?" >> gpurun_out/r2n_checked.txt
