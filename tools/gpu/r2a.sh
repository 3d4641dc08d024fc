set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "from paper_2405_12052_b200 import build; build.build()" 
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_gputest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_gputest.txt
timeout 600 python bench.py --steps 500 --warmup 10 --e2e-steps 2 > gpurun_out/r2a_bench_ns.txt 2>&1
timeout 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --N 12500000 > gpurun_out/r2a_sweep.txt 2>&1
timeout 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 >> gpurun_out/r2a_sweep.txt 2>&1
for tool in memcheck synccheck initcheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/r2a_san_$tool.txt 2>&1; echo "rc=$?" >> gpurun_out/r2a_san_$tool.txt
done
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize_cases.py c1 ns ns_big c5 unsorted p2p > gpurun_out/r2a_san_racecheck.txt 2>&1; echo "rc=$?" >> gpurun_out/r2a_san_racecheck.txt
