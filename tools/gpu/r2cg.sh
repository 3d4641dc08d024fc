# round 2, call cg: heavy tiles at 64 < K <= 128 and 2D (new test)
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "heavy" > gpurun_out/r2cg_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2cg_tests.txt
