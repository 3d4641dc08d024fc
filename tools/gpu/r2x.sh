# round 2, call x: pinned state readback (NCCL wait polling), L2 keep default for small shards
set -x
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -k "nccl or p2p" > gpurun_out/r2x_nccl.txt 2>&1; echo "rc=$?" >> gpurun_out/r2x_nccl.txt
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/r2x_gputest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2x_gputest.txt
for N in 12500000 25000000 100000000; do
  timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --N $N >> gpurun_out/r2x_sweep.txt 2>&1
done
