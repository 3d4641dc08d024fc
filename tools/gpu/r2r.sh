# round 2, call r: cross-process P2P exchange over CUDA IPC (loopback turns) + full GPU suite
set -x
timeout -s KILL 300 python -m pytest tests/test_p2p_ipc.py -x -q > gpurun_out/r2r_ipc.txt 2>&1; echo "rc=$?" >> gpurun_out/r2r_ipc.txt
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2r_gputest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2r_gputest.txt
