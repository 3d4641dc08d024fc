# round 2, call bc: the smem-limit test against the library before and after allow_smem
set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "smem_sizes or interleaved" > gpurun_out/r2bc_new.txt 2>&1; echo "rc=$?" >> gpurun_out/r2bc_new.txt
KMEANS_LIB_OVERRIDE=tune/libkmeans_oldsmem.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "smem_sizes" > gpurun_out/r2bc_old.txt 2>&1; echo "rc=$?" >> gpurun_out/r2bc_old.txt
