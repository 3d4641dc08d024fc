# round 2, call cj: the whole GPU suite on the KM_CHECKS build of the final tree (device bounds checks + red zones)
set -x
KMEANS_LIB_OVERRIDE=tune/libkmeans_checked.so timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2cj_checked.txt 2>&1; echo "rc=$?" >> gpurun_out/r2cj_checked.txt
