# round 2, call bp: the full GPU suite against the KM_CHECKS build (device traps + red zones)
set -x
KMEANS_LIB_OVERRIDE=tune/libkmeans_checked.so timeout -s KILL 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2bp_checked.txt 2>&1; echo "rc=$?" >> gpurun_out/r2bp_checked.txt
