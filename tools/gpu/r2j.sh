# round 2, call j: is the persistent kernel's streaming slower even without candidate imbalance (K = 1)?
set -x
for K in 1 4; do
for N in 12500000 100000000; do
  for lib in tune/libkmeans_pw20.so tune/libkmeans_pnw20.so; do
    timeout -s KILL 300 python tools/sweep.py $lib --N $N --K $K >> gpurun_out/r2j_sweep.txt 2>&1
  done
  timeout -s KILL 300 python tools/sweep.py tune/libkmeans_pw20.so --N $N --K $K --no-persist >> gpurun_out/r2j_sweep.txt 2>&1
done
done
