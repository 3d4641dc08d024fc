"""One persistent-kernel launch on an NS-shaped shard, for ncu captures:

    ncu --set full -k regex:k_persist -c 1 python tools/persist_probe.py --N 12500000 --iters 20

Also prints the per-iteration time of that launch (CUDA events; not a bench
number when run under ncu).
"""
import argparse
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2405_12052_b200 import datagen  # noqa: E402
from paper_2405_12052_b200 import kmeans as km  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=12_500_000)
    ap.add_argument("--workload", default="NS")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--graph", action="store_true", help="the per-iteration kernel graph instead")
    a = ap.parse_args()
    w = dataclasses.replace(datagen.WORKLOADS[a.workload], N=a.N)
    X = torch.empty((w.N, w.d), dtype=torch.float32, pin_memory=True)
    datagen.generate(w, out=X.numpy())
    init = datagen.init_indices(w)
    with km.Context(X, w.K, sort=True, persist=not a.graph) as c:
        c.start(init_idx=init, tol=0.0, max_iter=1 << 30)
        c.iterate(3)
        c.poll()
        st = torch.cuda.ExternalStream(c.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        c.iterate(a.iters)
        e1.record(st)
        e1.synchronize()
        print(f"N={w.N} persistent={c.info()['persistent']} iters={a.iters} "
              f"ms/iter={e0.elapsed_time(e1) / a.iters:.4f}", flush=True)


if __name__ == "__main__":
    main()
