"""Break the end-to-end call (create + fit + destroy from host memory) into parts.

    python tools/e2e_profile.py [--workload NS] [--reps 3]

Prints wall-clock seconds for: raw pinned H2D / D2H copies of the same bytes
(torch), kmeans_create from host and from device memory, fit with and without
labels, destroy.  Tuning aid only (bench.py's e2e is the measurement of record).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2405_12052_b200 import datagen  # noqa: E402
from paper_2405_12052_b200 import kmeans as km  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="NS")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--no-sort", action="store_true")
    a = ap.parse_args()
    w = datagen.WORKLOADS[a.workload]
    Xh = torch.empty((w.N, w.d), dtype=torch.float32, pin_memory=True)
    datagen.generate(w, out=Xh.numpy())
    init = datagen.init_indices(w)
    lab = torch.empty(w.N, dtype=torch.int32, pin_memory=True)
    Xd = Xh.cuda()
    torch.cuda.synchronize()
    for rep in range(a.reps):
        r = {}
        t = time.perf_counter()
        Xd.copy_(Xh, non_blocking=True)
        torch.cuda.synchronize()
        r["torch_h2d"] = time.perf_counter() - t
        ld = torch.empty(w.N, dtype=torch.int32, device="cuda")
        t = time.perf_counter()
        lab.copy_(ld, non_blocking=True)
        torch.cuda.synchronize()
        r["torch_d2h_labels"] = time.perf_counter() - t
        t = time.perf_counter()
        c = km.Context(Xh, w.K, sort=False if a.no_sort else (True if getattr(a, "force_sort", False) else None))
        r["create_host"] = time.perf_counter() - t
        t = time.perf_counter()
        c.fit(init, 0.0, a.iters, labels=False, traces=False)
        r["fit_nolabels"] = time.perf_counter() - t
        t = time.perf_counter()
        c.fit(init, 0.0, a.iters, out_labels=lab.numpy(), traces=False)
        r["fit_labels"] = time.perf_counter() - t
        t = time.perf_counter()
        c.close()
        r["destroy"] = time.perf_counter() - t
        t = time.perf_counter()
        c = km.Context(Xd, w.K, sort=False if a.no_sort else (True if getattr(a, "force_sort", False) else None))
        r["create_device"] = time.perf_counter() - t
        c.close()
        print(json.dumps({k: round(v * 1e3, 2) for k, v in r.items()}), flush=True)


if __name__ == "__main__":
    main()
