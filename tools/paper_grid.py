"""The paper's experiment grid on one B200.

    python tools/paper_grid.py [--reps 5] [--md profiles/r1_paper_grid.md]

For every cell of PAPER.md Tables 1-5 (datagen.paper_grid(): 2D N = 1e5..5e5,
3D N = 1e5..1e6, K = 4 / 8 / 11) it runs Lloyd to convergence (tol = 1e-6,
the paper's "tolerance value of the order of 10^-6") from K seeded
random points and reports
  iters       iterations to convergence,
  fit_ms      kmeans_fit_ctx on device-resident points (median of --reps),
  e2e_ms      kmeans_create from pinned host memory + fit (labels back) + destroy,
beside the paper's own times for the same (N, K) -- context only: other
hardware, other (unpublished) data, and its convergence counts are unknown.
GPU only; the oracle parity of these runs is tests/test_gpu_parity.py
(test_paper_grid_full_runs).
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2405_12052_b200 import datagen  # noqa: E402
from paper_2405_12052_b200 import kmeans as km  # noqa: E402

# PAPER.md seconds: Table 1 serial, Table 2/3 OpenMP at the
# best thread count listed, Table 4/5 OpenACC.  Keys (d, N, K).
PAPER = {
    (2, 500_000, 4): {"serial": 1.664616},
    (2, 500_000, 8): {"serial": 5.313805, "openmp_p16": 3.648641, "openacc": 0.518219},
    (2, 500_000, 11): {"serial": 25.744963},
    (3, 1_000_000, 4): {"serial": 2.255409, "openmp_p16": 13.495912, "openacc": 0.802407},
    (3, 1_000_000, 8): {"serial": 34.27957},
    (3, 1_000_000, 11): {"serial": 73.925911},
    (2, 100_000, 8): {"openmp_p8": 0.273247, "openacc": 0.7213},
    (2, 200_000, 8): {"openmp_p16": 0.310875, "openacc": 0.283524},
    (3, 100_000, 4): {"openmp_p8": 1.220420, "openacc": 0.087148},
    (3, 200_000, 4): {"openmp_p16": 2.359286, "openacc": 0.486771},
    (3, 400_000, 4): {"openmp_p16": 4.937502, "openacc": 0.548548},
    (3, 800_000, 4): {"openmp_p16": 9.245712, "openacc": 0.743832},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--md", default="")
    a = ap.parse_args()
    rows = []
    for w in datagen.paper_grid():
        Xh = torch.empty((w.N, w.d), dtype=torch.float32, pin_memory=True)
        datagen.generate(w, out=Xh.numpy())
        Xd = Xh.cuda()
        init = datagen.init_indices(w)
        lab = torch.empty(w.N, dtype=torch.int32, pin_memory=True)
        torch.cuda.synchronize()
        with km.Context(Xd, w.K) as c:
            c.fit(init, w.tol, w.max_iter, labels=False, traces=False)   # warm-up
            ts = []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                r = c.fit(init, w.tol, w.max_iter, labels=False, traces=False)
                ts.append(time.perf_counter() - t0)
            info = c.info()
        e2e = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            with km.Context(Xh, w.K) as c2:
                r2 = c2.fit(init, w.tol, w.max_iter, out_labels=lab.numpy(), traces=False)
            e2e.append(time.perf_counter() - t0)
        assert r2["iters"] == r["iters"]
        row = {"cell": w.name, "d": w.d, "N": w.N, "K": w.K, "iters": r["iters"],
               "inertia": r["inertia"], "fit_ms": statistics.median(ts) * 1e3,
               "e2e_ms": statistics.median(e2e) * 1e3, "sorted": info["sorted"],
               "paper_s": PAPER.get((w.d, w.N, w.K), {})}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if a.md:
        with open(a.md, "w") as f:
            f.write("# The paper's experiment grid on one B200 (tools/paper_grid.py)\n\n")
            f.write("Lloyd to convergence (tol 1e-6, K seeded random initial points), "
                    "synthetic Gaussian mixtures of datagen.paper_grid(); medians of "
                    f"{a.reps} runs.  fit = kmeans_fit_ctx on device-resident points; e2e = "
                    "create from pinned host memory + fit + labels back + destroy.  Paper "
                    "seconds are context only (other hardware, unpublished data, unknown "
                    "iteration counts).\n\n")
            f.write("| d | N | K | iters | fit ms | e2e ms | path | paper (s) |\n"
                    "|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                p = ", ".join(f"{k} {v:g}" for k, v in r["paper_s"].items()) or "--"
                f.write(f"| {r['d']} | {r['N']} | {r['K']} | {r['iters']} | {r['fit_ms']:.3f} | "
                        f"{r['e2e_ms']:.2f} | {'sorted' if r['sorted'] else 'full scan'} | "
                        f"{p} |\n")


if __name__ == "__main__":
    main()
