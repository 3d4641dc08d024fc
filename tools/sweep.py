"""Time the assign kernel of several libkmeans.so builds on one dataset.

    python tools/sweep.py --workload NS tune/libkmeans_base.so tune/libkmeans_c32.so ...

Prints one line per library: ms per assign launch (CUDA events over `reps`
launches of kmeans_profile_assign) and the HBM fraction of 4 d N bytes.
Tuning aid only (bench.py is the measurement of record).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2405_12052_b200 import datagen  # noqa: E402
from paper_2405_12052_b200 import kmeans as km  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--workload", default="NS")
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--iters", type=int, default=10, help="Lloyd iterations before timing")
    ap.add_argument("--no-sort", action="store_true")
    ap.add_argument("--force-sort", action="store_true")
    ap.add_argument("--big-chunks", action="store_true", help="2048-point chunks at any N")
    ap.add_argument("--persist", action="store_true",
                    help="sorted K <= 16: k_persist_iterate instead of the per-iteration kernel graph")
    ap.add_argument("--K", type=int, default=0, help="override K (init = first K seeded indices)")
    ap.add_argument("--N", type=int, default=0, help="override N (a prefix-shaped draw of the workload)")
    a = ap.parse_args()
    w = datagen.WORKLOADS[a.workload]
    if a.N:
        import dataclasses
        w = dataclasses.replace(w, N=a.N)
    X = torch.empty((w.N, w.d), dtype=torch.float32, pin_memory=True)
    datagen.generate(w, out=X.numpy())
    init = datagen.init_indices(w)
    if a.K:
        w = datagen.dataclasses.replace(w, K=a.K) if hasattr(datagen, "dataclasses") else w
        import dataclasses
        w = dataclasses.replace(w, K=a.K)
        init = datagen.init_indices(w)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    for lib in a.libs:
        km._lib = None
        km.LIB_PATH = os.path.abspath(lib)
        ctx = km.Context(X, w.K, sort=False if a.no_sort else (True if getattr(a, "force_sort", False) else None),
                         big_chunks=a.big_chunks, persist=a.persist)
        ctx.start(init_idx=init, tol=0.0, max_iter=1 << 30)
        ctx.iterate(a.iters)
        ctx.poll()
        st = torch.cuda.ExternalStream(ctx.stream)
        t = ctx.profile_stage(a.reps, 1, timed=True)        # assign kernels alone
        t_rm = ctx.profile_stage(a.reps, 2, timed=True)     # chunk-row merge alone
        # (unsorted small-K path: stage 2 = k_merge_rows)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ctx.iterate(a.reps)
        e1.record(st)
        e1.synchronize()
        ti = e0.elapsed_time(e1) / a.reps
        info = ctx.info()
        cand = ctx.candidate_stats() if info["sorted"] else {}
        gbs = 4 * w.d * w.N / (t / 1e3) / 1e9
        print(json.dumps({"lib": os.path.basename(lib), "N": w.N, "sorted": info["sorted"], "assign_ms": round(t, 4), "row_merge_ms": round(t_rm, 4),
                          "iter_ms": round(ti, 4), "hbm_frac": round(gbs / peak, 4),
                          "iter_hbm_frac": round(4 * w.d * w.N / (ti / 1e3) / 1e9 / peak, 4),
                          "grid": info["grid"], "smem": info["smem_bytes"], "persistent": info["persistent"],
                          "cand_mean": round(cand.get("mean", 0), 3)}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
