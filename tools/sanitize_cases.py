"""Small runs of every kernel family for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Cases (all through the C ABI, no oracle -- correctness is the parity tests'
job; here only the sanitizer's verdict counts):
  c1        C1 fit: k_fused_iterate (cooperative, grid barrier per iteration)
  ns        3e5-point NS-shaped shard, sorted path: k_assign_pruned (TMA ring,
            mbarriers, PDL), k_merge_sparse16, k_merge_update; assign with labels
  ns_big    the same with 2048-point chunks
  c5        6e4-point C5-shaped shard with far outliers, K = 1024: k_prune,
            k_assign_pruned<large>, k_assign_heavy, k_merge_sparse (match_any rounds)
  unsorted  full-scan kernels: k_assign_chunk (K = 16) and k_assign_large (K = 40)
  p2p       the exchange protocol: 4 emulated ranks, then a dead rank (timeout)
  persist   the persistent sorted iteration (k_persist_iterate), if built
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2405_12052_b200 import datagen  # noqa: E402
from paper_2405_12052_b200 import kmeans as km  # noqa: E402


def c1():
    w = datagen.WORKLOADS["C1"]
    X = datagen.generate(w)
    with km.Context(X, w.K) as c:
        c.fit(datagen.init_indices(w), w.tol, w.max_iter)


def ns(big=False):
    w = datagen.WORKLOADS["NS"]
    N = 300_000
    X = datagen.generate(w, N=N)
    init = datagen.init_indices(w, N=N)
    with km.Context(X, w.K, sort=True, big_chunks=big) as c:
        r = c.fit(init, 0.0, 3)
        c.assign(r["centroids"])
        c.update()


def c5():
    rng = np.random.default_rng(21)
    w = datagen.WORKLOADS["C5"]
    N = 60_000
    X = datagen.generate(w, N=N)
    far = rng.uniform(-3000, 3000, (1000, 3)).astype(np.float32)
    X[rng.choice(N, 1000, replace=False)] = far
    init = datagen.init_indices(w, N=N)
    with km.Context(X, w.K) as c:
        r = c.fit(init, 0.0, 2)
        c.assign(r["centroids"])
        st = c.candidate_stats()
    print("c5 candidates", st)


def unsorted():
    w = datagen.WORKLOADS["NS"]
    N = 100_003
    X = datagen.generate(w, N=N)
    for K in (16, 40):
        init = datagen.init_indices(w, N=N, K=K)
        with km.Context(X, K, sort=False, fused=False) as c:
            r = c.fit(init, 0.0, 2)
            c.assign(r["centroids"])


def p2p():
    vals = np.random.default_rng(0).standard_normal((3, 4, 65))
    km.p2p_selftest(vals)
    try:
        km.p2p_selftest(vals, dead_rank=2, timeout_s=0.05)
    except km.KMeansError as e:
        assert e.name == "KMEANS_ENCCL"


def persist():
    w = datagen.WORKLOADS["NS"]
    N = 300_000
    X = datagen.generate(w, N=N)
    init = datagen.init_indices(w, N=N)
    with km.Context(X, w.K, sort=True) as c:
        if not c.info().get("persistent", 0):
            print("persist: not built for this shard")
            return
        c.fit(init, 0.0, 3)


CASES = {"c1": c1, "ns": ns, "ns_big": lambda: ns(True), "c5": c5, "unsorted": unsorted,
         "p2p": p2p, "persist": persist}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        print("case", n, "done", flush=True)
