"""Bitwise A/B of one Lloyd step between two builds of libkmeans.so.

    python tools/ab_bitwise.py dump OUT.npz      (library from KMEANS_LIB_OVERRIDE)
    python tools/ab_bitwise.py compare A.npz B.npz

`dump` runs one step (kmeans_assign + kmeans_update) on the heavy-chunk case of
tests/test_gpu_parity.py::test_heavy_chunks_large_k (C5 blobs, 2e5 points, a
sparse shell of far points) and on C5 at 60k, and stores labels, counts, sums,
J, mu^{t+1} and E; `compare` requires them bit-identical (used for
KM_HEAVY_TILES=1 vs 0, whose chunk rows are claimed identical bit for bit).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def cases():
    from paper_2405_12052_b200 import datagen
    w = datagen.WORKLOADS["C5"]
    rng = np.random.default_rng(21)
    X = datagen.generate(w, N=200_000)
    far = rng.uniform(-3000, 3000, (3000, 3)).astype(np.float32)
    X[rng.choice(200_000, 3000, replace=False)] = far
    yield "heavy", X, X[datagen.init_indices(w, N=200_000)].astype(np.float64), w.K
    X = datagen.generate(w, N=60_000)
    yield "c5", X, X[datagen.init_indices(w, N=60_000)].astype(np.float64), w.K


def dump(out):
    from paper_2405_12052_b200 import kmeans as km
    res = {}
    for tag, X, mu, K in cases():
        with km.Context(X, K) as c:
            g = c.assign(mu)
            mu1, E = c.update()
            st = c.candidate_stats()
        res.update({f"{tag}_labels": g["labels"], f"{tag}_counts": g["counts"],
                    f"{tag}_sums": g["sums"], f"{tag}_J": np.float64(g["inertia"]),
                    f"{tag}_mu1": mu1, f"{tag}_E": np.float64(E),
                    f"{tag}_candmax": np.int64(st["max"])})
    np.savez(out, **res)


def compare(a, b):
    A, B = np.load(a), np.load(b)
    ok = True
    for k in A.files:
        same = A[k].tobytes() == B[k].tobytes()
        ok &= same
        print(f"{k}: {'identical' if same else 'DIFFERENT'}")
    print("ALL IDENTICAL" if ok else "MISMATCH")
    return 0 if ok else 1


if __name__ == "__main__":
    if sys.argv[1] == "dump":
        dump(sys.argv[2])
    else:
        sys.exit(compare(sys.argv[2], sys.argv[3]))
