"""GPU parity: the sm_100a path through the C ABI against the CPU oracle.

Bars (BASELINE.json north_star):
  - labels: bit-exact per step, given identical fp64 input centroids;
  - counts: exact;
  - sums, inertia, mu^{t+1}: within 1e-9 relative in the sense of reading R13
    (|delta| <= 1e-9 * scale, scale = sum of |x| over the cluster, since an fp64
    sum's rounding error scales with sum|x|, not with |sum x|);
  - E per step: |dE| <= 1e-9 * max(E, 1e-3 * sum ||mu||^2) plus the error E
    inherits from mu (R13);
  - full runs on well-separated blobs: iters exact, labels exact, centroids
    within 1e-6 relative.
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2405_12052_b200 import datagen
from paper_2405_12052_b200 import kmeans as km

pytestmark = pytest.mark.gpu

REL = 1e-9


def cluster_abs_scale(X, labels, K):
    """sum_i |x_ij| over each cluster (the scale of fp64 summation error)."""
    d = X.shape[1]
    s = np.zeros((K, d))
    for j in range(d):
        s[:, j] = np.bincount(labels, weights=np.abs(X[:, j].astype(np.float64)), minlength=K)
    return s


def check_step(X, mu, ctx=None, tag="", sort=True):
    """One Lloyd step on the GPU vs the oracle at identical mu^t."""
    N, d = X.shape
    K = mu.shape[0]
    own = ctx is None
    if own:
        ctx = km.Context(X, K, **ctx_kwargs(sort))
    try:
        g = ctx.assign(mu)
        mu_next, E = ctx.update()
    finally:
        if own:
            ctx.close()
    o = oracle.step(X, mu)
    lab_g, lab_o = g["labels"], o["labels"]
    bad = np.nonzero(lab_g != lab_o)[0]
    assert bad.size == 0, f"{tag}: {bad.size} labels differ, first at {bad[:5]}"
    assert np.array_equal(g["counts"], o["counts"]), tag
    scale = cluster_abs_scale(X, lab_o, K)
    assert np.all(np.abs(g["sums"] - o["sums"]) <= REL * scale + 1e-300), tag
    if np.isinf(o["J"]):   # fp32 distances overflowed on both sides
        assert g["inertia"] == o["J"], tag
    else:
        assert abs(g["inertia"] - o["J"]) <= REL * max(o["J"], 1e-300), tag
    n = np.maximum(o["counts"], 1)[:, None]
    mscale = np.maximum(np.abs(o["mu_next"]), scale / n)
    assert np.all(np.abs(mu_next - o["mu_next"]) <= REL * mscale + 1e-300), tag
    # E inherits |d mu| * 2 |mu_next - mu| per entry, plus its own rounding
    dmu = REL * mscale
    e_tol = np.sum(2 * np.abs(o["mu_next"] - mu) * dmu + dmu ** 2) + \
        REL * max(o["E"], 1e-3 * float(np.sum(mu ** 2)))
    assert abs(E - o["E"]) <= e_tol, f"{tag}: E {E} vs {o['E']}"
    return g, o


def perturbed_centroids(X, K, seed):
    """K data points plus fp64 noise that is not fp32-representable (so the
    fp64 -> fp32 staging rounding is exercised)."""
    rng = np.random.default_rng(seed)
    idx = rng.choice(X.shape[0], K, replace=False)
    return X[idx].astype(np.float64) + rng.normal(0, 0.3, (K, X.shape[1]))


# --------------------------------------------------------------------------
# per-step parity over the configs (small N) and K / ragged-N sweeps
# --------------------------------------------------------------------------
SORT = [pytest.param(True, id="sorted"), pytest.param(False, id="unsorted"),
        pytest.param("big", id="sorted2048")]


def ctx_kwargs(sort):
    """Context options of a SORT parameter ("big": sorted, 2048-point chunks)."""
    return dict(sort=True, big_chunks=True) if sort == "big" else dict(sort=sort)


@pytest.mark.parametrize("sort", SORT)
@pytest.mark.parametrize("name,N", [("C1", 10_000), ("C2", 200_000), ("C3", 300_001),
                                    ("NS", 250_003), ("C5", 60_000)])
def test_step_parity_configs(name, N, sort):
    w = datagen.WORKLOADS[name]
    X = datagen.generate(w, N=N)
    init = datagen.init_indices(w, N=N)
    mu0 = X[init].astype(np.float64)
    check_step(X, mu0, tag=f"{name} init", sort=sort)
    check_step(X, perturbed_centroids(X, w.K, 5), tag=f"{name} perturbed", sort=sort)


@pytest.mark.parametrize("sort", SORT)
@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("K", [1, 2, 3, 5, 8, 11, 13, 16, 17, 31, 64, 100, 257])
def test_step_parity_k_sweep(d, K, sort):
    w = datagen.WORKLOADS["NS" if d == 3 else "C3"]
    N = 20_011
    X = datagen.generate(w, N=N)
    check_step(X, perturbed_centroids(X, K, K), tag=f"d={d} K={K}", sort=sort)


@pytest.mark.parametrize("sort", SORT)
@pytest.mark.parametrize("N", [1, 2, 3, 7, 511, 512, 513, 1023, 1025, 2047, 2049, 4097, 65_537])
def test_step_parity_ragged_n(N, sort):
    w = datagen.WORKLOADS["NS"]
    X = datagen.generate(w, N=max(N, 16))[:N].copy()
    for K in sorted({1, min(N, 5), min(N, 16), min(N, 40)}):
        check_step(X, perturbed_centroids(X, K, N + K), tag=f"N={N} K={K}", sort=sort)


@pytest.mark.parametrize("sort", SORT)
@pytest.mark.parametrize("K,frac", [(40, 1.0), (64, 0.9), (257, 0.5), (1024, 0.97)])
def test_step_parity_dominant_label(K, frac, sort):
    """A label mix where one cluster takes most points of every warp (the
    large-K full scan sums equal labels by a rank tree; up to all 32 lanes of
    a slot in one group), the rest spread over the other centroids, ragged N."""
    rng = np.random.default_rng(K)
    N = 70_001
    mu = np.zeros((K, 3))
    mu[1:] = rng.uniform(-50, 50, (K - 1, 3)) + np.sign(rng.standard_normal((K - 1, 3))) * 20
    own = rng.random(N) < frac
    X = np.where(own[:, None], rng.normal(0, 1.0, (N, 3)),
                 mu[rng.integers(1, K, N)] + rng.normal(0, 0.5, (N, 3))).astype(np.float32)
    check_step(X, mu + rng.normal(0, 1e-3, mu.shape), tag=f"K={K} frac={frac}", sort=sort)


@pytest.mark.parametrize("sort", SORT)
def test_step_parity_exact_ties_and_empty_clusters(sort):
    """Integer data -> exact fp32 distances -> genuine ties (lowest k wins);
    duplicated centroids -> clusters that stay empty (keep mu^t)."""
    rng = np.random.default_rng(1)
    X = rng.integers(-4, 5, (50_000, 3)).astype(np.float32)
    C = rng.integers(-4, 5, (12, 3)).astype(np.float64)
    C[7] = C[2]
    C[9] = C[2]
    C[11] = [1000.0, 1000.0, 1000.0]
    g, o = check_step(X, C, tag="ties", sort=sort)
    assert g["counts"][7] == 0 and g["counts"][9] == 0 and g["counts"][11] == 0
    X2 = rng.integers(-3, 4, (40_000, 2)).astype(np.float32)
    C2 = np.array([[0, 0], [0, 0], [1, 1], [-1, 1], [1, 1], [2, -2], [0, 3], [-3, 0],
                   [3, 3], [1, 1], [0, 0], [-2, -2], [2, 2], [-1, -1], [1, -1], [3, -3],
                   [0, 1], [1, 0], [0, -1], [-1, 0]], np.float64)
    check_step(X2, C2, tag="ties 2D K=20 (large path)", sort=sort)
    check_step(X2, C2[:16], tag="ties 2D K=16 (small path)", sort=sort)


@pytest.mark.parametrize("sort", SORT)
@pytest.mark.parametrize("scale", [3e19, 1e-20, 1e-30, 1.0])
def test_step_parity_extreme_scales(scale, sort):
    """Distances that overflow fp32 (all +inf -> every point ties -> label 0),
    that underflow to subnormals or zero (ties again), and uniform
    (non-clustered) data: the pruning bound must never drop a possible argmin."""
    rng = np.random.default_rng(11)
    X = (rng.uniform(-1, 1, (30_011, 3)) * scale).astype(np.float32)
    C = X[rng.choice(30_011, 16, replace=False)].astype(np.float64) * 1.0000001
    check_step(X, C, tag=f"scale {scale}", sort=sort)


@pytest.mark.parametrize("sort", SORT)
def test_step_parity_near_bisector_points(sort):
    """Points placed on (and one fp32 ulp off) the bisector planes of pairs
    of centroids: near-ties decided by the last bit of form D."""
    rng = np.random.default_rng(12)
    C = rng.normal(0, 5, (16, 3))
    P = []
    for _ in range(40_000):
        a, b = rng.choice(16, 2, replace=False)
        t = rng.uniform(0.3, 0.7)
        m = C[a] * t + C[b] * (1 - t)
        P.append(m)
    X = np.array(P, np.float32)
    X[1::3] = np.nextafter(X[1::3], np.float32(np.inf))
    X[2::3] = np.nextafter(X[2::3], np.float32(-np.inf))
    mid = ((C[:8] + C[8:]) / 2).astype(np.float32)
    X[:8] = mid
    check_step(X, C, tag="bisectors", sort=sort)


def test_step_parity_soa_layout_and_device_input():
    import torch
    w = datagen.WORKLOADS["NS"]
    X = datagen.generate(w, N=30_000)
    mu = perturbed_centroids(X, 16, 3)
    o = oracle.step(X, mu)
    Xs = np.ascontiguousarray(X.T)
    with km.Context(Xs, 16, layout="soa") as c:
        g = c.assign(mu)
        assert np.array_equal(g["labels"], o["labels"])
    Xd = torch.from_numpy(X).cuda()
    lab = torch.empty(30_000, dtype=torch.int32, device="cuda")
    with km.Context(Xd, 16) as c:
        g = c.assign(torch.from_numpy(mu).cuda(), out_labels=lab)
        assert np.array_equal(lab.cpu().numpy(), o["labels"])
        assert np.array_equal(g["counts"], o["counts"])


# --------------------------------------------------------------------------
# full runs
# --------------------------------------------------------------------------
def check_fit(X, K, init, tol, max_iter, tag="", sort=True, fused=True):
    o = oracle.fit(X, K, init, tol, max_iter)
    with km.Context(X, K, fused=fused, **ctx_kwargs(sort)) as c:
        g = c.fit(init, tol, max_iter)
    assert g["iters"] == o["iters"], f"{tag}: iters {g['iters']} vs {o['iters']}"
    assert np.array_equal(g["labels"], o["labels"]), tag
    np.testing.assert_allclose(g["centroids"], o["centroids"], rtol=1e-6, atol=1e-9)
    assert abs(g["inertia"] - o["inertia"]) <= 1e-6 * max(o["inertia"], 1e-300)
    return g, o


@pytest.mark.parametrize("sort", SORT)
@pytest.mark.parametrize("name,N", [("C1", 10_000), ("C2", 300_000), ("C3", 200_000),
                                    ("NS", 1_000_000)])
def test_full_run_parity_one_init_per_blob(name, N, sort):
    w = datagen.WORKLOADS[name]
    X = datagen.generate(w, N=N)
    init = datagen.one_per_blob_init(w, N=N)
    g, o = check_fit(X, w.M, init, w.tol, w.max_iter, tag=name, sort=sort)
    np.testing.assert_allclose(g["centroids"], w.centers(), atol=0.05)


@pytest.mark.parametrize("sort", SORT)
@pytest.mark.parametrize("K", [600, 1024])
def test_full_run_large_k(K, sort):
    """kmeans_fit at large K on every path: the iteration graph and the final
    labels pass (unsorted K = 1024: the labels pass + k_accum_large split;
    K = 600: the fused kernel at 8 points per lane; sorted: prune + pruned +
    heavy), against the oracle's run -- iterations, labels, centroids, J."""
    w = datagen.WORKLOADS["C5"]
    N = 80_000
    X = datagen.generate(w, N=N)
    init = datagen.init_indices(w, N=N, K=K)
    check_fit(X, K, init, 0.0, 3, tag=f"K={K}", sort=sort)


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("name,N,K", [("C1", 10_000, 4), ("C2", 1_000_000, 8), ("C2", 77_777, 3),
                                      ("NS", 3_000_000, 16), ("C3", 2_100_000, 13)])
def test_fused_iteration_kernel(name, N, K, fused):
    """Full-scan path on one GPU: k_fused_iterate (many iterations per
    cooperative launch, one grid barrier each) and the per-iteration graph give
    the oracle's run -- iterations, labels, centroids, traces."""
    w = datagen.WORKLOADS[name]
    X = datagen.generate(w, N=N)
    init = datagen.init_indices(w, N=N, K=K)
    g, o = check_fit(X, K, init, 1e-6, 60, tag=f"{name} fused={fused}", sort=False, fused=fused)
    with km.Context(X, K, sort=False, fused=fused) as c:
        assert c.info()["fused"] == int(fused)
        r = c.fit(init, 1e-6, 60)
        np.testing.assert_allclose(r["E_trace"], o["E_trace"], rtol=1e-6, atol=1e-12)
        np.testing.assert_allclose(r["J_trace"], o["J_trace"], rtol=1e-9)
        # split launches: iterate 3 + 2 == a 5-iteration run, bit for bit
        ref = c.fit(init, 0.0, 5)
        c.start(init_idx=init, tol=0.0, max_iter=5)
        c.iterate(3)
        c.iterate(2)
        c.iterate(4)   # past max_iter: no-op
        st = c.poll()
        assert st["iters"] == 5 and st["done"]
        assert np.array_equal(c.read_centroids(), ref["centroids"])
        assert np.array_equal(c.final_labels(), ref["labels"])


@pytest.mark.parametrize("cell", ["P2D-N100000-K8", "P3D-N100000-K4", "P2D-N200000-K8",
                                  "P2D-N500000-K11"])
def test_paper_grid_full_runs(cell):
    """cells of the paper's experiment grid (PAPER.md Tables
    1-5, datagen.paper_grid) run to convergence from the paper's seeded random
    initial points (tol 1e-6): same iteration count, labels and
    centroids as the oracle (K = 11 on 8 blobs is a local optimum, reached
    identically)."""
    w = {x.name: x for x in datagen.paper_grid()}[cell]
    X = datagen.generate(w)
    init = datagen.init_indices(w)
    check_fit(X, w.K, init, w.tol, w.max_iter, tag=cell, sort=None)


def test_full_run_parity_c1_seeded_init():
    """BASELINE.json configs[0]: N=1e4 2D blobs, K=4, seeded init, tol 1e-6, max_iter 100."""
    w = datagen.WORKLOADS["C1"]
    X = datagen.generate(w)
    init = datagen.init_indices(w)
    g, o = check_fit(X, w.K, init, w.tol, w.max_iter, tag="C1")
    with km.Context(X, w.K) as c:
        r = c.fit(init, w.tol, w.max_iter)
    np.testing.assert_allclose(r["E_trace"], o["E_trace"], rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(r["J_trace"], o["J_trace"], rtol=1e-9)


def test_kmeans_fit_convenience_call():
    w = datagen.WORKLOADS["C1"]
    X = datagen.generate(w)
    init = datagen.init_indices(w)
    o = oracle.fit(X, w.K, init, w.tol, w.max_iter)
    g = km.fit(X, w.K, init, w.tol, w.max_iter)
    assert g["iters"] == o["iters"]
    assert np.array_equal(g["labels"], o["labels"])
    np.testing.assert_allclose(g["centroids"], o["centroids"], rtol=1e-6)


@pytest.mark.parametrize("path", [dict(), dict(fused=False), dict(sort=True)],
                         ids=["fused", "unfused", "sorted"])
@pytest.mark.parametrize("name", ["w1.json", "w2.json", "w3.json", "w4.json"])
def test_hand_worked_runs_on_gpu(golden_dir, name, path):
    """Tiny integer examples: every sum is exact in any order, so the GPU's
    per-iteration E and J must equal the hand-derived values exactly -- on the
    one-launch fused kernel, the per-iteration graph (k_merge_update: E summed
    serially k-major like the oracle) and the sorted path."""
    g = json.load(open(os.path.join(golden_dir, name)))
    X = np.array(g["points"], np.float32)
    K = len(g["init_idx"])
    with km.Context(X, K, **path) as c:
        r = c.fit(g["init_idx"], g["tol"], g["max_iter"])
    assert r["iters"] == g["iters"]
    assert r["labels"].tolist() == g["labels"]
    assert r["centroids"].tolist() == g["centroids"]
    assert r["E_trace"].tolist() == [it["E"] for it in g["per_iter"]]
    assert r["J_trace"].tolist() == [it["J"] for it in g["per_iter"]]
    assert r["inertia"] == g["inertia"]


@pytest.mark.parametrize("sort", SORT)
@pytest.mark.parametrize("reps", [1, 3000])
def test_form_d_fma_golden_on_gpu(golden_dir, sort, reps):
    """tests/golden/fma_form_d.json (reading R6): the GPU's
    form D rounds its fma once -- the 2D distance is the hand-derived
    29.23716926574707 (inertia of one point at one centroid), and in 3D the
    fma decides the argmin (label 1; a separately rounded evaluation ties and
    gives 0).  reps > 1 fills several chunks (every chunk box is one point:
    both centroids stay candidates on the pruned path)."""
    g = json.load(open(os.path.join(golden_dir, "fma_form_d.json")))
    d2 = g["distance_2d"]
    X2 = np.array([d2["x"]] * reps, np.float32)
    with km.Context(X2, 1, **ctx_kwargs(sort)) as c:
        r = c.assign(np.array([d2["c"]], np.float64))
    assert r["inertia"] == reps * d2["expect"] or \
        abs(r["inertia"] - reps * d2["expect"]) <= 1e-12 * reps * d2["expect"]
    if reps == 1:
        assert r["inertia"] == d2["expect"]
    a = g["argmin_3d"]
    n3 = max(reps, 2)   # K = 2 needs N >= 2
    X3 = np.array([a["x"]] * n3, np.float32)
    with km.Context(X3, 2, **ctx_kwargs(sort)) as c:
        r = c.assign(np.array(a["centroids"], np.float64))
    assert np.all(r["labels"] == a["expect_label"])
    assert r["counts"].tolist() == [0, n3]
    if n3 == 2:
        assert r["inertia"] == 2 * a["expect_dmin"]   # exact: one fp64 doubling
    else:
        assert abs(r["inertia"] - n3 * a["expect_dmin"]) <= 1e-12 * n3 * a["expect_dmin"]


def test_special_cases_k1_kn_tol0_maxiter1():
    rng = np.random.default_rng(8)
    X = rng.normal(0, 1, (9, 2)).astype(np.float32)
    init = rng.permutation(9)
    with km.Context(X, 9) as c:
        r = c.fit(init, 1e-6, 10)
    assert r["iters"] == 1 and r["inertia"] == 0.0
    for k, i in enumerate(init):
        assert r["labels"][i] == k
    X = datagen.generate(datagen.WORKLOADS["NS"], N=5000)
    o = oracle.fit(X, 1, [3], 1e-6, 10)
    with km.Context(X, 1) as c:
        r = c.fit([3], 1e-6, 10)
    assert r["iters"] == o["iters"] == 2
    np.testing.assert_allclose(r["centroids"], o["centroids"], rtol=1e-12)
    init = datagen.init_indices(datagen.WORKLOADS["NS"], N=5000)
    with km.Context(X, 16) as c:
        r0 = c.fit(init, 0.0, 9)
        r1 = c.fit(init, 1e-6, 1)
    assert r0["iters"] == 9 and r1["iters"] == 1


def test_errors():
    X = datagen.generate(datagen.WORKLOADS["C1"], N=100)
    Xn = X.copy()
    Xn[17, 1] = np.inf
    with pytest.raises(km.KMeansError) as e:
        km.Context(Xn, 4)
    assert e.value.name == "KMEANS_ENONFINITE"
    with km.Context(X, 4) as c:
        with pytest.raises(km.KMeansError) as e:
            c.update()
        assert e.value.name == "KMEANS_ESTATE"
        with pytest.raises(km.KMeansError) as e:
            c.fit([1, 2, 2, 3], 1e-6, 10)
        assert e.value.name == "KMEANS_EINVAL"
        with pytest.raises(km.KMeansError) as e:
            c.fit([1, 2, 3, 100], 1e-6, 10)
        assert e.value.name == "KMEANS_EINVAL"
        bad = np.zeros((4, 2))
        bad[2, 0] = np.nan
        with pytest.raises(km.KMeansError) as e:
            c.assign(bad)
        assert e.value.name == "KMEANS_ENONFINITE"
        # the context is still usable after argument errors
        r = c.fit([1, 2, 3, 4], 1e-6, 10)
        assert r["iters"] >= 1


def test_auto_path_selection():
    """Default flags: the full scan below N*K*d = 3.84e8 with K <= 16, the
    sorted (pruned) path above it or for K > 16; both flags -> EINVAL."""
    X = datagen.generate(datagen.WORKLOADS["C2"], N=50_000)
    with km.Context(X, 16) as c:
        assert c.info()["sorted"] == 0
    with km.Context(X, 40) as c:
        assert c.info()["sorted"] == 1
    with km.Context(X, 16, sort=True) as c:
        assert c.info()["sorted"] == 1
    with km.Context(X, 40, sort=False) as c:
        assert c.info()["sorted"] == 0
    L = km.lib()
    o = km.Opts()
    L.kmeans_opts_init(km.ctypes.byref(o))
    o.flags = km.FLAG_NO_SORT | km.FLAG_FORCE_SORT
    h = km.ctypes.c_void_p()
    Xc = np.ascontiguousarray(X)
    rc = L.kmeans_create(km.ctypes.byref(h), km.ctypes.c_void_p(Xc.ctypes.data), Xc.shape[0], 3, 8,
                         km.ctypes.byref(o))
    assert rc == -1 and not h.value   # KMEANS_EINVAL


@pytest.mark.parametrize("sort", SORT)
@pytest.mark.parametrize("K", [8, 40])
def test_profile_stages_leave_state(sort, K):
    """kmeans_profile_stage (bench.py's per-stage timing) does not move the
    iteration: after timed launches of every stage the fit continues exactly."""
    w = datagen.WORKLOADS["C2"]
    X = datagen.generate(w, N=200_000)
    init = datagen.init_indices(w, N=200_000)[:8]
    init = np.concatenate([init, np.arange(1000, 1000 + K - 8)]) if K > 8 else init
    with km.Context(X, K, **ctx_kwargs(sort)) as c:
        ref = c.fit(init, 0.0, 5)
        c.start(init_idx=init, tol=0.0, max_iter=5)
        c.iterate(2)
        for stage in range(4):
            ms = c.profile_stage(5, stage, timed=True)
            assert ms >= 0.0
        c.profile_stage(2, 1)
        c.iterate(3)
        st = c.poll()
        assert st["iters"] == 5
        assert np.array_equal(c.read_centroids(), ref["centroids"])
        with pytest.raises(km.KMeansError) as e:
            c.profile_stage(1, 4)
        assert e.value.name == "KMEANS_EINVAL"


@pytest.mark.parametrize("sort", SORT)
def test_deterministic_bitwise(sort):
    w = datagen.WORKLOADS["NS"]
    X = datagen.generate(w, N=400_000)
    init = datagen.init_indices(w, N=400_000)
    with km.Context(X, 16, **ctx_kwargs(sort)) as c:
        a = c.fit(init, 0.0, 6)
        b = c.fit(init, 0.0, 6)
    with km.Context(X, 16, **ctx_kwargs(sort)) as c:
        e = c.fit(init, 0.0, 6)
    for r in (b, e):
        assert np.array_equal(a["labels"], r["labels"])
        assert np.array_equal(a["centroids"], r["centroids"])
        assert np.array_equal(a["E_trace"], r["E_trace"])
        assert np.array_equal(a["J_trace"], r["J_trace"])


# --------------------------------------------------------------------------
# sharding (T4'): P contexts on one device, partials summed in rank order
# --------------------------------------------------------------------------
@pytest.mark.parametrize("sort", SORT)
@pytest.mark.parametrize("P", [2, 3, 8])
def test_fake_sharding_matches_oracle(P, sort):
    w = datagen.WORKLOADS["NS"]
    N = 100_003
    X = datagen.generate(w, N=N)
    mu = perturbed_centroids(X, 16, P)
    o = oracle.step(X, mu)
    counts = np.zeros(16, np.int64)
    sums = np.zeros((16, 3))
    J = 0.0
    labels = []
    for r in range(P):
        a, b = datagen.shard_range(N, P, r)
        Xs = datagen.generate(w, a, b - a, N=N)
        with km.Context(Xs, 16, **ctx_kwargs(sort)) as c:
            g = c.assign(mu)
        labels.append(g["labels"])
        counts += g["counts"]
        sums += g["sums"]
        J += g["inertia"]
    assert np.array_equal(np.concatenate(labels), o["labels"])
    assert np.array_equal(counts, o["counts"])
    scale = cluster_abs_scale(X, o["labels"], 16)
    assert np.all(np.abs(sums - o["sums"]) <= REL * scale)
    assert abs(J - o["J"]) <= REL * o["J"]


def test_nccl_single_rank_communicator_path():
    """The distributed code path (NCCL allreduce inside the graph, CC1 init
    gather) with a 1-rank communicator equals the single-GPU path."""
    w = datagen.WORKLOADS["C2"]
    N = 200_000
    X = datagen.generate(w, N=N)
    init = datagen.one_per_blob_init(w, N=N)
    uid = km.comm_unique_id()
    comm = km.comm_init(1, uid, 0, 0)
    try:
        with km.Context(X, w.M, comm=comm, global_offset=0, global_N=N) as c:
            rd = c.fit(init, w.tol, w.max_iter)
            assert c.info()["nranks"] == 1
    finally:
        km.comm_destroy(comm)
    with km.Context(X, w.M) as c:
        rs = c.fit(init, w.tol, w.max_iter)
    assert rd["iters"] == rs["iters"]
    assert np.array_equal(rd["labels"], rs["labels"])
    assert np.array_equal(rd["centroids"], rs["centroids"])


@pytest.mark.parametrize("name,N,start,count", [("C1", 10_000, 0, 10_000),
                                                ("C5", 2_000_000, 0, 2_000_000),
                                                ("C4", 1_000_000_000, 625_000_000, 3_000_001),
                                                ("C3", 100_000_000, 77_777_777, 1_000_000)])
def test_device_generator_matches_host_recipe(name, N, start, count):
    """kmeans_generate reproduces datagen.generate: blob
    choice and planted sites exactly; coordinates bit-identical except where
    the device libm's fp64 log1p / cos / sin differ from the host's by an ulp,
    which may move an fp32 value by one ulp (a tiny fraction, bounded here)."""
    import torch
    w = datagen.WORKLOADS[name]
    host = datagen.generate(w, start, count, N=N)
    dev = torch.empty((count, w.d), dtype=torch.float32, device="cuda")
    km.generate(datagen.mixture_spec(w, N), start, count, dev)
    got = dev.cpu().numpy()
    diff = got != host
    frac = diff.mean()
    assert frac <= 1e-5, frac
    if diff.any():
        ulp = np.abs(got.view(np.int32).astype(np.int64) - host.view(np.int32).astype(np.int64))
        assert ulp[diff].max() == 1
    if w.planted_sites:
        p = datagen.planted_indices(w, N)
        p = p[(p >= start) & (p < start + count)] - start
        assert np.array_equal(got[p], host[p])


def test_generator_and_memory_cache_edges():
    """kmeans_generate rejects out-of-range requests; kmeans_release_memory
    empties the block cache and later contexts still work."""
    import torch
    w = datagen.WORKLOADS["C2"]
    spec = datagen.mixture_spec(w, 1000)
    out = torch.empty((10, 3), dtype=torch.float32, device="cuda")
    with pytest.raises(km.KMeansError) as e:
        km.generate(spec, 995, 10, out)   # past N
    assert e.value.name == "KMEANS_EINVAL"
    km.generate(spec, 990, 10, out)
    assert np.array_equal(out.cpu().numpy(), datagen.generate(w, 990, 10, N=1000))
    X = datagen.generate(w, N=50_000)
    init = datagen.init_indices(w, N=50_000)
    with km.Context(X, 8) as c:
        a = c.fit(init, 0.0, 3)
    km.release_memory(0)
    with km.Context(X, 8) as c:
        b = c.fit(init, 0.0, 3)
    assert np.array_equal(a["centroids"], b["centroids"])


def test_contexts_with_different_smem_sizes_interleave():
    """Kernels' shared-memory limits are process-wide: a context needing
    less (smaller K, smaller shard) must not shrink the limit under a live
    context that needs more (the large-K full scan)."""
    w = datagen.WORKLOADS["C5"]
    X = datagen.generate(w, N=60_000)
    # the same k_assign_large instance (8 points per lane, one block per SM)
    # at ~144 KB and ~120 KB of shared memory
    big = km.Context(X, 600, sort=False)
    small = km.Context(X[:20_000], 500, sort=False)
    mu_b = perturbed_centroids(X, 600, 7)
    mu_s = perturbed_centroids(X[:20_000], 500, 8)
    try:
        gb = big.assign(mu_b)
        gs = small.assign(mu_s)
        gb2 = big.assign(mu_b)                # after the small context configured
        assert np.array_equal(gb["labels"], gb2["labels"])
        assert np.array_equal(gb["labels"], oracle.step(X, mu_b)["labels"])
        assert np.array_equal(gs["labels"], oracle.step(X[:20_000], mu_s)["labels"])
    finally:
        big.close()
        small.close()
    w2 = datagen.WORKLOADS["C2"]
    Xa = datagen.generate(w2, N=400_000)      # fused kernel
    init = datagen.init_indices(w2, N=400_000)
    a = km.Context(Xa, 8)
    b = km.Context(Xa[:5_000], 8)             # fused, smaller grid
    try:
        ra = a.fit(init, 0.0, 3)
        b.fit(datagen.init_indices(w2, N=5_000), 0.0, 3)
        ra2 = a.fit(init, 0.0, 3)
        assert np.array_equal(ra["centroids"], ra2["centroids"])
    finally:
        a.close()
        b.close()


def test_interleaved_contexts_reuse_cached_blocks():
    """Contexts created and destroyed in an interleaved order (device blocks
    and the pinned state mirrors come back from the caches) each keep their
    own state: every run matches a run on a fresh context, and the stop rule
    of one does not leak into another."""
    w = datagen.WORKLOADS["C2"]
    X = datagen.generate(w, N=40_000)
    init = datagen.init_indices(w, N=40_000)
    with km.Context(X, 8) as c:
        ref = c.fit(init, 0.0, 4)
        ref_conv = c.fit(init, 1e-6, 100)
    live = []
    for i in range(24):
        live.append(km.Context(X, 8, sort=bool(i % 2)))
        if i % 3 == 2:   # destroy an older one while others stay alive
            live.pop(0).close()
    for i, c in enumerate(live):
        r = c.fit(init, 0.0, 4) if i % 2 else c.fit(init, 1e-6, 100)
        e = ref if i % 2 else ref_conv
        assert r["iters"] == e["iters"], i
        assert np.allclose(r["centroids"], e["centroids"], rtol=1e-9, atol=1e-9), i
    for c in live:
        c.close()


@pytest.mark.parametrize("P,n,rounds", [(1, 5, 3), (2, 65, 6), (3, 1, 4), (8, 4097, 5),
                                         (16, 33, 9), (64, 200, 3)])
def test_p2p_exchange_protocol_emulated(P, n, rounds):
    """The P2P exchange with P emulated ranks as the blocks
    of one cooperative launch: every rank receives, bit for bit, the rank-order
    sum of all ranks' vectors, every round (slot reuse, epochs)."""
    rng = np.random.default_rng(P * 1000 + n)
    vals = rng.standard_normal((rounds, P, n)) * 10.0 ** rng.integers(-3, 8, (rounds, P, n))
    out = km.p2p_selftest(vals)
    for i in range(rounds):
        expect = np.zeros(n)
        for q in range(P):   # rank order, fp64
            expect = expect + vals[i, q]
        for r in range(P):
            assert np.array_equal(out[i, r], expect), (i, r)


@pytest.mark.parametrize("sort", SORT)
@pytest.mark.parametrize("K", [8, 40])
def test_p2p_single_rank_iteration(sort, K):
    """The iteration with the exchange over peer memory (k_p2p_update, 1-rank
    communicator: the rank maps only itself) equals the single-GPU run."""
    w = datagen.WORKLOADS["C2"]
    N = 200_000
    X = datagen.generate(w, N=N)
    init = datagen.one_per_blob_init(w, N=N) if K == 8 else datagen.init_indices(w, N=N, K=K)
    uid = km.comm_unique_id()
    comm = km.comm_init(1, uid, 0, 0)
    try:
        with km.Context(X, K, comm=comm, global_offset=0, global_N=N, **ctx_kwargs(sort)) as c:
            c.p2p_open([c.p2p_handle()])
            rd = c.fit(init, w.tol, w.max_iter)
            a = c.assign(rd["centroids"])
            with pytest.raises(km.KMeansError):
                c.p2p_open([c.p2p_handle()])   # only once
    finally:
        km.comm_destroy(comm)
    with km.Context(X, K, **ctx_kwargs(sort)) as c:
        rs = c.fit(init, w.tol, w.max_iter)
        b = c.assign(rs["centroids"])
    assert rd["iters"] == rs["iters"]
    assert np.array_equal(rd["labels"], rs["labels"])
    assert np.array_equal(rd["centroids"], rs["centroids"])
    assert np.array_equal(a["counts"], b["counts"]) and np.array_equal(a["sums"], b["sums"])


def test_p2p_disable_returns_to_nccl():
    """kmeans_p2p_disable after a P2P run: the next run uses the NCCL
    allreduce (graphs rebuilt) and gives the same result."""
    w = datagen.WORKLOADS["C2"]
    N = 100_000
    X = datagen.generate(w, N=N)
    init = datagen.one_per_blob_init(w, N=N)
    comm = km.comm_init(1, km.comm_unique_id(), 0, 0)
    try:
        with km.Context(X, w.M, comm=comm, global_offset=0, global_N=N) as c:
            c.p2p_open([c.p2p_handle()])
            a = c.fit(init, w.tol, w.max_iter)
            c.p2p_disable()
            b = c.fit(init, w.tol, w.max_iter)
    finally:
        km.comm_destroy(comm)
    assert a["iters"] == b["iters"] and np.array_equal(a["centroids"], b["centroids"])
    assert np.array_equal(a["labels"], b["labels"])


# --------------------------------------------------------------------------
# full-size checks in the launch configuration bench.py times
# --------------------------------------------------------------------------
@pytest.mark.slow
@pytest.mark.parametrize("sort", SORT)
def test_full_size_ns_step_parity(sort):
    """BASELINE north-star size (N=1e8, 3D, K=16): one full step against the
    oracle on all N points (labels bit-exact, counts exact, sums / J / mu / E
    per R13), through the same Context configuration bench.py uses."""
    w = datagen.WORKLOADS["NS"]
    X = datagen.generate(w)
    mu = X[datagen.init_indices(w)].astype(np.float64)
    with km.Context(X, w.K, **ctx_kwargs(sort)) as c:
        info = c.info()
        assert info["path"] == 0 and info["sorted"] == int(bool(sort))
        assert info["grid"] == (w.N + 2047) // 2048   # 2048-point chunks at this N (both paths)
        check_step(X, mu, ctx=c, tag="NS full")


@pytest.mark.slow
def test_full_size_c3_step_parity():
    """C3 at P = 1 (N=1e8, 2D, K=16): one full step against the oracle on all
    N points, in the launch configuration bench.py --workload C3 uses."""
    w = datagen.WORKLOADS["C3"]
    X = datagen.generate(w)
    mu = X[datagen.init_indices(w)].astype(np.float64)
    with km.Context(X, w.K) as c:
        assert c.info()["sorted"] == 1
        check_step(X, mu, ctx=c, tag="C3 full")


# Full-size oracle in a process pool: oracle.partials (single-threaded C) over
# fixed contiguous shards, one per worker call, the shard partials added in
# shard order.  Children are forked and read the arrays below (copy-on-write);
# they compare the GPU's labels themselves and return only small results.
_POOL = {}


def _pool_shard(job):
    import oracle as _o
    lo, hi = job
    X, mu, lab_g = _POOL["X"], _POOL["mu"], _POOL["labels"]
    r = _o.partials(X[lo:hi], mu)
    bad = np.nonzero(r["labels"] != lab_g[lo:hi])[0]
    K, d = mu.shape
    scale = np.zeros((K, d))
    for j in range(d):
        scale[:, j] = np.bincount(r["labels"], weights=np.abs(X[lo:hi, j].astype(np.float64)),
                                  minlength=K)
    return dict(sums=r["sums"], counts=r["counts"], J=r["J"], scale=scale,
                n_bad=int(bad.size), first_bad=(lo + bad[:5]).tolist())


def oracle_step_pooled(X, mu, labels_gpu, shard=1_000_000):
    """One oracle step over all of X (labels compared element by element in
    the workers), sums / counts / J added over shards in ascending order, then
    oracle.update -- the same arithmetic as oracle.step up to the fp64
    summation order across shards (within reading R13's bar)."""
    import multiprocessing as mp
    _POOL.update(X=X, mu=mu, labels=labels_gpu)
    jobs = [(lo, min(lo + shard, X.shape[0])) for lo in range(0, X.shape[0], shard)]
    with mp.get_context("fork").Pool(max(1, os.cpu_count() or 1)) as pool:
        parts = pool.map(_pool_shard, jobs, chunksize=1)
    _POOL.clear()
    K, d = mu.shape
    sums, counts, J, scale = np.zeros((K, d)), np.zeros(K, np.int64), 0.0, np.zeros((K, d))
    n_bad, first_bad = 0, []
    for p in parts:   # shard order
        sums = sums + p["sums"]
        counts = counts + p["counts"]
        J = J + p["J"]
        scale = scale + p["scale"]
        n_bad += p["n_bad"]
        first_bad += p["first_bad"]
    mu_next, E = oracle.update(sums, counts, mu)
    return dict(sums=sums, counts=counts, J=J, scale=scale, mu_next=mu_next, E=E,
                n_bad=n_bad, first_bad=first_bad[:5])


def check_step_full(g, mu_next, E, o, mu, tag):
    """check_step's bars, against oracle_step_pooled (all labels, every
    per-cluster sum and count, J, mu^{t+1}, E)."""
    assert o["n_bad"] == 0, f"{tag}: {o['n_bad']} labels differ, first at {o['first_bad']}"
    assert np.array_equal(g["counts"], o["counts"]), tag
    assert np.all(np.abs(g["sums"] - o["sums"]) <= REL * o["scale"] + 1e-300), tag
    assert abs(g["inertia"] - o["J"]) <= REL * o["J"], tag
    n = np.maximum(o["counts"], 1)[:, None]
    mscale = np.maximum(np.abs(o["mu_next"]), o["scale"] / n)
    assert np.all(np.abs(mu_next - o["mu_next"]) <= REL * mscale + 1e-300), tag
    dmu = REL * mscale
    e_tol = np.sum(2 * np.abs(o["mu_next"] - mu) * dmu + dmu ** 2) + \
        REL * max(o["E"], 1e-3 * float(np.sum(mu ** 2)))
    assert abs(E - o["E"]) <= e_tol, f"{tag}: E {E} vs {o['E']}"


@pytest.mark.slow
def test_full_size_c4_rank_shard_parity():
    """C4 (N=1e9, 3D, K=16, P=8): the shard of rank 5 (1.25e8 points, global
    offset 6.25e8) as bench.py --gpus 8 generates it, one step at the global
    init centroids: every label, count and per-cluster sum, J, mu^{t+1} and E
    against the oracle (process pool over fixed shards)."""
    w = datagen.WORKLOADS["C4"]
    P, r = 8, 5
    a, b = datagen.shard_range(w.N, P, r)
    Xs = datagen.generate(w, a, b - a)
    init = datagen.init_indices(w)
    rows = np.stack([datagen.generate(w, int(i), 1)[0] for i in init])   # global init points
    mu = rows.astype(np.float64)
    with km.Context(Xs, w.K) as c:   # (global offsets need a communicator; assign takes mu)
        assert c.info()["sorted"] == 1
        g = c.assign(mu)
        mu_next, E = c.update()
    o = oracle_step_pooled(Xs, mu, g["labels"], shard=4_000_000)
    check_step_full(g, mu_next, E, o, mu, "C4 rank 5")


@pytest.mark.slow
def test_full_size_c5_parity():
    """C5 (N=5e7, 3D, K=1024, forced empty clusters) at full size, in the
    configuration bench.py --workload C5 times: every label, all 1024 counts
    (the 56 forced-empty clusters included) and per-cluster sums, J,
    mu^{t+1} and E against the oracle (process pool; R2)."""
    w = datagen.WORKLOADS["C5"]
    X = datagen.generate(w)
    init = datagen.init_indices(w)
    mu = X[init].astype(np.float64)
    with km.Context(X, w.K) as c:
        assert c.info()["sorted"] == 1
        g = c.assign(mu)
        mu_next, E = c.update()
    o = oracle_step_pooled(X, mu, g["labels"], shard=250_000)
    check_step_full(g, mu_next, E, o, mu, "C5 full")
    for s in range(w.planted_sites):   # R2: 7 of every site's 8 centroids stay empty
        ks = list(range(8 * s, 8 * s + 8))
        assert g["counts"][ks[0]] >= 8 and all(g["counts"][k] == 0 for k in ks[1:])
        assert np.array_equal(mu_next[ks[1:]], mu[ks[1:]])


@pytest.mark.parametrize("d,K", [(3, 100), (3, 128), (2, 100), (2, 300)])
def test_heavy_tiles_mid_k(d, K):
    """Heavy chunks at 64 < K <= 128 (each tile's stretch of the chunk row is
    K < 128 entries) and in 2D: k_assign_heavy_tiles against the oracle, one
    step and a 2-iteration fit through the iteration graph."""
    rng = np.random.default_rng(1000 + 10 * K + d)
    w = datagen.WORKLOADS["NS" if d == 3 else "C3"]
    N = 100_003
    X = datagen.generate(w, N=N)
    far = rng.uniform(-3000, 3000, (5000, d)).astype(np.float32)
    X[rng.choice(N, 5000, replace=False)] = far
    init = rng.choice(N, K, replace=False)
    mu = X[init].astype(np.float64)
    with km.Context(X, K, sort=True) as c:
        check_step(X, mu, ctx=c, tag=f"heavy d={d} K={K}")
        st = c.candidate_stats()
    assert st["max"] > 64, st   # the heavy path was exercised
    o1 = oracle.fit(X, K, init, 0.0, 2)
    with km.Context(X, K, sort=True) as c:
        r = c.fit(init, 0.0, 2)
    assert np.array_equal(r["labels"], o1["labels"])


def test_heavy_chunks_large_k():
    """Large K with far outliers and sparse tails: chunk boxes that span huge
    empty regions keep more than 64 candidates and go to k_assign_heavy_tiles
    (one block per 128-point tile); labels must stay bit-exact."""
    rng = np.random.default_rng(21)
    w = datagen.WORKLOADS["C5"]
    X = datagen.generate(w, N=200_000)
    # a sparse shell of far points between the blobs and the planted sites
    far = rng.uniform(-3000, 3000, (3000, 3)).astype(np.float32)
    X[rng.choice(200_000, 3000, replace=False)] = far
    init = datagen.init_indices(w, N=200_000)
    mu = X[init].astype(np.float64)
    with km.Context(X, w.K) as c:
        g, o = check_step(X, mu, ctx=c, tag="heavy")
        st = c.candidate_stats()
    assert st["max"] > 64, st   # the heavy path was exercised
    # a 2-step run through the iteration graph (prune -> assign -> heavy -> merges)
    o1 = oracle.fit(X, w.K, init, 0.0, 2)
    with km.Context(X, w.K) as c:
        r = c.fit(init, 0.0, 2)
    assert np.array_equal(r["labels"], o1["labels"])


@pytest.mark.gpu
@pytest.mark.parametrize("n_blobs", [1, 2, 5])
def test_large_k_row_merge_repeated_k_windows(n_blobs):
    """Large-K row merge (k_merge_sparse) when consecutive chunks hold the same
    few clusters: K = 64 with only n_blobs occupied, so each chunk row has 1-2
    entries and one 32-entry window of the merge repeats the same k up to 31
    times (the __match_any_sync rounds).  Counts must stay exact and sums,
    inertia, mu^{t+1}, E within the step bars; the other 64 - n_blobs clusters
    are empty and keep their centroids."""
    rng = np.random.default_rng(100 + n_blobs)
    N, K = 500_003, 64
    centers = rng.uniform(-50, 50, (n_blobs, 3))
    X = (centers[rng.integers(0, n_blobs, N)] + rng.normal(0, 1.0, (N, 3))).astype(np.float32)
    mu = np.concatenate([centers, rng.uniform(1e3, 2e3, (K - n_blobs, 3))]).astype(np.float64)
    g, o = check_step(X, mu, tag=f"repeated-k {n_blobs}")
    assert np.count_nonzero(o["counts"]) == n_blobs


# --------------------------------------------------------------------------
# failure behaviour of the distributed path, trace sizing, path choice
# --------------------------------------------------------------------------
@pytest.mark.parametrize("P,dead", [(2, 1), (4, 0), (8, 5)])
def test_p2p_exchange_dead_rank_times_out(P, dead):
    """A rank that never publishes (dead or hung peer): every other emulated
    rank gives up after the timeout -- the exchange fails with KMEANS_ENCCL
    in round 1 instead of spinning forever (kernels.cuh p2p_exchange)."""
    vals = np.ones((3, P, 17))
    failed = np.zeros(P, np.int32)
    with pytest.raises(km.KMeansError) as e:
        km.p2p_selftest(vals, dead_rank=dead, timeout_s=0.05, failed=failed)
    assert e.value.name == "KMEANS_ENCCL"
    assert failed[dead] == 0
    assert all(failed[r] == 1 for r in range(P) if r != dead), failed


def test_p2p_only_group_without_nccl():
    """A P2P-only context (opts.rank / opts.nranks, no NCCL communicator):
    iterating before kmeans_p2p_open is KMEANS_ESTATE; after opening (1 rank:
    it maps only itself) the run equals the single-GPU run bit for bit."""
    w = datagen.WORKLOADS["C2"]
    N = 120_000
    X = datagen.generate(w, N=N)
    init = datagen.one_per_blob_init(w, N=N)
    with km.Context(X, w.M) as c:
        ref = c.fit(init, w.tol, w.max_iter)
    with km.Context(X, w.M, rank=0, nranks=1) as c:
        assert c.info()["nranks"] == 1 and c.info()["fused"] == 0
        with pytest.raises(km.KMeansError) as e:
            c.fit(init, w.tol, w.max_iter)
        assert e.value.name == "KMEANS_ESTATE"
        c.p2p_open([c.p2p_handle()])
        r = c.fit(init, w.tol, w.max_iter)
    assert r["iters"] == ref["iters"]
    assert np.array_equal(r["labels"], ref["labels"])
    assert np.array_equal(r["centroids"], ref["centroids"])


def test_p2p_open_failure_is_not_sticky():
    """a failing cudaIpcOpenMemHandle (corrupt peer handle) returns
    KMEANS_ECUDA without poisoning the context: it answers later calls, and a
    second open attempt is still possible."""
    X = datagen.generate(datagen.WORKLOADS["C2"], N=10_000)
    with km.Context(X, 8, rank=0, nranks=2, global_N=20_000) as c:
        own = c.p2p_handle()
        with pytest.raises(km.KMeansError) as e:
            c.p2p_open([own, bytes(64)])
        assert e.value.name == "KMEANS_ECUDA"
        assert c.info()["nranks"] == 2          # not sticky
        c.p2p_disable()
        with pytest.raises(km.KMeansError) as e:
            c.p2p_open([own, b"\x01" * 64])
        assert e.value.name == "KMEANS_ECUDA"


def test_start_does_not_size_traces_by_max_iter():
    """kmeans_start(max_iter = 2^30) must not allocate 2 x 8 GiB of
    E/J traces; kmeans_fit_ctx with caller trace buffers beyond the default
    cap still returns every iteration's E and J."""
    import torch
    w = datagen.WORKLOADS["C1"]
    X = datagen.generate(w)
    init = datagen.init_indices(w)
    with km.Context(X, w.K, fused=False) as c:
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
        c.start(init_idx=init, tol=0.0, max_iter=1 << 30)
        c.iterate(3)
        assert c.poll()["iters"] == 3
        free1 = torch.cuda.mem_get_info()[0]
        assert free0 - free1 < (256 << 20), (free0 - free1)
    with km.Context(X, w.K) as c:
        r = c.fit(init, 0.0, 5000)
    o = oracle.fit(X, w.K, init, 0.0, 30)
    assert r["iters"] == 5000 and r["E_trace"].shape == (5000,)
    assert np.array_equal(r["E_trace"][30:], np.zeros(4970))   # converged long before
    np.testing.assert_allclose(r["J_trace"][:30], o["J_trace"], rtol=1e-9)


def test_expected_iters_weighs_the_sort():
    """opts.expected_iters: at N K d >= 3.84e8 (K <= 16) the sorted path is the
    default, but a 20-iteration run does not pay back the create-time sort
    (DESIGN.md section 5): full scan.  Results are identical either way."""
    w = datagen.WORKLOADS["NS"]
    N = 8_100_000
    X = datagen.generate(w, N=N)
    init = datagen.init_indices(w, N=N)
    res = {}
    for hint, sorted_ in [(0, 1), (20, 0), (1000, 1)]:
        with km.Context(X, w.K, expected_iters=hint) as c:
            assert c.info()["sorted"] == sorted_, hint
            res[hint] = c.fit(init, 0.0, 3)
    for hint in (20, 1000):
        assert np.array_equal(res[hint]["labels"], res[0]["labels"])
        np.testing.assert_allclose(res[hint]["centroids"], res[0]["centroids"], rtol=1e-12)


# --------------------------------------------------------------------------
# k_persist_iterate (sorted path, K <= 16: the whole iteration in one kernel)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("big", [False, True])
@pytest.mark.parametrize("name,N,K", [("NS", 1_100_003, 16), ("C3", 1_300_000, 16),
                                      ("C2", 1_200_000, 8), ("C1", 1_400_001, 4),
                                      ("NS", 300_001, 16), ("NS", 1_000, 3)])
def test_persistent_iteration_matches_oracle(name, N, K, big):
    """The persistent kernel (one launch, many iterations, static unit ranges,
    last-arriver block / grid merges, flag-released updates) against the
    oracle over several iterations -- labels and counts exact, centroids per
    R13 -- and against the multi-kernel path (same labels, centroids within
    1e-12), including launches split at arbitrary iteration counts.  Shards
    too small to give every warp of the grid a 256-point unit (the last two
    cases) run the multi-kernel path instead."""
    w = datagen.WORKLOADS[name]
    X = datagen.generate(w, N=N)
    init = datagen.init_indices(w, N=N, K=K)
    T = 7
    o = oracle.fit(X, K, init, 0.0, T)
    with km.Context(X, K, sort=True, big_chunks=big, persist=True) as c:
        assert c.info()["persistent"] == int(N > 1_000_000)
        r = c.fit(init, 0.0, T)
        c.start(init_idx=init, tol=0.0, max_iter=T)
        for n in (1, 2, 3, 5):   # 1 + 2 + 3 + (1 of 5: max_iter stops it)
            c.iterate(n)
        st = c.poll()
        assert st["iters"] == T and st["done"]
        split = c.read_centroids()
        split_labels = c.final_labels()
    with km.Context(X, K, sort=True, big_chunks=big) as c:
        assert c.info()["persistent"] == 0
        g = c.fit(init, 0.0, T)
    assert r["iters"] == T
    assert np.array_equal(r["labels"], o["labels"])
    assert np.array_equal(r["labels"], g["labels"]) and np.array_equal(split_labels, r["labels"])
    np.testing.assert_allclose(r["centroids"], o["centroids"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(r["centroids"], g["centroids"], rtol=1e-12, atol=1e-14)
    assert np.array_equal(split, r["centroids"])   # same bits however the launches are split
    np.testing.assert_allclose(r["J_trace"], o["J_trace"], rtol=1e-9)


def test_persistent_stop_rule_inside_a_launch():
    """E < tol fires in the middle of one persistent launch: the iteration
    count is the oracle's, later iterations are no-ops, and the next launch
    returns immediately."""
    w = datagen.WORKLOADS["NS"]
    N = 1_500_000
    X = datagen.generate(w, N=N)
    init = datagen.one_per_blob_init(w, N=N)
    o = oracle.fit(X, w.M, init, w.tol, w.max_iter)
    with km.Context(X, w.M, sort=True, persist=True) as c:
        assert c.info()["persistent"] == 1
        c.start(init_idx=init, tol=w.tol, max_iter=w.max_iter)
        c.iterate(w.max_iter)
        st = c.poll()
        assert st["done"] and st["iters"] == o["iters"]
        c.iterate(10)
        assert c.poll()["iters"] == o["iters"]
        cent = c.read_centroids()
        lab = c.final_labels()
    assert np.array_equal(lab, o["labels"])
    np.testing.assert_allclose(cent, o["centroids"], rtol=1e-9)


def test_persistent_deterministic_and_p2p_single_rank():
    """Bit-reproducible across runs and contexts (dynamic chunk tickets do not
    change the sums), and a 1-rank P2P group runs the exchange inside the
    persistent kernel with the same bits as the single-GPU run."""
    w = datagen.WORKLOADS["NS"]
    N = 1_600_000
    X = datagen.generate(w, N=N)
    init = datagen.init_indices(w, N=N)
    runs = []
    for _ in range(2):
        with km.Context(X, 16, sort=True, persist=True) as c:
            runs.append(c.fit(init, 0.0, 6))
            runs.append(c.fit(init, 0.0, 6))
    with km.Context(X, 16, sort=True, persist=True, rank=0, nranks=1) as c:
        c.p2p_open([c.p2p_handle()])
        assert c.info()["persistent"] == 1
        runs.append(c.fit(init, 0.0, 6))
    for r in runs[1:]:
        assert np.array_equal(r["labels"], runs[0]["labels"])
        assert np.array_equal(r["centroids"], runs[0]["centroids"])
        assert np.array_equal(r["E_trace"], runs[0]["E_trace"])


def test_nccl_wait_is_bounded_and_aborts():
    """With an NCCL communicator the host wait polls the stream and the
    communicator; a collective that does not finish within comm_timeout_s
    (here a deliberately tiny 1 us, so the first long wait trips it) aborts
    the communicator and fails with a sticky KMEANS_ENCCL instead of
    blocking; kmeans_comm_destroy then skips the aborted communicator."""
    w = datagen.WORKLOADS["C2"]
    N = 2_000_000
    X = datagen.generate(w, N=N)
    init = datagen.init_indices(w, N=N)
    comm = km.comm_init(1, km.comm_unique_id(), 0, 0)
    c = km.Context(X, w.K, comm=comm, global_offset=0, global_N=N, comm_timeout_s=1e-6)
    try:
        c.start(init_idx=init, tol=0.0, max_iter=1000)   # (its own waits may trip first)
        c.iterate(500)
        c.poll()
        raised = None
    except km.KMeansError as e:
        raised = e
    assert raised is not None and raised.name == "KMEANS_ENCCL", raised
    with pytest.raises(km.KMeansError) as e2:   # sticky
        c.poll()
    assert e2.value.name == "KMEANS_ENCCL"
    c.close()
    km.comm_destroy(comm)   # already aborted: skipped, no double free
