"""Pins for the CPU oracle (oracle/lloyd_oracle.c) -- no GPU needed.

Every oracle function is checked against something other than itself:
hand-derived worked examples (tests/golden), SPEC.md's printed examples,
exhaustive enumeration of all K^N assignments, exact rational arithmetic
(fractions), closed forms, invariants of Lloyd's method and scikit-learn's
Lloyd.  Chosen so that a plausible mistake (a dropped coordinate, a wrong sign,
a wrong index, a transposed operand, a missing empty-cluster rule, a sqrt in E)
fails at least one of them.
"""
import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_2405_12052_b200 import datagen

pytestmark = pytest.mark.filterwarnings("ignore::DeprecationWarning")


def load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------------------
# Form-D distance (reading R6)
# ---------------------------------------------------------------------------
def test_spec_squared_l2_examples(golden_dir):
    g = load(golden_dir, "spec_examples.json")
    for ex in g["squared_l2"]:
        assert float(oracle.dist(ex["a"], ex["b"])) == ex["expect"]


@pytest.mark.parametrize("d", [1, 2, 3, 5])
def test_dist_exact_on_integers(d):
    """|v| < 2^10 integers: every fp32 op of form D is exact, so D must equal
    the integer sum of squares (catches dropped terms, sign and index errors)."""
    rng = np.random.default_rng(7 + d)
    for _ in range(300):
        x = rng.integers(-1023, 1024, d)
        c = rng.integers(-1023, 1024, d)
        assert float(oracle.dist(x, c)) == float(sum(int(a - b) ** 2 for a, b in zip(x, c)))


@pytest.mark.parametrize("d", [2, 3])
def test_dist_within_rounding_bound_of_exact(d):
    """Random reals: form D is within (d+2) * 2^-24 relative of the exact
    rational distance between the same fp32 operands."""
    rng = np.random.default_rng(11 + d)
    for _ in range(500):
        x = rng.normal(0, 10, d).astype(np.float32)
        c = rng.normal(0, 10, d).astype(np.float32)
        exact = sum((Fraction(float(a)) - Fraction(float(b))) ** 2 for a, b in zip(x, c))
        got = Fraction(float(oracle.dist(x, c)))
        assert abs(got - exact) <= Fraction(d + 2, 2 ** 24) * exact


def test_dist_symmetry_and_zero():
    rng = np.random.default_rng(3)
    for _ in range(200):
        a = rng.normal(0, 100, 3).astype(np.float32)
        b = rng.normal(0, 100, 3).astype(np.float32)
        assert oracle.dist(a, b) == oracle.dist(b, a)
        assert float(oracle.dist(a, a)) == 0.0


def test_dist_fma_step_single_rounding(golden_dir):
    """Form D's fma step rounds ONCE (reading R6): the
    hand-derived value of tests/golden/fma_form_d.json, which a separately
    rounded s + e_j*e_j (or another coordinate order) misses by one ulp."""
    g = load(golden_dir, "fma_form_d.json")
    d2 = g["distance_2d"]
    assert float(oracle.dist(d2["x"], d2["c"])) == d2["expect"]
    assert d2["expect"] != d2["separately_rounded_would_give"]
    a = g["argmin_3d"]
    for c, want in zip(a["centroids"], a["expect_dist"]):
        assert float(oracle.dist(a["x"], c)) == want


def test_argmin_decided_by_fma_rounding(golden_dir):
    """The label of golden argmin_3d: with form D's single rounding centroid 1
    is strictly nearer; a separately rounded evaluation would tie and give 0."""
    a = load(golden_dir, "fma_form_d.json")["argmin_3d"]
    X = np.array([a["x"]] * 3, np.float32)
    r = oracle.partials(X, np.array(a["centroids"], float))
    assert r["labels"].tolist() == [a["expect_label"]] * 3
    assert [float(v) for v in r["dmin"]] == [a["expect_dmin"]] * 3
    assert r["J"] == 3 * a["expect_dmin"]


def test_dist_operand_order_matters_not_reassociated():
    """Form D subtracts per coordinate before squaring.  The expanded form
    |x|^2 - 2x.c + |c|^2 loses everything here (catastrophic cancellation);
    form D gives the exact 1.0."""
    x = np.array([16777216.0, 0.0], np.float32)   # 2^24
    c = np.array([16777215.0, 0.0], np.float32)
    assert float(oracle.dist(x, c)) == 1.0


# ---------------------------------------------------------------------------
# Argmin with lowest-index ties (reading R1)
# ---------------------------------------------------------------------------
def test_spec_tie_and_assign_examples(golden_dir):
    g = load(golden_dir, "spec_examples.json")
    t = g["tie_lowest_index"]
    r = oracle.partials(np.array([t["x"]], np.float32), np.array(t["centers"], float))
    assert r["labels"].tolist() == [t["expect_label"]]
    a = g["assign"]
    r = oracle.partials(np.array(a["points"], np.float32), np.array(a["centers"], float))
    assert r["labels"].tolist() == a["expect_labels"]


def _int_J(X, C, z):
    return sum(sum(int(X[i][j] - C[z[i]][j]) ** 2 for j in range(X.shape[1]))
               for i in range(X.shape[0]))


@pytest.mark.parametrize("seed", range(24))
def test_labels_are_lexicographically_smallest_minimiser_bruteforce(seed):
    """Exhaustive enumeration of all K^N assignments (N <= 7, K <= 3) with
    integer data (exact in fp32): the oracle's labels must minimise
    J(z) = sum ||x_i - mu_{z_i}||^2 and be the lexicographically smallest
    minimiser, which is exactly 'argmin per point, lowest index on ties'.
    Small coordinate range forces many exact ties."""
    rng = np.random.default_rng(seed)
    N = int(rng.integers(1, 8))
    K = int(rng.integers(1, 4))
    d = int(rng.integers(1, 4))
    X = rng.integers(-3, 4, (N, d)).astype(np.float32)
    C = rng.integers(-3, 4, (K, d)).astype(np.float64)
    r = oracle.partials(X, C)
    best, best_z = None, None
    for z in itertools.product(range(K), repeat=N):   # lexicographic order
        J = _int_J(X, C, z)
        if best is None or J < best:
            best, best_z = J, z
    assert tuple(r["labels"].tolist()) == best_z
    assert r["J"] == float(best)
    assert r["counts"].sum() == N


def test_staging_rounds_mu_to_fp32_once(golden_dir):
    """Reading R7: the fp64 centroid is rounded to fp32 before distances.  A
    point halfway between two fp64 centroids that round to the same fp32 value
    is a tie -> label 0; an fp64-distance oracle would pick label 1."""
    x = np.array([[1.0]], np.float32)
    c = np.array([[1.0 + 2.0 ** -40], [1.0 - 2.0 ** -41]])   # both stage to 1.0f
    r = oracle.partials(x, c)
    assert r["labels"].tolist() == [0]
    assert float(r["dmin"][0]) == 0.0


# ---------------------------------------------------------------------------
# Mean calculation, empty clusters (R2), E
# ---------------------------------------------------------------------------
def test_spec_update_and_shift_examples(golden_dir):
    g = load(golden_dir, "spec_examples.json")
    u = g["update"]
    X = np.array(u["members"], np.float32)
    r = oracle.step(X, np.array([X[0]], float))
    assert r["mu_next"][0].tolist() == u["expect_center"]
    s = g["shift_error"]
    assert oracle.shift_error(np.array(s["prev"], float), np.array(s["next"], float)) == s["expect"]


def test_shift_error_closed_form():
    """E(mu, mu + delta) = K*d*delta^2 for an exactly representable delta;
    squared, no sqrt (reading R4)."""
    rng = np.random.default_rng(5)
    for K, d in [(1, 1), (4, 2), (16, 3), (1024, 3)]:
        mu = rng.integers(-1000, 1000, (K, d)).astype(np.float64)
        assert oracle.shift_error(mu, mu + 0.5) == K * d * 0.25
        assert oracle.shift_error(mu, mu) == 0.0


@pytest.mark.parametrize("seed", range(10))
def test_sums_and_means_match_exact_rationals(seed):
    """S_k and mu_k^{t+1} against exact rational sums of the same fp32 inputs;
    fp64 accumulation of n terms is within n * 2^-53 * sum|x| of exact."""
    rng = np.random.default_rng(100 + seed)
    N, K, d = 200, 5, 3
    X = rng.normal(0, 50, (N, d)).astype(np.float32)
    mu = X[rng.choice(N, K, replace=False)].astype(np.float64)
    r = oracle.step(X, mu)
    z = r["labels"]
    for k in range(K):
        members = np.nonzero(z == k)[0]
        assert r["counts"][k] == len(members)
        for j in range(d):
            exact = sum((Fraction(float(X[i, j])) for i in members), Fraction(0))
            absum = sum((abs(Fraction(float(X[i, j]))) for i in members), Fraction(0))
            bound = Fraction(len(members) + 1, 2 ** 53) * absum
            assert abs(Fraction(float(r["sums"][k, j])) - exact) <= bound
            if len(members):
                m_exact = exact / len(members)
                assert abs(Fraction(float(r["mu_next"][k, j])) - m_exact) <= \
                    bound / len(members) + abs(m_exact) * Fraction(1, 2 ** 52)
    # J: sum of the fp32 dmin values in fp64
    J_exact = sum((Fraction(float(v)) for v in r["dmin"]), Fraction(0))
    assert abs(Fraction(r["J"]) - J_exact) <= Fraction(N, 2 ** 53) * J_exact
    # dmin is the form-D distance to the chosen centroid
    c32 = mu.astype(np.float32)
    for i in range(0, N, 17):
        assert oracle.dist(X[i], c32[z[i]]) == r["dmin"][i]


def test_empty_cluster_keeps_previous_centroid():
    """Reading R2: a centroid planted far away gets no points and stays
    bit-identical; its shift contributes 0 to E."""
    X = np.array([[0, 0], [1, 0], [0, 1]], np.float32)
    mu = np.array([[0.25, 0.25], [1e6 + 0.1, -3.3]])
    r = oracle.step(X, mu)
    assert r["counts"].tolist() == [3, 0]
    assert r["mu_next"][1].tolist() == mu[1].tolist()
    assert r["E"] == oracle.shift_error(mu[:1], r["mu_next"][:1])


def test_k1_gives_dataset_mean():
    rng = np.random.default_rng(9)
    X = rng.normal(3, 2, (1000, 3)).astype(np.float32)
    res = oracle.fit(X, 1, [17], tol=1e-6, max_iter=10)
    for j in range(3):
        m = math.fsum(float(v) for v in X[:, j]) / 1000
        assert abs(res["centroids"][0, j] - m) <= 1e-12 * max(1.0, abs(m))
    assert res["iters"] == 2     # step 2 recomputes the same mean: E = 0
    assert res["labels"].tolist() == [0] * 1000


def test_k_equals_n_each_point_its_own_centre():
    """k == n -> every point its own centre, counts all 1;
    J = 0 and E = 0 at the first iteration (iters = 1)."""
    rng = np.random.default_rng(4)
    X = rng.normal(0, 1, (12, 2)).astype(np.float32)
    init = rng.permutation(12)
    res = oracle.fit(X, 12, init, tol=1e-6, max_iter=5)
    assert res["iters"] == 1 and res["inertia"] == 0.0
    for k, i in enumerate(init):
        assert res["labels"][i] == k
        assert res["centroids"][k].tolist() == X[i].astype(np.float64).tolist()


# ---------------------------------------------------------------------------
# The serial loop: hand-worked full runs
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["w1.json", "w2.json", "w3.json", "w4.json"])
def test_hand_worked_runs(golden_dir, name):
    g = load(golden_dir, name)
    X = np.array(g["points"], np.float32)
    K = len(g["init_idx"])
    res = oracle.fit(X, K, g["init_idx"], g["tol"], g["max_iter"])
    assert res["iters"] == g["iters"]
    assert res["E_trace"].tolist() == [it["E"] for it in g["per_iter"]]
    assert res["J_trace"].tolist() == [it["J"] for it in g["per_iter"]]
    assert res["labels"].tolist() == g["labels"]
    assert res["centroids"].tolist() == g["centroids"]
    assert res["inertia"] == g["inertia"]
    # per-iteration labels via the step function from the same mu^t
    mu = X[g["init_idx"]].astype(np.float64)
    for it in g["per_iter"]:
        r = oracle.step(X, mu)
        assert r["labels"].tolist() == it["labels"]
        assert r["J"] == it["J"] and r["E"] == it["E"]
        mu = r["mu_next"]


def test_max_iter_and_tol_zero():
    X = datagen.generate(datagen.WORKLOADS["C1"], N=2000)
    init = datagen.init_indices(datagen.WORKLOADS["C1"], N=2000)
    res = oracle.fit(X, 4, init, tol=0.0, max_iter=7)
    assert res["iters"] == 7                  # E < 0 never holds (R3)
    res1 = oracle.fit(X, 4, init, tol=1e-6, max_iter=1)
    assert res1["iters"] == 1


# ---------------------------------------------------------------------------
# Invariants of Lloyd's method on the paper-shaped synthetic data
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,N", [("C1", 10_000), ("C2", 20_000), ("C3", 20_000), ("C5", 20_000)])
def test_invariants_on_blobs(name, N):
    w = datagen.WORKLOADS[name]
    X = datagen.generate(w, N=N)
    K = min(w.K, 64)
    init = datagen.init_indices(w, N=N, K=K) if w.planted_sites == 0 else \
        datagen.init_indices(w, N=N)[:K]
    res = oracle.fit(X, K, init, tol=1e-6, max_iter=60)
    J = res["J_trace"]
    # inertia non-increasing up to fp32-distance slack (R10)
    assert np.all(J[1:] <= J[:-1] * (1 + 1e-6) + 1e-9)
    # each centroid equals the mean of its assigned points (north_star)
    z = res["labels"]
    counts = np.bincount(z, minlength=K)
    assert counts.sum() == N
    prev = res["centroids"]
    r = oracle.step(X, prev)
    assert np.array_equal(r["labels"], z) or res["iters"] == 60
    for k in range(K):
        if counts[k]:
            for j in range(w.d):
                m = math.fsum(float(v) for v in X[z == k, j]) / counts[k]
                assert abs(prev[k, j] - m) <= 1e-9 * max(1.0, abs(m))
    if res["iters"] < 60:
        # fixed point: rerunning from converged centroids gives E = 0
        assert r["E"] == 0.0


def test_planted_sites_force_empty_clusters():
    """C5 recipe: 8 sites x 8 duplicates, all 64 initial centroids on sites; per
    site the lowest k takes all duplicates, the other 7 stay empty."""
    w = datagen.WORKLOADS["C5"]
    N = 30_000
    X = datagen.generate(w, N=N)
    init = datagen.init_indices(w, N=N)[:80]
    mu = X[init].astype(np.float64)
    r = oracle.step(X, mu)
    for g in range(8):
        ks = list(range(8 * g, 8 * g + 8))
        assert r["counts"][ks[0]] == 8
        assert all(r["counts"][k] == 0 for k in ks[1:])
        for k in ks[1:]:
            assert r["mu_next"][k].tolist() == mu[k].tolist()


def test_deterministic():
    X = datagen.generate(datagen.WORKLOADS["C2"], N=5000)
    init = datagen.init_indices(datagen.WORKLOADS["C2"], N=5000)
    a = oracle.fit(X, 8, init, 1e-6, 50)
    b = oracle.fit(X, 8, init, 1e-6, 50)
    assert a["iters"] == b["iters"]
    assert np.array_equal(a["labels"], b["labels"])
    assert np.array_equal(a["centroids"], b["centroids"])
    assert np.array_equal(a["E_trace"], b["E_trace"])


def test_matches_sklearn_lloyd_on_well_separated_blobs():
    """A library Lloyd (scikit-learn, fp64 distances, its own stop rule) reaches
    the same fixed point on well-separated blobs with one init per blob."""
    sk = pytest.importorskip("sklearn.cluster")
    w = datagen.WORKLOADS["C2"]
    N = 20_000
    X = datagen.generate(w, N=N)
    init = datagen.one_per_blob_init(w, N=N)
    res = oracle.fit(X, w.M, init, tol=1e-6, max_iter=100)
    km = sk.KMeans(n_clusters=w.M, init=X[init].astype(np.float64), n_init=1,
                   algorithm="lloyd", tol=0.0, max_iter=300)
    km.fit(X.astype(np.float64))
    assert np.array_equal(km.labels_, res["labels"])
    np.testing.assert_allclose(res["centroids"], km.cluster_centers_, rtol=1e-6, atol=1e-9)
    # ground truth: one centroid per blob within sampling error of the blob centre
    np.testing.assert_allclose(res["centroids"], w.centers(), atol=0.1)


# ---------------------------------------------------------------------------
# Validation
# ---------------------------------------------------------------------------
def test_invalid_inputs_rejected():
    X = np.zeros((5, 2), np.float32)
    X[:, 0] = np.arange(5)
    with pytest.raises(oracle.OracleError):
        oracle.fit(X, 6, list(range(6)), 1e-6, 10)          # K > N
    with pytest.raises(oracle.OracleError):
        oracle.fit(X, 2, [1, 1], 1e-6, 10)                   # duplicate index
    with pytest.raises(oracle.OracleError):
        oracle.fit(X, 2, [0, 5], 1e-6, 10)                   # out of range
    with pytest.raises(oracle.OracleError):
        oracle.fit(X, 2, [0, 1], -1.0, 10)                   # tol < 0
    with pytest.raises(oracle.OracleError):
        oracle.fit(X, 2, [0, 1], float("nan"), 10)           # tol NaN
    with pytest.raises(oracle.OracleError):
        oracle.fit(X, 2, [0, 1], 1e-6, 0)                    # max_iter < 1
    Xn = X.copy()
    Xn[3, 1] = np.nan
    with pytest.raises(oracle.OracleError, match="non-finite"):
        oracle.fit(Xn, 2, [0, 1], 1e-6, 10)


def test_spec_chunk_partition(golden_dir):
    g = load(golden_dir, "spec_examples.json")["chunks"]
    sizes = [b - a for a, b in (datagen.shard_range(g["N"], g["p"], r) for r in range(g["p"]))]
    assert sizes == g["expect"]
