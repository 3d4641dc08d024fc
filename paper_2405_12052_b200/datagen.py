"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no distance, argmin, mean or
error term): only the input recipe of DESIGN.md "Inputs", which stands in for
the paper's unpublished "mixture of Bivariate Gaussian Distributions of some
mean and covariance" datasets (§SERIAL LLOYD'S ALGORITHM) and the
"randomly selecting K points from the dataset" initialisation.

Generator (counter based, so any shard [start, start+count) is bit-identical
to the same slice of the full dataset, on any number of ranks):

  key        = mix64(seed)
  u64(i, s)  = mix64(key + (8*i + s + 1) * 0x9E3779B97F4A7C15)   (mod 2^64)
  U(i, s)    = (u64(i, s) >> 11) * 2^-53                           in [0, 1)
  blob_i     = floor(U(i, 0) * M)
  Box-Muller in fp64:  r = sqrt(-2 ln(1 - U(i,1))),  th = 2 pi U(i,2)
                       n0 = r cos th, n1 = r sin th
                       (d = 3: n2 = sqrt(-2 ln(1 - U(i,3))) cos(2 pi U(i,4)))
  x_ij       = fp32(center[blob_i][j] + sigma * n_j)     (one rounding)

mix64 is the SplitMix64 finaliser.  Blob centres sit on a regular grid with
spacing 10 sigma, centred at the origin.
"""
from __future__ import annotations

import dataclasses
import math
import os

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK = (1 << 64) - 1


def _mix64_np(z: np.ndarray) -> np.ndarray:
    z = z.copy()
    z ^= z >> np.uint64(30)
    z *= _M1
    z ^= z >> np.uint64(27)
    z *= _M2
    z ^= z >> np.uint64(31)
    return z


def mix64(z: int) -> int:
    """SplitMix64 finaliser on a Python int (mod 2^64)."""
    z &= _MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


def uniforms(seed: int, idx: np.ndarray, stream: int) -> np.ndarray:
    """U(i, s) in [0, 1) as float64 for every i in idx."""
    key = np.uint64(mix64(seed))
    with np.errstate(over="ignore"):
        ctr = idx.astype(np.uint64) * np.uint64(8) + np.uint64(stream + 1)
        z = key + ctr * GOLDEN
        u = _mix64_np(z)
    return (u >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def grid_centers(shape: tuple[int, ...], spacing: float = 10.0) -> np.ndarray:
    """M x d blob centres on a regular grid centred at the origin."""
    axes = [(np.arange(n, dtype=np.float64) - (n - 1) / 2.0) * spacing for n in shape]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.ravel() for m in mesh], axis=1)


@dataclasses.dataclass(frozen=True)
class Workload:
    """One configuration of BASELINE.json `configs` (or the north-star one)."""
    name: str
    N: int
    d: int
    K: int
    grid: tuple[int, ...]          # blob grid shape; M = prod(grid)
    data_seed: int
    init_seed: int
    tol: float = 1e-6
    max_iter: int = 100
    sigma: float = 1.0
    planted_sites: int = 0         # C5: outlier sites that force empty clusters
    planted_dups: int = 0

    @property
    def M(self) -> int:
        return int(np.prod(self.grid))

    def centers(self) -> np.ndarray:
        return grid_centers(self.grid, 10.0 * self.sigma)


WORKLOADS = {
    # BASELINE.json configs[0..4] and the north-star target.
    "C1": Workload("C1", 10_000, 2, 4, (2, 2), 1001, 2001),
    "C2": Workload("C2", 1_000_000, 3, 8, (2, 2, 2), 1002, 2002),
    "C3": Workload("C3", 100_000_000, 2, 16, (4, 4), 1003, 2003),
    "C4": Workload("C4", 1_000_000_000, 3, 16, (4, 2, 2), 1004, 2004),
    "C5": Workload("C5", 50_000_000, 3, 1024, (4, 4, 4), 1005, 2005,
                   planted_sites=8, planted_dups=8),
    "NS": Workload("NS", 100_000_000, 3, 16, (4, 2, 2), 1006, 2006),
}


def paper_grid() -> list[Workload]:
    """The paper's experiment grid as synthetic workloads:
    Table 1 (serial): 2D N = 5e5 and 3D N = 1e6 at K = 4, 8, 11;
    Tables 2/4: 2D N = 1e5, 2e5, 5e5 at K = 8;
    Tables 3/5: 3D N = 1e5 ... 1e6 at K = 4.
    The paper's mixtures are unpublished ("Bivariate Gaussian Distributions of
    some mean and covariance"): here 8 blobs on a 4 x 2 grid (2D)
    and 4 blobs on a 2 x 2 x 1 grid (3D), sigma = 1, spacing 10 sigma; the
    dataset of a given (d, N) is the same for every K (seed by d and N)."""
    out = []

    def wl(d, N, K):
        grid = (4, 2) if d == 2 else (2, 2, 1)
        seed = 1100 + 10 * d + int(round(math.log10(N) * 10))
        return Workload(f"P{d}D-N{N}-K{K}", N, d, K, grid, seed, seed + 1000,
                        tol=1e-6, max_iter=1000)
    for K in (4, 8, 11):
        out.append(wl(2, 500_000, K))
    for K in (4, 8, 11):
        out.append(wl(3, 1_000_000, K))
    for N in (100_000, 200_000):
        out.append(wl(2, N, 8))
    for N in (100_000, 200_000, 400_000, 800_000):
        out.append(wl(3, N, 4))
    return out


def mixture_spec(w: Workload, N: int | None = None) -> dict:
    """The parameters of this recipe for the on-device generator
    (kmeans_generate): seed, blob centres, sigma, planted sites."""
    N = w.N if N is None else N
    return {"seed": w.data_seed, "d": w.d, "M": w.M, "centers": w.centers(), "sigma": w.sigma,
            "n_sites": w.planted_sites, "site_dups": w.planted_dups,
            "sites": planted_site_coords(w) if w.planted_sites else None, "N": N}


def planted_indices(w: Workload, N: int | None = None) -> np.ndarray:
    """Indices of the planted duplicate points (C5): site g occupies
    [g * (N // G), g * (N // G) + r)."""
    N = w.N if N is None else N
    G, r = w.planted_sites, w.planted_dups
    if G == 0:
        return np.zeros(0, np.int64)
    stride = N // G
    return np.array([g * stride + q for g in range(G) for q in range(r)], np.int64)


def planted_site_coords(w: Workload) -> np.ndarray:
    """G x d outlier sites, >= 1000 sigma from the blob grid and from each other."""
    G = w.planted_sites
    out = np.zeros((G, w.d), np.float64)
    for g in range(G):
        out[g, 0] = 2000.0 + 1500.0 * g
        out[g, 1] = -1000.0
        if w.d > 2:
            out[g, 2] = 1000.0
    return out * w.sigma


def generate(w: Workload, start: int = 0, count: int | None = None, *,
             N: int | None = None, layout: str = "aos",
             chunk: int = 1 << 20, out: np.ndarray | None = None,
             threads: int | None = None) -> np.ndarray:
    """Points [start, start + count) of workload w (N overrides w.N for smaller
    parity cases).  layout 'aos' -> (count, d) float32; 'soa' -> (d, count).
    Chunks are generated on `threads` host threads (numpy releases the GIL);
    the result does not depend on the thread count."""
    N = w.N if N is None else N
    count = (N - start) if count is None else count
    assert 0 <= start and start + count <= N
    d = w.d
    centers = w.centers()
    if out is None:
        out = np.empty((count, d) if layout == "aos" else (d, count), np.float32)
    planted = planted_indices(w, N)
    sites = planted_site_coords(w) if w.planted_sites else None
    starts = list(range(0, count, chunk))
    if threads is None:
        threads = min(16, os.cpu_count() or 1)
    if threads > 1 and len(starts) > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda c0: _gen_chunk(w, N, start, c0, min(count, c0 + chunk), d,
                                              centers, planted, sites, layout, out), starts))
    else:
        for c0 in starts:
            _gen_chunk(w, N, start, c0, min(count, c0 + chunk), d, centers, planted, sites,
                       layout, out)
    return out


def _gen_chunk(w, N, start, c0, c1, d, centers, planted, sites, layout, out):
    """Fill rows [c0, c1) of `out` with points start+c0 .. start+c1-1."""
    idx = np.arange(start + c0, start + c1, dtype=np.int64)
    blob = np.minimum((uniforms(w.data_seed, idx, 0) * w.M).astype(np.int64), w.M - 1)
    u1 = uniforms(w.data_seed, idx, 1)
    u2 = uniforms(w.data_seed, idx, 2)
    r = np.sqrt(-2.0 * np.log1p(-u1))
    th = 2.0 * math.pi * u2
    cols = [r * np.cos(th), r * np.sin(th)]
    if d > 2:
        u3 = uniforms(w.data_seed, idx, 3)
        u4 = uniforms(w.data_seed, idx, 4)
        cols.append(np.sqrt(-2.0 * np.log1p(-u3)) * np.cos(2.0 * math.pi * u4))
    for j in range(d):
        v = (centers[blob, j] + w.sigma * cols[j]).astype(np.float32)
        if layout == "aos":
            out[c0:c1, j] = v
        else:
            out[j, c0:c1] = v
    if sites is not None:
        sel = (planted >= start + c0) & (planted < start + c1)
        for p in planted[sel]:
            g = int(np.searchsorted(planted, p, side="right") - 1) // w.planted_dups
            for j in range(d):
                if layout == "aos":
                    out[p - start, j] = np.float32(sites[g, j])
                else:
                    out[j, p - start] = np.float32(sites[g, j])


class SplitMix64:
    """Sequential SplitMix64 (state += golden; return mix64(state))."""

    def __init__(self, seed: int):
        self.state = seed & _MASK

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK
        return mix64(self.state)


def floyd_sample(N: int, K: int, seed: int, exclude=()) -> np.ndarray:
    """K distinct indices in [0, N) by Floyd's algorithm over SplitMix64(seed),
    in insertion order (reading R8: the paper's 'randomly selecting K points',
    PAPER.md:44, made explicit and seeded).  Indices in `exclude` are never
    returned (the pool shrinks by skipping them)."""
    if K > N - len(exclude):
        raise ValueError("K larger than the pool")
    rng = SplitMix64(seed)
    excl = sorted(set(int(e) for e in exclude))
    pool = N - len(excl)

    def to_index(t):  # t-th index of [0, N) \ exclude
        for e in excl:
            if e <= t:
                t += 1
            else:
                break
        return t

    chosen: list[int] = []
    seen: set[int] = set()
    for j in range(pool - K, pool):
        t = rng.next() % (j + 1)
        if t in seen:
            t = j
        seen.add(t)
        chosen.append(t)
    return np.array([to_index(t) for t in chosen], np.int64)


def init_indices(w: Workload, N: int | None = None, K: int | None = None) -> np.ndarray:
    """init_idx for workload w: K distinct seeded indices; for planted workloads
    (C5) the planted duplicates come first (so per site the lowest-k centroid
    takes the duplicates and the other r-1 stay empty every iteration)."""
    N = w.N if N is None else N
    K = w.K if K is None else K
    planted = planted_indices(w, N)
    if len(planted) == 0:
        return floyd_sample(N, K, w.init_seed)
    rest = floyd_sample(N, K - len(planted), w.init_seed, exclude=planted)
    return np.concatenate([planted, rest])


def blob_of(w: Workload, idx: np.ndarray) -> np.ndarray:
    """Ground-truth blob index of points idx (for one-init-per-blob runs)."""
    idx = np.asarray(idx, np.int64)
    return np.minimum((uniforms(w.data_seed, idx, 0) * w.M).astype(np.int64), w.M - 1)


def one_per_blob_init(w: Workload, N: int | None = None) -> np.ndarray:
    """K = M indices, the lowest-index point of each blob, ordered by blob.
    Used for full-run parity on well-separated blobs."""
    N = w.N if N is None else N
    found = {}
    step = 4096
    for s in range(0, N, step):
        idx = np.arange(s, min(N, s + step), dtype=np.int64)
        b = blob_of(w, idx)
        for i, bi in zip(idx, b):
            if int(bi) not in found:
                found[int(bi)] = int(i)
        if len(found) == w.M:
            break
    if len(found) < w.M:
        raise ValueError("some blob has no point")
    return np.array([found[m] for m in range(w.M)], np.int64)


def shard_range(N: int, P: int, r: int) -> tuple[int, int]:
    """Contiguous ceiling partition: rank r owns [r*ceil(N/P), min((r+1)*ceil(N/P), N))
    ('dataset is to be divided among the number of threads' PAPER.md:97)."""
    c = -(-N // P)
    a = min(N, r * c)
    b = min(N, (r + 1) * c)
    return a, b
