"""Thin ctypes binding of libkmeans.so (include/kmeans.h) -- argument
marshalling only; every step of the Lloyd iteration runs in the library's
sm_100a kernels.  There is no CPU fallback: if the library is missing or the
GPU is absent the calls raise.

Arrays may be numpy arrays (host) or torch tensors (host or CUDA); pointers
are passed straight through (the library resolves host vs device memory).
Outputs are numpy arrays unless a preallocated torch tensor is passed.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KMEANS_LIB_OVERRIDE") or os.path.join(HERE, "libkmeans.so")

KMEANS_OK = 0
ABI_VERSION = 3   # include/kmeans.h KMEANS_ABI_VERSION
STATUS = {0: "KMEANS_OK", -1: "KMEANS_EINVAL", -2: "KMEANS_ENONFINITE", -3: "KMEANS_ENOMEM",
          -4: "KMEANS_ECUDA", -5: "KMEANS_ENCCL", -6: "KMEANS_ESTATE"}
LAYOUT_AOS, LAYOUT_SOA = 0, 1
FLAG_NO_SORT = 1
FLAG_FORCE_SORT = 2
FLAG_NO_FUSED = 4
FLAG_BIG_CHUNKS = 8
FLAG_PERSIST = 16
MAX_K = 1024


class KMeansError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{where}: {self.name}: {msg}")


class Opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("layout", ctypes.c_int),
                ("nccl_comm", ctypes.c_void_p), ("global_offset", ctypes.c_int64),
                ("global_N", ctypes.c_int64), ("flags", ctypes.c_int), ("rank", ctypes.c_int),
                ("nranks", ctypes.c_int), ("expected_iters", ctypes.c_int),
                ("comm_timeout_s", ctypes.c_double)]


class Info(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("global_N", ctypes.c_int64),
                ("global_offset", ctypes.c_int64), ("ldx", ctypes.c_int64),
                ("d", ctypes.c_int), ("K", ctypes.c_int), ("grid", ctypes.c_int),
                ("block", ctypes.c_int), ("smem_bytes", ctypes.c_int), ("path", ctypes.c_int),
                ("kernels_per_iter", ctypes.c_int), ("kernel_launches", ctypes.c_int64),
                ("nranks", ctypes.c_int), ("rank", ctypes.c_int), ("sorted", ctypes.c_int),
                ("fused", ctypes.c_int), ("fused_grid", ctypes.c_int),
                ("persistent", ctypes.c_int), ("persist_grid", ctypes.c_int)]


class Mixture(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("d", ctypes.c_int), ("M", ctypes.c_int),
                ("centers", ctypes.c_void_p), ("sigma", ctypes.c_double),
                ("n_sites", ctypes.c_int), ("site_dups", ctypes.c_int),
                ("sites", ctypes.c_void_p), ("N", ctypes.c_int64)]


# Every exported symbol with (restype, argtypes); tests check the header matches.
P, I, I64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
SIGNATURES = {
    "kmeans_opts_init": (None, [P]),
    "kmeans_create": (I, [P, P, I64, I, I, P]),
    "kmeans_assign": (I, [P, P, P, P, P, P]),
    "kmeans_update": (I, [P, P, P]),
    "kmeans_fit": (I, [P, I64, I, I, P, D, I, P, P, P, P]),
    "kmeans_fit_ctx": (I, [P, P, D, I, P, P, P, P, P, P]),
    "kmeans_start": (I, [P, P, P, D, I]),
    "kmeans_iterate": (I, [P, I]),
    "kmeans_poll": (I, [P, P, P, P, P]),
    "kmeans_read_centroids": (I, [P, P]),
    "kmeans_final_labels": (I, [P, P]),
    "kmeans_profile_assign": (I, [P, I]),
    "kmeans_profile_stage": (I, [P, I, I, P]),
    "kmeans_candidate_stats": (I, [P, P, P, P, P]),
    "kmeans_get_stream": (I, [P, P]),
    "kmeans_get_info": (I, [P, P]),
    "kmeans_comm_unique_id": (I, [P]),
    "kmeans_comm_init": (I, [P, I, P, I, I]),
    "kmeans_comm_destroy": (I, [P]),
    "kmeans_destroy": (None, [P]),
    "kmeans_status_string": (ctypes.c_char_p, [I]),
    "kmeans_last_error": (ctypes.c_char_p, []),
    "kmeans_abi_version": (I, []),
    "kmeans_release_memory": (I, [I]),
    "kmeans_generate": (I, [P, I64, I64, P, I, P]),
    "kmeans_p2p_handle": (I, [P, P]),
    "kmeans_p2p_open": (I, [P, P]),
    "kmeans_p2p_disable": (I, [P]),
    "kmeans_p2p_selftest": (I, [I, I, I, I, P, P, I, D, P]),
    "kmeans_p2p_loopback": (I, [P, I, I, P, P]),
}

_lib = None


def lib():
    """Load libkmeans.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() "
                              "or python -m paper_2405_12052_b200.build")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.kmeans_abi_version() != ABI_VERSION:   # the Info / Opts layouts below
            raise ImportError(f"{LIB_PATH}: ABI {L.kmeans_abi_version()}, binding expects "
                              f"{ABI_VERSION}; rebuild the library")
        _lib = L
    return _lib


def _check(rc: int, where: str):
    if rc != KMEANS_OK:
        raise KMeansError(rc, where, lib().kmeans_last_error().decode(errors="replace"))


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _ptr(a):
    """Address of a numpy array / torch tensor (contiguous), or None."""
    if a is None:
        return None
    if _is_torch(a):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(a.data_ptr())
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return ctypes.c_void_p(a.ctypes.data)


def _torch_checked(a, dtype_name: str):
    import torch
    want = getattr(torch, dtype_name)
    if a.dtype != want:
        raise TypeError(f"tensor must be {dtype_name}, got {a.dtype}")
    if not a.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return a


def _as_f32_points(points):
    if _is_torch(points):
        return _torch_checked(points, "float32")
    return np.ascontiguousarray(points, dtype=np.float32)


def _as_f64(a):
    if _is_torch(a):
        return _torch_checked(a, "float64")
    return np.ascontiguousarray(a, dtype=np.float64)


def _as_i64(a):
    if _is_torch(a):
        return _torch_checked(a, "int64")
    return np.ascontiguousarray(a, dtype=np.int64)


class Context:
    """One GPU's shard of the points plus the Lloyd iteration state
    (kmeans_create ... kmeans_destroy)."""

    def __init__(self, points, K: int, *, d: int | None = None, layout: str = "aos",
                 device: int = -1, stream=None, comm=None, global_offset: int = 0,
                 global_N: int = 0, sort: bool | None = None, fused: bool = True,
                 big_chunks: bool = False, persist: bool = False, rank: int = 0, nranks: int = 0,
                 expected_iters: int = 0, comm_timeout_s: float = 0.0):
        pts = _as_f32_points(points)
        shape = tuple(pts.shape)
        if layout not in ("aos", "soa"):
            raise ValueError(f"layout must be 'aos' or 'soa', got {layout!r}")
        if layout == "aos":
            if len(shape) == 2:
                N, dd = shape
            elif len(shape) == 1:
                if d is None:
                    raise ValueError("1-D AoS points need d (points are N*d floats)")
                if shape[0] % d:
                    raise ValueError(f"{shape[0]} floats is not a multiple of d={d}")
                N, dd = shape[0] // d, d
            else:
                raise ValueError(f"AoS points must be N x d (or flat with d), got shape {shape}")
        else:
            if len(shape) != 2:
                raise ValueError(f"SoA points must be d x N, got shape {shape}")
            dd, N = shape
        if d is not None and int(d) != int(dd):
            raise ValueError(f"d={d} does not match the points' shape {shape}")
        self.N, self.d, self.K = int(N), int(dd), int(K)
        o = Opts()
        lib().kmeans_opts_init(ctypes.byref(o))
        o.device = device
        o.stream = stream
        o.layout = LAYOUT_AOS if layout == "aos" else LAYOUT_SOA
        o.nccl_comm = comm
        o.global_offset = global_offset
        o.global_N = global_N
        # sort: None = the library's choice, True = sorted (pruned) path, False = full scan
        o.flags = 0 if sort is None else (FLAG_FORCE_SORT if sort else FLAG_NO_SORT)
        if not fused:   # full-scan path: one graph launch per iteration instead of k_fused_iterate
            o.flags |= FLAG_NO_FUSED
        if big_chunks:  # sorted path: 2048-point chunks regardless of N
            o.flags |= FLAG_BIG_CHUNKS
        if persist:  # sorted path: k_persist_iterate instead of the per-iteration kernel graph
            o.flags |= FLAG_PERSIST
        o.rank = rank                   # P2P-only group (no NCCL communicator)
        o.nranks = nranks
        o.expected_iters = expected_iters
        o.comm_timeout_s = comm_timeout_s
        h = ctypes.c_void_p()
        _check(lib().kmeans_create(ctypes.byref(h), _ptr(pts), self.N, self.d, self.K,
                                   ctypes.byref(o)), "kmeans_create")
        self._h = h
        self.global_N = global_N or self.N
        self.global_offset = global_offset

    # -- lifetime ------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().kmeans_destroy(self._h)
            self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- per-step API ----------------------------------------------------------
    def assign(self, centroids, *, labels=True, out_labels=None):
        """One reassignment + fused reduction at mu^t.
        Returns dict(labels, inertia, counts, sums)."""
        c = _as_f64(centroids)
        lab = out_labels if out_labels is not None else (
            np.empty(self.N, np.int32) if labels else None)
        inertia = ctypes.c_double()
        counts = np.empty(self.K, np.int64)
        sums = np.empty((self.K, self.d), np.float64)
        _check(lib().kmeans_assign(self._h, _ptr(c), _ptr(lab), ctypes.byref(inertia),
                                   _ptr(counts), _ptr(sums)), "kmeans_assign")
        return dict(labels=lab, inertia=inertia.value, counts=counts, sums=sums)

    def update(self):
        """mu^{t+1} and E after assign."""
        mu = np.empty((self.K, self.d), np.float64)
        E = ctypes.c_double()
        _check(lib().kmeans_update(self._h, _ptr(mu), ctypes.byref(E)), "kmeans_update")
        return mu, E.value

    # -- whole run -------------------------------------------------------------
    def fit(self, init_idx, tol: float, max_iter: int, *, labels=True, out_labels=None,
            traces=True):
        idx = _as_i64(init_idx)
        lab = out_labels if out_labels is not None else (
            np.empty(self.N, np.int32) if labels else None)
        cent = np.empty((self.K, self.d), np.float64)
        iters = ctypes.c_int()
        inertia = ctypes.c_double()
        Et = np.zeros(max_iter, np.float64) if traces else None
        Jt = np.zeros(max_iter, np.float64) if traces else None
        _check(lib().kmeans_fit_ctx(self._h, _ptr(idx), float(tol), int(max_iter), _ptr(lab),
                                    _ptr(cent), ctypes.byref(iters), ctypes.byref(inertia),
                                    _ptr(Et), _ptr(Jt)), "kmeans_fit_ctx")
        T = iters.value
        return dict(labels=lab, centroids=cent, iters=T, inertia=inertia.value,
                    E_trace=Et[:T] if traces else None, J_trace=Jt[:T] if traces else None)

    # -- device-resident loop ------------------------------------------------------
    def start(self, init_idx=None, centroids=None, tol: float = 0.0, max_iter: int = 1 << 30):
        _check(lib().kmeans_start(self._h, _ptr(None if init_idx is None else _as_i64(init_idx)),
                                  _ptr(None if centroids is None else _as_f64(centroids)),
                                  float(tol), int(max_iter)), "kmeans_start")

    def iterate(self, n: int):
        _check(lib().kmeans_iterate(self._h, int(n)), "kmeans_iterate")

    def poll(self):
        it, done, E, J = ctypes.c_int(), ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
        _check(lib().kmeans_poll(self._h, ctypes.byref(it), ctypes.byref(done), ctypes.byref(E),
                                 ctypes.byref(J)), "kmeans_poll")
        return dict(iters=it.value, done=bool(done.value), E=E.value, J=J.value)

    def read_centroids(self, out=None):
        out = np.empty((self.K, self.d), np.float64) if out is None else out
        _check(lib().kmeans_read_centroids(self._h, _ptr(out)), "kmeans_read_centroids")
        return out

    def final_labels(self, out=None):
        out = np.empty(self.N, np.int32) if out is None else out
        _check(lib().kmeans_final_labels(self._h, _ptr(out)), "kmeans_final_labels")
        return out

    def profile_assign(self, n: int):
        """Enqueue n assignment passes (assign kernels + chunk-row merge; no state change)."""
        _check(lib().kmeans_profile_assign(self._h, int(n)), "kmeans_profile_assign")

    def profile_stage(self, n: int, stage: int, timed: bool = False):
        """n launches of one iteration stage (see kmeans_profile_stage).  timed:
        run them as one CUDA graph between two events and return ms per launch;
        else enqueue them and return None."""
        if not timed:
            _check(lib().kmeans_profile_stage(self._h, int(n), int(stage), None),
                   "kmeans_profile_stage")
            return None
        ms = ctypes.c_float()
        _check(lib().kmeans_profile_stage(self._h, int(n), int(stage), ctypes.byref(ms)),
               "kmeans_profile_stage")
        return ms.value

    def p2p_handle(self) -> bytes:
        """This rank's exchange-buffer IPC handle (kmeans_p2p_handle, 64 bytes)."""
        buf = (ctypes.c_ubyte * 64)()
        _check(lib().kmeans_p2p_handle(self._h, buf), "kmeans_p2p_handle")
        return bytes(buf)

    def p2p_open(self, handles):
        """Map every rank's exchange buffer (kmeans_p2p_open); handles in rank order."""
        blob = b"".join(handles)
        buf = (ctypes.c_ubyte * len(blob)).from_buffer_copy(blob)
        _check(lib().kmeans_p2p_open(self._h, buf), "kmeans_p2p_open")

    def p2p_loopback(self, vals):
        """kmeans_p2p_loopback: every rank of the opened group emulated on this
        GPU over the real (IPC-mapped) buffers; vals (rounds, nranks, n)."""
        v = np.ascontiguousarray(vals, dtype=np.float64)
        rounds, P, n = v.shape
        out = np.empty_like(v)
        _check(lib().kmeans_p2p_loopback(self._h, int(rounds), int(n), _ptr(v), _ptr(out)),
               "kmeans_p2p_loopback")
        return out

    def p2p_disable(self):
        """Back to the NCCL allreduce (kmeans_p2p_disable)."""
        _check(lib().kmeans_p2p_disable(self._h), "kmeans_p2p_disable")

    def candidate_stats(self) -> dict:
        """Sorted path: centroid candidates per chunk in the last assign pass."""
        m, mx, one, nch = ctypes.c_double(), ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().kmeans_candidate_stats(self._h, ctypes.byref(m), ctypes.byref(mx),
                                            ctypes.byref(one), ctypes.byref(nch)),
               "kmeans_candidate_stats")
        return dict(mean=m.value, max=mx.value, single_frac=one.value / max(nch.value, 1),
                    chunks=nch.value)

    @property
    def stream(self) -> int:
        s = ctypes.c_void_p()
        _check(lib().kmeans_get_stream(self._h, ctypes.byref(s)), "kmeans_get_stream")
        return s.value or 0

    def info(self) -> dict:
        i = Info()
        _check(lib().kmeans_get_info(self._h, ctypes.byref(i)), "kmeans_get_info")
        return {f: getattr(i, f) for f, _ in Info._fields_}


def fit(points, K: int, init_idx, tol: float, max_iter: int, *, labels=True):
    """kmeans_fit: the whole Lloyd run on one GPU, points N x d."""
    pts = _as_f32_points(points)
    if len(pts.shape) != 2:
        raise ValueError(f"points must be N x d, got shape {tuple(pts.shape)}")
    N, d = int(pts.shape[0]), int(pts.shape[1])
    idx = _as_i64(init_idx)
    lab = np.empty(N, np.int32) if labels else None
    cent = np.empty((K, d), np.float64)
    iters = ctypes.c_int()
    inertia = ctypes.c_double()
    _check(lib().kmeans_fit(_ptr(pts), N, d, int(K), _ptr(idx), float(tol), int(max_iter),
                            _ptr(lab), _ptr(cent), ctypes.byref(iters), ctypes.byref(inertia)),
           "kmeans_fit")
    return dict(labels=lab, centroids=cent, iters=iters.value, inertia=inertia.value)


# -- multi-GPU plumbing -----------------------------------------------------------
def comm_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _check(lib().kmeans_comm_unique_id(buf), "kmeans_comm_unique_id")
    return bytes(buf)


def comm_init(nranks: int, uid: bytes, rank: int, device: int) -> int:
    if len(uid) != 128:
        raise ValueError("an NCCL unique id is 128 bytes")
    buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
    c = ctypes.c_void_p()
    _check(lib().kmeans_comm_init(ctypes.byref(c), int(nranks), buf, int(rank), int(device)),
           "kmeans_comm_init")
    return c.value


def comm_destroy(comm: int):
    _check(lib().kmeans_comm_destroy(ctypes.c_void_p(comm)), "kmeans_comm_destroy")


def release_memory(device: int = 0):
    """Give the library pool's unused device memory back to the driver."""
    _check(lib().kmeans_release_memory(int(device)), "kmeans_release_memory")


def p2p_selftest(vals, device: int = 0, dead_rank: int = -1, timeout_s: float = 0.0,
                 failed=None):
    """kmeans_p2p_selftest: vals (rounds, P, n) float64 -> what each emulated
    rank computed, same shape.  dead_rank never publishes; `failed` (P int32,
    optional) receives each rank's failed round (1-based, 0 = none)."""
    v = np.ascontiguousarray(vals, dtype=np.float64)
    rounds, P, n = v.shape
    out = np.empty_like(v)
    f = failed if failed is not None else np.zeros(P, np.int32)
    _check(lib().kmeans_p2p_selftest(int(device), int(P), int(n), int(rounds), _ptr(v), _ptr(out),
                                     int(dead_rank), float(timeout_s), _ptr(f)),
           "kmeans_p2p_selftest")
    return out


def generate(spec: dict, start: int, count: int, out, device: int = 0, stream=None):
    """kmeans_generate: points [start, start + count) of the mixture `spec`
    (datagen.mixture_spec) into the device tensor `out` (count x d, float32)."""
    centers = np.ascontiguousarray(spec["centers"], np.float64)
    sites = np.ascontiguousarray(spec["sites"], np.float64) if spec["n_sites"] else None
    m = Mixture(spec["seed"], spec["d"], spec["M"], centers.ctypes.data, spec["sigma"],
                spec["n_sites"], spec["site_dups"], None if sites is None else sites.ctypes.data,
                spec["N"])
    _check(lib().kmeans_generate(ctypes.byref(m), int(start), int(count), _ptr(out), int(device),
                                 stream), "kmeans_generate")
    return out
