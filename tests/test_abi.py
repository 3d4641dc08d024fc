"""The C-ABI library loads, exports every symbol include/kmeans.h declares, and
rejects invalid arguments before any device work (so these run without a GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2405_12052_b200 import build as kbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def km():
    kbuild.build()
    from paper_2405_12052_b200 import kmeans
    kmeans.lib()
    return kmeans


def header_functions():
    src = open(os.path.join(ROOT, "include", "kmeans.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(kmeans_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_header_declares_the_north_star_calls():
    names = header_functions()
    for n in ["kmeans_create", "kmeans_assign", "kmeans_update", "kmeans_fit", "kmeans_destroy"]:
        assert n in names


def test_every_declared_symbol_is_exported(km):
    L = km.lib()
    names = header_functions()
    assert names, "no declarations parsed"
    for n in names:
        assert hasattr(L, n), f"{n} declared in kmeans.h but not exported"
    # the binding's signature table covers exactly the header
    assert sorted(km.SIGNATURES) == names


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2405_12052_b200", "libkmeans.so")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_status_strings_and_version(km):
    L = km.lib()
    assert L.kmeans_abi_version() == 3 == km.ABI_VERSION
    for code, name in km.STATUS.items():
        assert L.kmeans_status_string(code).decode().startswith(name)


def test_invalid_arguments_rejected_before_device_work(km):
    L = km.lib()
    h = ctypes.c_void_p()
    pts = np.zeros((10, 3), np.float32)
    p = ctypes.c_void_p(pts.ctypes.data)
    assert L.kmeans_create(ctypes.byref(h), p, 0, 3, 2, None) == -1        # N < 1
    assert L.kmeans_create(ctypes.byref(h), p, 10, 4, 2, None) == -1       # d not in {2,3}
    assert L.kmeans_create(ctypes.byref(h), p, 10, 1, 2, None) == -1
    assert L.kmeans_create(ctypes.byref(h), p, 10, 3, 0, None) == -1       # K < 1
    assert L.kmeans_create(ctypes.byref(h), p, 10, 3, 11, None) == -1      # K > N
    assert L.kmeans_create(ctypes.byref(h), None, 10, 3, 2, None) == -1    # NULL points
    big = np.zeros((2000, 3), np.float32)
    assert L.kmeans_create(ctypes.byref(h), ctypes.c_void_p(big.ctypes.data), 2000, 3,
                           km.MAX_K + 1, None) == -1                       # K > KMEANS_MAX_K
    # distributed shard outside global_N
    o = km.Opts()
    L.kmeans_opts_init(ctypes.byref(o))
    o.global_N = 15
    o.global_offset = 10
    assert L.kmeans_create(ctypes.byref(h), p, 10, 3, 2, ctypes.byref(o)) == -1
    assert not h.value
    idx = np.array([0, 1], np.int64)
    out = np.zeros((2, 3))
    it = ctypes.c_int()
    j = ctypes.c_double()
    ip = ctypes.c_void_p(idx.ctypes.data)
    op = ctypes.c_void_p(out.ctypes.data)
    assert L.kmeans_fit(p, 10, 3, 2, ip, -1.0, 5, None, op, ctypes.byref(it), ctypes.byref(j)) == -1
    assert L.kmeans_fit(p, 10, 3, 2, ip, float("nan"), 5, None, op, ctypes.byref(it),
                        ctypes.byref(j)) == -1
    assert L.kmeans_fit(p, 10, 3, 2, ip, 1e-6, 0, None, op, ctypes.byref(it), ctypes.byref(j)) == -1
    assert L.kmeans_fit(p, 10, 3, 2, None, 1e-6, 5, None, op, ctypes.byref(it), ctypes.byref(j)) == -1
    # NULL context
    assert L.kmeans_iterate(None, 1) == -1
    assert L.kmeans_update(None, None, None) == -1
    assert L.kmeans_profile_stage(None, 1, 1, None) == -1
    assert L.kmeans_p2p_handle(None, None) == -1
    assert L.kmeans_p2p_open(None, None) == -1
    assert L.kmeans_p2p_disable(None) == -1
    assert L.kmeans_p2p_loopback(None, 1, 1, None, None) == -1
    assert L.kmeans_p2p_selftest(0, 0, 5, 1, None, None, -1, 0.0, None) == -1     # P < 1
    assert L.kmeans_p2p_selftest(0, 65, 5, 1, None, None, -1, 0.0, None) == -1    # P > 64
    v = np.zeros((1, 2, 5))
    vp = ctypes.c_void_p(v.ctypes.data)
    assert L.kmeans_p2p_selftest(0, 2, 5, 1, vp, vp, 2, 0.0, None) == -1   # dead_rank >= P
    assert L.kmeans_p2p_selftest(0, 2, 5, 1, vp, vp, -1, -1.0, None) == -1  # timeout < 0
    # P2P-only group: rank outside [0, nranks), negative hints
    o2 = km.Opts()
    L.kmeans_opts_init(ctypes.byref(o2))
    assert o2.nranks == 0 and o2.rank == 0 and o2.expected_iters == 0 and o2.comm_timeout_s == 0.0
    o2.nranks, o2.rank = 2, 2
    assert L.kmeans_create(ctypes.byref(h), p, 10, 3, 2, ctypes.byref(o2)) == -1
    o2.nranks, o2.rank, o2.expected_iters = 2, 0, -1
    assert L.kmeans_create(ctypes.byref(h), p, 10, 3, 2, ctypes.byref(o2)) == -1
    o2.expected_iters, o2.comm_timeout_s = 0, float("nan")
    assert L.kmeans_create(ctypes.byref(h), p, 10, 3, 2, ctypes.byref(o2)) == -1
    assert L.kmeans_release_memory(-1) == -1
    assert L.kmeans_generate(None, 0, 1, None, 0, None) == -1
    L.kmeans_destroy(None)  # NULL-safe
    assert L.kmeans_last_error()  # a message was recorded


def test_binding_validates_shapes_and_dtypes(km):
    """Python-side validation raises ValueError / TypeError (not assert, which
    python -O strips) before any library call."""
    with pytest.raises(ValueError):
        km.Context(np.zeros(6, np.float32), K=2)            # 1-D AoS without d
    with pytest.raises(ValueError):
        km.Context(np.zeros(7, np.float32), K=2, d=3)       # not a multiple of d
    with pytest.raises(ValueError):
        km.Context(np.zeros((4, 3), np.float32), K=2, d=2)  # d contradicts the shape
    with pytest.raises(ValueError):
        km.Context(np.zeros((4, 3), np.float32), K=2, layout="xyz")
    with pytest.raises(ValueError):
        km._ptr(np.zeros((4, 6))[:, ::2])                    # not contiguous
    torch = pytest.importorskip("torch")
    with pytest.raises(TypeError):
        km._as_f64(torch.zeros(3, dtype=torch.float32))
    with pytest.raises(ValueError):
        km.comm_init(2, b"short", 0, 0)


def test_binding_raises_typed_error(km):
    with pytest.raises(km.KMeansError) as ei:
        km.Context(np.zeros((3, 5), np.float32), K=2, d=5)
    assert ei.value.name == "KMEANS_EINVAL"
