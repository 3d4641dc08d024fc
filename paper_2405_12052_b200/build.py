"""Builds libkmeans.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2405_12052_b200.build          # or __graft_entry__.build()

NCCL comes from the torch wheel (nvidia/nccl); the library is linked against
that libnccl.so.2 with an rpath, so it shares the communicator runtime torch
loads.  If the headers are missing the library is built without NCCL and the
multi-GPU calls return KMEANS_ENCCL.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libkmeans.so")
SOURCES = [os.path.join(HERE, "csrc", "runtime.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", "kernels.cuh"),
                  os.path.join(ROOT, "include", "kmeans.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def nccl_dirs():
    try:
        import nvidia.nccl  # noqa: F401  (torch's bundled NCCL)
        base = os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl, "__file__", None) \
            else list(nvidia.nccl.__path__)[0]
    except Exception:
        cands = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages",
                                       "nvidia", "nccl"))
        if not cands:
            return None
        base = cands[0]
    inc = os.path.join(base, "include")
    lib = os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and glob.glob(os.path.join(lib, "libnccl.so*")):
        return inc, lib
    return None


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile libkmeans.so (or a tuning variant `out` with -D `defines`)."""
    target = out or LIB
    if not force and out is None and not needs_build():
        return LIB
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
           "-shared", "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include")]
    nd = nccl_dirs()
    if nd:
        inc, lib = nd
        so = sorted(glob.glob(os.path.join(lib, "libnccl.so*")))[0]
        cmd += ["-DKMEANS_WITH_NCCL", "-I", inc, "-L", lib, f"-l:{os.path.basename(so)}",
                "-Xlinker", f"-rpath={lib}"]
    cmd += [f"-D{d}" for d in defines]
    tmp = target + f".tmp{os.getpid()}"
    cmd += ["-o", tmp, *SOURCES]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
