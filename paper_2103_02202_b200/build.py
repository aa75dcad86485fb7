"""Build libpfs.so (sm_100a) in-tree with nvcc.

    python -m paper_2103_02202_b200.build [--verbose]

The shared library lands in paper_2103_02202_b200/_lib/libpfs.so so it travels
with the repo snapshot to the GPU box (a JIT cache would not).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIB_DIR, "libpfs.so")
PROFILE_LIB = os.path.join(LIB_DIR, "libpfs_profile.so")  # PFS_PROFILE=1: traces, ablations
SOURCES = ["pfs_compile.cpp", "pfs_tableau.cpp", "pfs_dem.cpp", "pfs_kernels.cu", "pfs_demkernel.cu", "pfs_writers.cu", "pfs_api.cu"]
HEADERS = ["pfs_internal.h", "pfs_device.cuh", os.path.join("..", "..", "include", "pfs.h")]
INCLUDE = os.path.join(os.path.dirname(PKG), "include")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(lib=LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    for f in SOURCES + HEADERS:
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    return False


def build(force: bool = False, verbose: bool = False, profile: bool = False,
          out: str | None = None, csrc: str = CSRC, defines: tuple = ()) -> str:
    """out/csrc/defines: experimental builds for A/B timing (tools only)."""
    lib = out or (PROFILE_LIB if profile else LIB)
    if not force and out is None and not _stale(lib):
        return lib
    os.makedirs(LIB_DIR, exist_ok=True)
    tmp = lib + ".tmp"
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "--threads", "0",
           "-Xcompiler", "-fPIC,-O3,-fopenmp", "-shared", "-I", INCLUDE, "-o", tmp]
    if profile:
        cmd += ["-DPFS_PROFILE=1"]
    cmd += [f"-D{d}" for d in defines]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += [os.path.join(csrc, f) for f in SOURCES]
    cmd += ["-lcudart", "-lgomp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--out", default=None, help="experimental build path (load with PFS_LIB=)")
    ap.add_argument("--csrc", default=CSRC)
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    print(build(force=True, verbose=a.verbose, profile=a.profile, out=a.out, csrc=a.csrc,
                defines=tuple(a.defines)))
