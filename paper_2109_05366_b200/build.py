"""Build libgfs.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2109_05366_b200.build [--force]

Output: paper_2109_05366_b200/_lib/libgfs.so (git-ignored, travels to the GPU box
with the repo snapshot).  Flags: -gencode arch=compute_100a,code=sm_100a -lineinfo -O3.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libgfs.so")
SOURCES = [os.path.join(CSRC, "gfs_host.cpp"), os.path.join(CSRC, "gfs_baseline.cpp"),
           os.path.join(CSRC, "gfs_kernels.cu")]
HEADERS = [os.path.join(CSRC, "gfs_shared.h"), os.path.join(CSRC, "gfs_device_impl.cuh"),
           os.path.join(ROOT, "include", "gfs.h"), os.path.join(ROOT, "include", "gfs_device.cuh")]
# A user kernel built the way an application would: only include/ headers + libgfs.so.
USER_LIB = os.path.join(OUT_DIR, "libgfs_user.so")
USER_SOURCES = [os.path.join(CSRC, "user_gemv.cu")]
GENCODE = "arch=compute_100a,code=sm_100a"


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def stale(lib: str = LIB, sources=None) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(p) > t for p in (sources or SOURCES) + HEADERS)


def _nvcc(out: str, sources, extra, verbose: bool) -> None:
    tmp = out + ".tmp"
    cmd = [nvcc(), "-O3", "-std=c++17", "-gencode", GENCODE, "-lineinfo",
           "-Xcompiler", "-fPIC,-Wall", "-shared",
           "-I" + os.path.join(ROOT, "include"), "-I" + CSRC,
           "-o", tmp, *sources, *extra]
    if verbose:
        cmd.append("-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-4000:]}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, out)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    if force or stale():
        _nvcc(LIB, SOURCES, ["-lpthread"], verbose)
    if force or stale(USER_LIB, USER_SOURCES) or os.path.getmtime(LIB) > os.path.getmtime(USER_LIB):
        _nvcc(USER_LIB, USER_SOURCES, ["-L" + OUT_DIR, "-lgfs", "-Xlinker", "-rpath,$ORIGIN"], verbose)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
