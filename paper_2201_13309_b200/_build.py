"""Build the CUDA library libdaxm.so in-tree for sm_100a (nvcc, no torch JIT)."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libdaxm.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build_library(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build libdaxm.so (or a variant at `out` with extra -D `defines`, for experiments)."""
    target = out or LIB
    if not force and out is None and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = target + f".tmp{os.getpid()}"
    # one object per source, compiled in parallel (no relocatable device code: every kernel is
    # launched from its own translation unit), then linked into the shared library
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    objs, procs = [], []
    for src in sources():
        obj = f"{tmp}.{os.path.basename(src)}.o"
        cmd = [nvcc, *flags, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        objs.append(obj)
        procs.append((src, subprocess.Popen(cmd)))
    failed = [src for src, pr in procs if pr.wait() != 0]
    try:
        if failed:
            raise subprocess.CalledProcessError(1, f"nvcc {failed}")
        subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                               "-o", tmp, *objs])
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build_library(force=True, verbose=True))
