"""In-tree build of libppa_b200.so (CUDA sm_100a kernels + C++ host + C-ABI).

nvcc compiles the kernels for sm_100a only (-gencode arch=compute_100a,
code=sm_100a); g++ compiles the host C++; LAPACK comes from the OpenBLAS
bundled with scipy in this image (linked with an rpath, so the .so runs
unchanged on the GPU box, which has the same image).
"""
from __future__ import annotations

import glob
import importlib.util
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "ppa_b200")
LIB = os.path.join(PKG, "libppa_b200.so")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def find_lapack() -> str:
    """Path of the scipy-bundled OpenBLAS (exports scipy_dgeevx_ etc.)."""
    env = os.environ.get("PPA_LAPACK")
    if env and os.path.exists(env):
        return env
    spec = importlib.util.find_spec("scipy")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("scipy (for its bundled OpenBLAS/LAPACK) not found")
    site = os.path.dirname(list(spec.submodule_search_locations)[0])
    hits = sorted(glob.glob(os.path.join(site, "scipy.libs", "libscipy_openblas-*.so")))
    if not hits:
        raise RuntimeError("libscipy_openblas not found under scipy.libs")
    return hits[0]


def _headers() -> list[str]:
    out = []
    for pat in ("csrc/ppa/*.hpp", "csrc/kernels/*.cuh"):
        out += glob.glob(os.path.join(PKG, pat))
    out.append(os.path.join(INCLUDE, "ppa_b200.h"))
    return out


def _stale(obj: str, src: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src, *deps, __file__])


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {os.path.basename(cmd[-1])}")


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    deps = _headers()
    inc = ["-I", CSRC, "-I", INCLUDE]
    jobs = []
    objs = []
    for src in sorted(glob.glob(os.path.join(CSRC, "kernels", "*.cu"))):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if _stale(obj, src, deps):
            jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                         "-Xptxas", "-v" if verbose else "-O3", *inc, "-c", "-o", obj, src])
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cpp"))):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if _stale(obj, src, deps):
            jobs.append(["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall",
                         "-I", os.path.join(CUDA_HOME, "include"), *inc, "-c", "-o", obj, src])
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(_run, jobs))
    if jobs or not os.path.exists(LIB):
        lapack = find_lapack()
        tmp = LIB + ".tmp"
        _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs,
              "-Xlinker", f"-rpath,{os.path.dirname(lapack)}",
              lapack, "-lpthread"])
        shutil.move(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
