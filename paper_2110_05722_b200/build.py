"""Build the sm_100a C-ABI library libls2.so in-tree (nvcc, parallel, incremental).

    python -m paper_2110_05722_b200.build [-v] [--force]
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "lib", "obj")
LIB = os.path.join(PKG, "lib", "libls2.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _site_nvidia():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    if spec is None or not spec.submodule_search_locations:
        return None
    return list(spec.submodule_search_locations)[0]


def _flags():
    inc = ["-I", os.path.join(ROOT, "include")]
    nv = _site_nvidia()
    if nv:  # compile against the cuBLAS headers of the runtime torch ships
        inc += ["-I", os.path.join(nv, "cublas", "include")]
    return ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"] + inc


def _link_flags():
    rp = []
    nv = _site_nvidia()
    libdirs = []
    if nv:
        libdirs += [os.path.join(nv, "cublas", "lib"), os.path.join(nv, "cuda_runtime", "lib")]
    libdirs.append("/usr/local/cuda/lib64")
    for d in libdirs:
        rp += ["-Xlinker", "-rpath", "-Xlinker", d]
    ldirs = []
    for d in libdirs:
        ldirs += ["-L", d]
    # link the soname libcublas.so.12 explicitly (the pip wheel has no unversioned symlink)
    cublas = None
    for d in libdirs:
        for name in ("libcublas.so.12", "libcublas.so"):
            p = os.path.join(d, name)
            if os.path.exists(p):
                cublas = p
                break
        if cublas:
            break
    lib = ["-Xlinker", "-l:" + os.path.basename(cublas)] if cublas else ["-lcublas"]
    lib += ["-Xlinker", "-l:libcublasLt.so.12"]
    return rp + ldirs + lib + ["-ldl", "-cudart", "shared"]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps_mtime():
    paths = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    paths.append(os.path.join(ROOT, "include", "ls2.h"))
    return max(os.path.getmtime(p) for p in paths)


def build(verbose: bool = False, force: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    dep_t = _deps_mtime()
    flags = _flags()
    todo = []
    objs = []
    for src in _sources():
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src[:-3] + ".o")
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), dep_t):
            todo.append((s, o))

    def run(pair):
        s, o = pair
        cmd = [NVCC] + flags + ["-c", s, "-o", o]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{r.stdout}\n{r.stderr}")
        return s

    if todo:
        jobs = jobs or min(len(todo), os.cpu_count() or 4)
        with cf.ThreadPoolExecutor(jobs) as ex:
            for s in ex.map(run, todo):
                if verbose:
                    print("compiled", os.path.basename(s), flush=True)
    if todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + _link_flags()
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args(argv)
    print(build(verbose=a.verbose, force=a.force))


if __name__ == "__main__":
    sys.exit(main())
