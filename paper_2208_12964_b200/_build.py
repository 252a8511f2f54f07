"""In-tree build of libuscg_b200.so for sm_100a (nvcc; no JIT cache).

The library is the product: the C ABI in include/uscg_b200.h over the CUDA
kernels in csrc/. It is built into paper_2208_12964_b200/lib/ so that it
travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libuscg_b200.so")
CLI = os.path.join(LIBDIR, "uscg_b200")  # the reference's CLI pipeline over the C ABI
CLI_SRC = os.path.join(HERE, "cli", "uscg_cli.cpp")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["api.cu", "kernels.cu", "mart_sweep.cu", "mart_tile.cu", "mart_levels.cu", "wave_build.cu", "metrics.cu", "cartesian.cu", "schedule_gpu.cu", "schedule.cpp"]
HEADERS = ["internal.cuh", "kernels.h", "schedule.h", "ddmath.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# --fmad=false: the fp64 index arithmetic must round exactly like the
# reference's g++ build (no contraction into FMA), see DESIGN.md §4.
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-O2", "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "uscg_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def _cli_stale() -> bool:
    if not os.path.exists(CLI):
        return True
    t = os.path.getmtime(CLI)
    deps = [CLI_SRC, LIB, os.path.join(ROOT, "include", "uscg_b200.h"),
            os.path.join(ROOT, "include", "uscg_b200_io.hpp")]
    return any(os.path.getmtime(d) > t for d in deps)


def build_cli() -> str:
    """g++ build of the CLI (host C++17 over the C ABI), rpath to lib/."""
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), CLI_SRC, "-o", CLI + ".tmp",
           "-L", LIBDIR, "-luscg_b200", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"CLI build failed:\n{r.stdout}\n{r.stderr}")
    os.replace(CLI + ".tmp", CLI)
    return CLI


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        if _cli_stale():
            build_cli()
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):
        obj = os.path.join(LIBDIR, os.path.splitext(src)[0] + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    objs = []
    log = []
    # translation units compile independently: one nvcc per source, in parallel
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as pool:
        results = list(pool.map(compile_one, SOURCES))
    for src, obj, r in results:
        log.append(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(os.path.join(LIBDIR, "ptxas.log"), "w") as f:
        f.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    build_cli()
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=False))
