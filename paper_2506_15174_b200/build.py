"""Build libescs.so in-tree: sm_100a kernels (nvcc) + host planner/ABI (g++).

    python -m paper_2506_15174_b200.build [--force] [--verbose]

Produces ``paper_2506_15174_b200/libescs.so`` (and, for the bench only,
``paper_2506_15174_b200/libescs_bench.so`` with the cuSPARSE/cuBLAS baselines).
nvcc cross-compiles for sm_100a without a GPU.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.environ.get("ESCS_BUILD_DIR") or os.path.join(HERE, "build")
LIB = os.environ.get("ESCS_LIB") or os.path.join(HERE, "libescs.so")
BENCH_LIB = os.path.join(HERE, "libescs_bench.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                  "-Xptxas", "-v", "-I", CSRC, "-I", os.path.join(ROOT, "include")] + \
    os.environ.get("ESCS_NVFLAGS", "").split()       # extra flags for A/B experiment builds
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-pthread", "-Wall", "-Wno-unused-function",
            "-I", os.path.join(CUDA, "include"), "-I", CSRC, "-I", os.path.join(ROOT, "include")]

LIB_CU = ["launch.cu", "k_b4.cu", "k_b8.cu", "k_b16.cu", "k_b32.cu", "k_b64.cu", "k_b128.cu", "k_b256.cu",
          "k_s1.cu", "k_s2.cu", "k_s4.cu", "k_s8.cu"]
LIB_CPP = ["plan.cpp", "abi.cpp"]
BENCH_CU = ["baselines.cu"]


def _deps():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "escs.h")]


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs if os.path.exists(s))


def _compile(src, force, verbose):
    path = os.path.join(CSRC, src)
    obj = os.path.join(BUILD, src + ".o")
    if not force and not _stale(obj, [path] + _deps()):
        return obj, ""
    if src.endswith(".cu"):
        cmd = [NVCC] + NVFLAGS + ["-c", path, "-o", obj]
    else:
        cmd = ["g++"] + CXXFLAGS + ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    with open(obj + ".log", "w") as f:
        f.write(r.stdout + r.stderr)
    return obj, (r.stdout + r.stderr) if verbose else ""


def build(force: bool = False, verbose: bool = False, bench: bool = True) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = LIB_CU + LIB_CPP + (BENCH_CU if bench and os.path.exists(os.path.join(CSRC, "baselines.cu")) else [])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, force, verbose), srcs))
    objs = {os.path.basename(o)[:-2]: o for o, _ in results}
    if verbose:
        for _, log in results:
            if log:
                print(log)
    lib_objs = [objs[s] for s in LIB_CU + LIB_CPP]
    if force or _stale(LIB, lib_objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + lib_objs + ["-cudart", "static", "-lpthread"]
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    if "baselines.cu" in objs:
        bobj = [objs["baselines.cu"]]
        if force or _stale(BENCH_LIB, bobj):
            tmp = BENCH_LIB + f".tmp{os.getpid()}"
            cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + bobj + \
                  ["-cudart", "static", "-lcusparse", "-lcublas"]
            subprocess.check_call(cmd)
            os.replace(tmp, BENCH_LIB)
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args(argv)
    print(build(a.force, a.verbose))


if __name__ == "__main__":
    sys.exit(main())
