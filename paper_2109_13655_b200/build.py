"""In-tree build of libsssvd_gpu.so (sm_100a only) and the oracle's RNG helper.

    python -m paper_2109_13655_b200.build        # or __graft_entry__.build()

Every .cu is compiled with -gencode arch=compute_100a,code=sm_100a -lineinfo; host mirrors of
the reference's O(N) logic (host_mirror.cpp) are compiled with g++ -O3 (no -march: the same
floating-point semantics as the reference's Release build). The .so lands next to this file so
it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsssvd_gpu.so")
CLI = os.path.join(HERE, "sssvd-gpu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
            "--expt-relaxed-constexpr", "-I", CSRC]
CU_SOURCES = ["zgemm.cu", "dgemm.cu", "lu.cu", "gram.cu", "moments.cu", "jacobi_svd.cu", "householder_qr.cu", "sparse.cu", "sssvd_gpu.cu"]
CXX_SOURCES = ["host_mirror.cpp", "matrix_market.cpp", "problems.cpp"]


def _run(cmd, log):
    p = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
    if p.returncode != 0:
        sys.stderr.write(p.stdout + p.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ... (see {log})")
    return p


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(HERE, "..", "include", "sssvd_gpu.h"))
    jobs, objs = [], []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append(([NVCC] + ARCH + CU_FLAGS + ["-c", s, "-o", o], o + ".log"))
    for src in CXX_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append((["g++", "-O3", "-std=c++20", "-fPIC", "-c", s, "-o", o], o + ".log"))
    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(lambda j: _run(*j), jobs))
    if force or jobs or _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs +
             ["-ldl"], os.path.join(BUILD, "link.log"))
    # the command-line front end (proj/tools/sssvd.cpp) over the C ABI, rpath'ed to this directory
    cli_src = os.path.join(CSRC, "cli.cpp")
    hpp = os.path.join(HERE, "..", "include", "sssvd_gpu.hpp")
    if force or _stale(CLI, [cli_src, LIB, hpp] + headers):
        _run(["g++", "-O2", "-std=c++20", cli_src, "-o", CLI, "-L", HERE, "-lsssvd_gpu",
              "-L/usr/local/cuda/lib64", "-Wl,-rpath,$ORIGIN"], os.path.join(BUILD, "cli.log"))
    if verbose:
        print(LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
