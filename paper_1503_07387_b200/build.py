"""In-tree build of the native libraries (run here on CPU; the .so files travel
to the GPU box with the repo snapshot).

  libmvb_cuda.so      the decoder: sm_100a kernels + C ABI (nvcc)
  libmvb_workload.so  host generators / encoder for bench and test inputs (g++)
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _run(cmd, verbose):
    if verbose:
        print("+", " ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=ROOT)


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_cuda(force: bool = False, verbose: bool = True, ptxas_verbose: bool = False) -> str:
    target = os.path.join(HERE, "libmvb_cuda.so")
    sources = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh"))]
    sources.append(os.path.join(ROOT, "include", "mvb_cuda.h"))
    if force or _stale(target, sources):
        if os.path.exists(target):
            os.remove(target)  # never leave a stale library behind a failed build
        cmd = [_nvcc(), *NVCC_FLAGS]
        if ptxas_verbose:
            cmd += ["-Xptxas", "-v"]
        cmd += ["-o", target, os.path.join(CSRC, "mvb_cuda.cu")]
        _run(cmd, verbose)
    return target


def build_workload(force: bool = False, verbose: bool = True) -> str:
    target = os.path.join(HERE, "libmvb_workload.so")
    src = os.path.join(CSRC, "workload.cpp")
    if force or _stale(target, [src]):
        cxx = os.environ.get("CXX", "g++")
        _run([cxx, "-O3", "-std=c++17", "-fPIC", "-shared", "-pthread", "-o", target, src], verbose)
    return target


def build_cpp_tests(force: bool = False, verbose: bool = True) -> str:
    """tests/cpp/sharded_abi_test: C++ driver of the multi-GPU C-ABI entry,
    checked against the test-only oracle (needs libmvb_cuda.so and
    oracle/liboracle.so)."""
    src = os.path.join(ROOT, "tests", "cpp", "sharded_abi_test.cpp")
    target = os.path.join(ROOT, "tests", "cpp", "sharded_abi_test")
    deps = [src, os.path.join(HERE, "libmvb_cuda.so"), os.path.join(ROOT, "include", "mvb_cuda.h")]
    if force or _stale(target, deps):
        cuda = os.path.dirname(os.path.dirname(_nvcc()))
        _run([os.environ.get("CXX", "g++"), "-O2", "-std=c++17", f"-I{cuda}/include", "-o", target, src,
              f"-L{HERE}", "-lmvb_cuda", f"-L{os.path.join(ROOT, 'oracle')}", "-loracle", f"-L{cuda}/lib64", "-lcudart",
              "-Wl,-rpath,$ORIGIN/../../paper_1503_07387_b200", "-Wl,-rpath,$ORIGIN/../../oracle",
              f"-Wl,-rpath,{cuda}/lib64"], verbose)
    return target


def build_all(force: bool = False, verbose: bool = True) -> None:
    build_cuda(force, verbose)
    build_workload(force, verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
