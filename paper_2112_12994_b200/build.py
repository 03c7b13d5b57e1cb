"""Build the in-tree CUDA library (sm_100a) with nvcc.  No JIT cache: the .so
lives next to this file so it travels with the repo snapshot."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["csrc/engine.cu"]
HEADERS = ["csrc/common.cuh", "csrc/k_pass.cuh", "csrc/k_sample.cuh", "csrc/k_gram.cuh",
           "csrc/k_cholinv.cuh", "csrc/k_tpu.cuh", "csrc/k_rh.cuh", "csrc/engine.h", "../include/toepfit_b200.h"]
OUT = os.path.join(HERE, "libtoepfit_b200.so")


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(os.path.join(HERE, d)) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    deps = SOURCES + HEADERS
    if force or _stale(OUT, deps):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
               "-o", OUT, *[os.path.join(HERE, s) for s in SOURCES]]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
