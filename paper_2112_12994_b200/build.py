"""Build the in-tree CUDA library (sm_100a) with nvcc.  No JIT cache: the .so
lives next to this file so it travels with the repo snapshot."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["csrc/engine.cu"]
HEADERS = sorted("csrc/" + f for f in os.listdir(os.path.join(HERE, "csrc")) if f.endswith((".cuh", ".h"))) + [
    "../include/toepfit_b200.h"]
OUT = os.path.join(HERE, "libtoepfit_b200.so")


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(os.path.join(HERE, d)) > t for d in deps)


def nccl_flags() -> list:
    """Link the NCCL that torch bundles (nvidia-nccl wheel) when present, with an
    rpath to it: a process that also loads torch then holds ONE libnccl.so.2
    (the system 2.27 copy lacks symbols torch 2.11 needs).  Else the system NCCL."""
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia")
        for base in (spec.submodule_search_locations or []) if spec else []:
            lib = os.path.join(base, "nccl", "lib")
            inc = os.path.join(base, "nccl", "include")
            if os.path.exists(os.path.join(lib, "libnccl.so.2")) and os.path.exists(os.path.join(inc, "nccl.h")):
                return ["-I", inc, "-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
    except Exception:
        pass
    return ["-lnccl"]


def build(force: bool = False, verbose: bool = False) -> str:
    deps = SOURCES + HEADERS
    if force or _stale(OUT, deps):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
               "-o", OUT, *[os.path.join(HERE, s) for s in SOURCES], *nccl_flags()]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
    return OUT


ROOT = os.path.dirname(HERE)
CPP_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp")
CPP_TEST_OUT = os.path.join(ROOT, "build", "test_cpp_api")


def build_cpp_api_test(force: bool = False) -> str:
    """C++ host-API program (include/toepfit_b200.hpp) linked against the library."""
    lib = build()
    deps = [CPP_TEST_SRC, os.path.join(ROOT, "include", "toepfit_b200.hpp"), lib]
    if force or not os.path.exists(CPP_TEST_OUT) or any(
            os.path.getmtime(d) > os.path.getmtime(CPP_TEST_OUT) for d in deps):
        os.makedirs(os.path.dirname(CPP_TEST_OUT), exist_ok=True)
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), CPP_TEST_SRC,
                               "-L", HERE, "-ltoepfit_b200",
                               "-Wl,-rpath,$ORIGIN/../paper_2112_12994_b200", "-o", CPP_TEST_OUT])
    return CPP_TEST_OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
