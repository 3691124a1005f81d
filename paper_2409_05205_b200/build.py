"""Builds libhe_rotfree.so (sm_100a) in-tree with nvcc."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libhe_rotfree.so")
U1_LIB = os.path.join(HERE, "libhe_u1.so")
U1_SRC = os.path.join(HERE, "csrc", "u1_microbench.cu")
SRCS = [os.path.join(HERE, "csrc", f) for f in ("he_host.cu", "he_kernels.cu")]
DEPS = SRCS + [os.path.join(HERE, "csrc", "he_internal.cuh"),
               os.path.join(ROOT, "include", "he_rotfree.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
         "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
         "-I" + os.path.join(ROOT, "include")]


def build(force: bool = False, verbose: bool = False) -> str:
    stale = not os.path.exists(LIB) or any(
        os.path.getmtime(d) > os.path.getmtime(LIB) for d in DEPS)
    if force or stale:
        cmd = [NVCC] + FLAGS + (["-Xptxas", "-v"] if verbose else []) + \
            ["-o", LIB] + SRCS
        subprocess.check_call(cmd)
    if force or not os.path.exists(U1_LIB) or any(
            os.path.getmtime(d) > os.path.getmtime(U1_LIB)
            for d in (U1_SRC, DEPS[2])):
        subprocess.check_call([NVCC] + FLAGS + ["-o", U1_LIB, U1_SRC])
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
