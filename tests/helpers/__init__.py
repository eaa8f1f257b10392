"""Test-only helpers: the third-party cross-check library (CUB radix sort, cuRAND Philox)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "thirdparty.cu")
LIB = os.path.join(HERE, "libthirdparty.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build() -> str:
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-Xcompiler", "-fPIC",
               "-shared", "-o", LIB, SRC]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    return LIB
