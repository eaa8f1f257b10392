"""Build lib/libcoulomb.so for sm_100a with nvcc (in-tree, travels with the repo)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = [os.path.join(HERE, "csrc", "cc_kernels.cu"), os.path.join(HERE, "csrc", "cc_dist.cu"),
           os.path.join(HERE, "csrc", "cc_migrate.cu")]
HEADERS = [os.path.join(HERE, "csrc", "cc_device.cuh"), os.path.join(ROOT, "include", "coulomb.h")]
OUT = os.path.join(HERE, "lib", "libcoulomb.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(p) > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        os.makedirs(os.path.dirname(OUT), exist_ok=True)
        # CC_NVCC_EXTRA: extra -D switches for design studies (tools/collide_shape.sh); unset in product builds
        cmd = [NVCC, *FLAGS, *os.environ.get("CC_NVCC_EXTRA", "").split(), "-o", OUT, *SOURCES, "-lnccl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
        if verbose:
            print(r.stderr)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
