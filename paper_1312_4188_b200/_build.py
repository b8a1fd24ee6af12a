"""Build libpfw.so (the C-ABI of include/pfw.h) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = os.path.join(PKG, "csrc", "pfw.cu")
SRC_HOST = os.path.join(PKG, "csrc", "hostio.cpp")
HEADERS = [os.path.join(PKG, "csrc", "matchset.cuh"), os.path.join(PKG, "csrc", "hostpool.h")]
LIB = os.path.join(PKG, "libpfw.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
]


def build_native(verbose: bool = False, force: bool = False, out: str = LIB, defines=()) -> str:
    """Compile csrc/pfw.cu -> libpfw.so unless the library is newer than its sources.
    ``defines`` (e.g. ["PFW_GROUP=4"]) build experiment variants into ``out``."""
    deps = [SRC, SRC_HOST, *HEADERS, os.path.join(ROOT, "include", "pfw.h"), os.path.abspath(__file__)]
    if not force and os.path.exists(out) and all(os.path.getmtime(out) >= os.path.getmtime(d) for d in deps):
        return out
    tmp = out + ".tmp"
    cmd = [NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", tmp, SRC, SRC_HOST, "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr}")
    if verbose:
        print(res.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    build_native(verbose=True, force=True)
