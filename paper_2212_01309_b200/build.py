"""Build libwdd.so in-tree for sm_100a with nvcc (no torch JIT, no cache outside the repo).

    python -m paper_2212_01309_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("WDD_LIB_OUT") or os.path.join(HERE, "_lib", "libwdd.so")
SOURCES = [os.path.join(CSRC, f) for f in ("kernels.cu", "bank.cu", "fullwdd.cu", "plan.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("internal.h", "tc.cuh", "fft.cuh")] + [os.path.join(ROOT, "include", "wdd.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "-Xcompiler", "-O2",
    "-Xptxas", "-v",
    "-shared",
]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = LIB + f".{os.getpid()}.tmp"      # (per-process temp: several ranks may build at once)
    extra = os.environ.get("WDD_NVCC_EXTRA", "").split()
    cmd = [nvcc, *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-o", tmp, *SOURCES,
           "-lcufft", "-lnccl", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed building libwdd.so")
    os.replace(tmp, LIB)
    if not os.environ.get("WDD_LIB_OUT"):
        # register / spill / shared-memory report of the shipped build (tracked); the compile-time
        # lines change on every build and are dropped so an unchanged source leaves no diff
        log = "".join(ln for ln in res.stderr.splitlines(True) if "Compile time" not in ln)
        path = os.path.join(HERE, "_lib", "ptxas.log")
        old = open(path).read() if os.path.exists(path) else None
        if log != old:
            with open(path, "w") as f:
                f.write(log)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
