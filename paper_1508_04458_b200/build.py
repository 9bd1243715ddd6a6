"""In-tree build of libwamgpu.so for sm_100a (no JIT cache; the .so travels
with the repo snapshot to the GPU box).

    python -m paper_1508_04458_b200.build        # or build() from __graft_entry__
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libwamgpu.so")
BUILD = os.path.join(HERE, "_build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# --fmad=false: no implicit FMA contraction anywhere on the device (the Siddon
# tracer and the root solver must round exactly like the -ffp-contract=off
# host code); the accumulation loops use explicit fma() whose products are
# exact (fp32 x fp32 in fp64), so they lose nothing.
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off",
           "-I" + os.path.join(ROOT, "include")]
CXXFLAGS = ["-O3", "-std=c++20", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
            "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError("build failed: " + cmd[0])
    return r.stdout + r.stderr


def _newer(out, deps):
    if not os.path.exists(out):
        return False
    t = os.path.getmtime(out)
    return all(os.path.getmtime(d) <= t for d in deps)


def build(verbose=False, force=False):
    os.makedirs(BUILD, exist_ok=True)
    srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))]
    hdrs = srcs + [os.path.join(ROOT, "include", "wamgpu.h")]
    if not force and _newer(OUT, hdrs):
        return OUT
    host_o = os.path.join(BUILD, "host_model.o")
    log = _run(["g++"] + CXXFLAGS + ["-c", os.path.join(CSRC, "host_model.cpp"), "-o", host_o])
    cu_o = os.path.join(BUILD, "wamgpu.o")
    log += _run([NVCC] + ARCH + NVFLAGS + ["-Xptxas", "-v", "-c", os.path.join(CSRC, "wamgpu.cu"), "-o", cu_o])
    log += _run([NVCC] + ARCH + ["-shared", "-o", OUT + ".tmp", cu_o, host_o,
                                 "-L/usr/lib/x86_64-linux-gnu", "-lnccl", "-lcudart"])
    os.replace(OUT + ".tmp", OUT)
    with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
        f.write(log)
    if verbose:
        print(log)
    return OUT


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(OUT)
