"""Builds libmoedc.so in-tree (sm_100a only).

    python -m paper_2504_19925_b200._build        # or __graft_entry__.build()

nvcc cross-compiles for sm_100a without a GPU.  Flags:
  -gencode arch=compute_100a,code=sm_100a -lineinfo -O3
  -fmad=false -prec-div=true -prec-sqrt=true -ftz=false   (IEEE fp32 per op: Adam bit parity)
  host: -ffp-contract=off (Alg. 1 float64 left to right, no FMA)
cudart is linked statically (nvcc's default), so the library does not depend on which
libcudart the host process (PyTorch) loaded.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(ROOT, "include")
OUT = os.path.join(HERE, "libmoedc.so")
OBJ = os.path.join(HERE, "build")

CU = ["ctx.cu", "dispatch.cu", "update.cu", "synth.cu", "tokens.cu"]
CPP = ["plan.cpp", "step.cpp"]
HEADERS = [os.path.join(CSRC, h) for h in ("common.h", "internal.h", "fastdiv.h")] + \
    [os.path.join(INC, h) for h in ("moe_dc.h", "moe_synth.h", "moe_tokens.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
                  "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
                  "-I", INC, "-I", CSRC]
CXXFLAGS = ["-O2", "-fPIC", "-std=c++17", "-ffp-contract=off", "-fno-fast-math",
            "-I", INC, "-I", CSRC, "-I", "/usr/local/cuda/include"]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr, flush=True)


def build(verbose: bool = False, ptxas_verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    objs = []
    for f in CU:
        src = os.path.join(CSRC, f)
        obj = os.path.join(OBJ, f + ".o")
        if _stale(obj, [src] + HEADERS) or ptxas_verbose:
            extra = ["-Xptxas", "-v"] if ptxas_verbose else []
            _run([NVCC] + NVFLAGS + extra + ["-c", src, "-o", obj], verbose or ptxas_verbose)
        objs.append(obj)
    for f in CPP:
        src = os.path.join(CSRC, f)
        obj = os.path.join(OBJ, f + ".o")
        if _stale(obj, [src] + HEADERS):
            _run(["g++"] + CXXFLAGS + ["-c", src, "-o", obj], verbose)
        objs.append(obj)
    if _stale(OUT, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", OUT] + objs, verbose)
    return OUT


if __name__ == "__main__":
    print(build(verbose=True, ptxas_verbose="-v" in sys.argv))
