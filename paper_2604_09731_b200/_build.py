"""Build libsmart.so in-tree with nvcc for sm_100a (B200).  No torch involvement.

    python -m paper_2604_09731_b200._build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libsmart.so")
SOURCES = ["expand.cu", "select.cu", "mask_verify.cu", "step.cu", "api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "-I" + os.path.join(ROOT, "include"),
         "-diag-suppress", "550"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    # SMART_PROBES=1: compile the globaltimer/clock64 probes in (debug timelines, tests/probe_*.py);
    # the objects then go to their own directory and the library is always relinked
    probes = os.environ.get("SMART_PROBES") == "1"
    obj_dir = OBJ + ("_probes" if probes else "")
    flags = FLAGS + (["-DSMART_PROBES=1"] if probes else [])
    mark = os.path.join(ROOT, "build", "libsmart.flavor")
    flavor = "probes" if probes else "product"
    if not os.path.exists(mark) or open(mark).read() != flavor:
        force_link = True
    else:
        force_link = False
    os.makedirs(obj_dir, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith(".cuh")]
    headers.append(os.path.join(ROOT, "include", "smart.h"))
    objs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(obj_dir, s.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            cmd = [NVCC, *flags, "-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd))
            subprocess.check_call(cmd)
    if force or force_link or _stale(LIB, objs):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
               "-o", LIB, *objs, "-ldl"]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        with open(mark, "w") as f:
            f.write(flavor)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
