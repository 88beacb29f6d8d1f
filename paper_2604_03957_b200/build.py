"""Build libbwta.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python paper_2604_03957_b200/build.py [--force] [-v]
(run it by path: importing the package loads libbwta.so, which may be stale)

The CUDA runtime is linked statically and the driver API (TMA descriptors) is
resolved at run time through cudaGetDriverEntryPoint, so the library loads on
a machine without a GPU driver (the CPU tests check its exported symbols).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libbwta.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-cudart", "static",
    "-Xptxas", "-warn-spills",
]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps() -> list[str]:
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.h"))) + sorted(
        glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "bwta.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force: bool = False, verbose: bool = False, trace: bool = False, variant: str = "",
          defines: tuple = ()) -> str:
    """trace=True builds libbwta_trace.so with the -DBWTA_TRACE timeline hooks (tools only);
    variant="x" + defines builds libbwta_x.so with extra -D flags (A/B experiments, tools only)."""
    tag = "_".join(t for t in ("trace" if trace else "", variant) if t)
    lib = LIB.replace("libbwta.so", f"libbwta_{tag}.so") if tag else LIB
    if not force and not tag and not stale():
        return LIB
    objdir = os.path.join(PKG, f"build_{tag}" if tag else "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        if trace:
            cmd.append("-DBWTA_TRACE")
        cmd += [f"-D{d}" for d in defines]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if out.strip() and (verbose or p.returncode != 0 or "warning" in out.lower()):
            sys.stderr.write(out)
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"nvcc failed for {src}\n")
    if failed:
        raise RuntimeError("libbwta.so build failed")
    tmp = lib + f".{os.getpid()}.tmp"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                           "-Xcompiler", "-fvisibility=hidden", "-o", tmp, *objs])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    defs = tuple(a[2:] for a in sys.argv if a.startswith("-D"))
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv, variant=var,
                defines=defs))
