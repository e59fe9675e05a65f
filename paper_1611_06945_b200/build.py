"""In-tree build of libb2conv.so for sm_100a (nvcc cross-compiles without a GPU).

Two translation units, compiled to objects separately (each rebuilt only when
its own sources changed) and linked into one shared library:
  csrc/b2conv.cu — the conv hot path (all kernels in csrc/k_*.cuh + the C ABI);
  csrc/b2net.cu  — pooling / ReLU / layout conversion for whole-network runs."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libb2conv.so")
OBJDIR = os.path.join(HERE, "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills"]
HEADER = os.path.join(INCLUDE, "b2conv.h")


def units() -> dict:
    """object name -> (main .cu, every source it depends on)."""
    cuh = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith(".cuh")]
    return {
        "b2conv.o": (os.path.join(CSRC, "b2conv.cu"), [os.path.join(CSRC, "b2conv.cu"), HEADER, *cuh]),
        "b2net.o": (os.path.join(CSRC, "b2net.cu"), [os.path.join(CSRC, "b2net.cu"), HEADER]),
    }


def sources() -> list:
    out = [HEADER]
    out += [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh"))]
    return out


def _newer(target: str, deps) -> bool:
    return os.path.exists(target) and all(os.path.getmtime(s) <= os.path.getmtime(target) for s in deps)


def up_to_date() -> bool:
    return _newer(LIB, sources())


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd))
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-4000:]}")


def build_lib(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    os.makedirs(OBJDIR, exist_ok=True)
    objs = []
    for name, (main, deps) in units().items():
        obj = os.path.join(OBJDIR, name)
        if force or not _newer(obj, deps):
            _run([nvcc, *NVCC_FLAGS, "-c", "-o", obj + ".tmp", main], verbose)
            os.replace(obj + ".tmp", obj)
        objs.append(obj)
    _run([nvcc, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", LIB + ".tmp", *objs], verbose)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build_lib(force=True, verbose=True))
