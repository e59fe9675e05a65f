"""In-tree build of libb2conv.so for sm_100a (nvcc cross-compiles without a GPU).

Two translation units, compiled to objects separately (each rebuilt only when
its own sources changed) and linked into one shared library:
  csrc/b2conv.cu — the conv hot path (all kernels in csrc/k_*.cuh + the C ABI);
  csrc/b2net.cu  — pooling / ReLU / layout conversion for whole-network runs."""

from __future__ import annotations

import hashlib
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
    out = {
        "b2conv.o": (os.path.join(CSRC, "b2conv.cu"), [os.path.join(CSRC, "b2conv.cu"), HEADER, *cuh]),
        "b2net.o": (os.path.join(CSRC, "b2net.cu"), [os.path.join(CSRC, "b2net.cu"), HEADER]),
    }
    # k_tconv instances, one translation unit per MODE (tconv_inst.cuh)
    for f in sorted(os.listdir(CSRC)):
        if f.startswith("inst_m") and f.endswith(".cu"):
            src = os.path.join(CSRC, f)
            out[f[:-3] + ".o"] = (src, [src, HEADER, *cuh])
    return out


def sources() -> list:
    out = [HEADER]
    out += [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh"))]
    return out


def _digest(deps, extra=()) -> str:
    """sha256 over the dependency files' contents and the compiler flags."""
    h = hashlib.sha256()
    for part in (*NVCC_FLAGS, *extra):
        h.update(part.encode() + b"\0")
    for path in sorted(deps):
        h.update(os.path.basename(path).encode() + b"\0")
        with open(path, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def _stamp_path(target: str) -> str:
    return target + ".sha256"


def _newer(target: str, deps) -> bool:
    """Up to date = the target exists and was built from exactly these source
    contents and flags (content hash, not mtimes: a copied tree has arbitrary
    mtimes, so an mtime gate could keep a stale library)."""
    stamp = _stamp_path(target)
    if not (os.path.exists(target) and os.path.exists(stamp)):
        return False
    with open(stamp) as fh:
        return fh.read().strip() == _digest(deps)


def _write_stamp(target: str, digest: str) -> None:
    with open(_stamp_path(target), "w") as fh:
        fh.write(digest + "\n")


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
    objs, todo = [], []
    for name, (main, deps) in units().items():
        obj = os.path.join(OBJDIR, name)
        if force or not _newer(obj, deps):
            todo.append((obj, main, _digest(deps)))  # digest of the sources as compiled (before nvcc reads them)
        objs.append(obj)

    def compile_one(job):
        obj, main, digest = job
        _run([nvcc, *NVCC_FLAGS, "-c", "-o", obj + ".tmp", main], verbose)
        os.replace(obj + ".tmp", obj)
        _write_stamp(obj, digest)

    # the translation units are independent: compile them in parallel (nvcc is single-threaded)
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        for _ in ex.map(compile_one, todo):
            pass
    digest = _digest(sources())
    if any(not _newer(o, d) for o, (_, d) in zip(objs, units().values())):
        raise RuntimeError("sources changed during the build; run it again")
    _run([nvcc, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", LIB + ".tmp", *objs], verbose)
    os.replace(LIB + ".tmp", LIB)
    _write_stamp(LIB, digest)
    return LIB


if __name__ == "__main__":
    print(build_lib(force=True, verbose=True))
