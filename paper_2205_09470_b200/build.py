"""Builds libnebula_sync.so in-tree for sm_100a (B200) with nvcc.

    python -m paper_2205_09470_b200.build [--force]

Flags: no --use_fast_math; -fmad=false -ftz=false -prec-div=true
-prec-sqrt=true so the codec arithmetic is IEEE binary32, one rounding per operation.  NCCL
is the torch-bundled libnccl.so.2 (same soname torch loads, so one NCCL per process).
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libnebula_sync.so")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def _nccl_dirs():
    cands = []
    try:
        import nvidia.nccl  # torch's bundled NCCL wheel
        base = list(nvidia.nccl.__path__)[0]
        cands.append((os.path.join(base, "include"), os.path.join(base, "lib")))
    except Exception:
        pass
    cands.append(("/usr/include", "/usr/lib/x86_64-linux-gnu"))
    for inc, lib in cands:
        if os.path.exists(os.path.join(inc, "nccl.h")) and glob.glob(os.path.join(lib, "libnccl.so*")):
            return inc, lib
    raise RuntimeError("nccl.h / libnccl.so not found")


def _cusolver_dirs():
    """torch's bundled cuSOLVER (the same libcublas.so.12 torch loads resolves its symbols)."""
    try:
        import nvidia.cusolver
        base = list(nvidia.cusolver.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "cusolverDn.h")) and glob.glob(os.path.join(lib, "libcusolver.so*")):
            return inc, lib
    except Exception:
        pass
    return "/usr/local/cuda/include", "/usr/local/cuda/lib64"


def _nvcc():
    for p in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if p and os.path.exists(p):
            return p
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu"))) + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + \
        sorted(glob.glob(os.path.join(CSRC, "*.h"))) + sorted(glob.glob(os.path.join(CSRC, "*.inc"))) + \
        [os.path.join(INCLUDE, "nebula_sync.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources() + [__file__])


def _compile_one(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    return r.returncode, r.stdout + r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every .cu to an object in parallel (one nvcc per file), then link the shared
    library.  Same flags for every translation unit."""
    if not force and up_to_date():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    inc, lib = _nccl_dirs()
    sinc, slib = _cusolver_dirs()
    cus = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    common = [_nvcc(), ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
              "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
              "-Xptxas", "-v" if verbose else "-O3", f"-I{INCLUDE}", f"-I{inc}", f"-I{sinc}"]
    objs, cmds = [], []
    for cu in cus:
        o = os.path.join(objdir, os.path.basename(cu)[:-3] + ".o")
        objs.append(o)
        cmds.append(common + ["-c", cu, "-o", o])
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        results = list(ex.map(_compile_one, cmds))
    for (rc, out), cu in zip(results, cus):
        if rc != 0:
            sys.stderr.write(out)
            raise RuntimeError(f"nvcc failed compiling {os.path.basename(cu)}")
        if verbose:
            sys.stderr.write(out)
    link = [_nvcc(), ARCH, "-shared", "-Xcompiler", "-fPIC", f"-L{lib}", "-l:libnccl.so.2",
            f"-Xlinker=-rpath,{lib}", f"-L{slib}", "-l:libcusolver.so.11", f"-Xlinker=-rpath,{slib}",
            "-o", LIB + ".tmp"] + objs
    rc, out = _compile_one(link)
    if rc != 0:
        sys.stderr.write(out)
        raise RuntimeError("nvcc failed linking libnebula_sync.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
