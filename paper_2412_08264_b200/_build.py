"""In-tree build of the sm_100a shared library (``_lib/libkrecycle_b200.so``).

Plain ``nvcc -shared``: no torch types cross the ABI, so the library is built
without torch headers and loaded through ctypes (see ``_lib.py``).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB_NAME = os.environ.get("KR_LIB_NAME", "libkrecycle_b200.so")
SOURCES = ["kr_capi.cu", "kr_ops.cu", "kr_rminres.cu", "kr_rminres_dyn.cu", "kr_cg.cu", "kr_eig.cu", "kr_small.cu", "kr_qrcp.cu", "kr_recycle.cu", "kr_gemm.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3"] + os.environ.get("KR_NVCC_FLAGS", "").split()


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def lib_path() -> Path:
    return OUT_DIR / LIB_NAME


def _stale(out: Path) -> bool:
    if not out.exists():
        return True
    mtime = out.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))
    deps.append(PKG.parent / "include" / "krecycle_b200.h")
    return any(d.exists() and d.stat().st_mtime > mtime for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every .cu into one shared library for sm_100a (objects in parallel)."""
    out = lib_path()
    if not force and not _stale(out):
        return out
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:
        obj = OUT_DIR / (Path(src).stem + ".o")
        cmd = [nvcc(), *ARCH, *FLAGS, "-I", str(PKG.parent / "include"), "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(str(obj))
    failed = []
    for src, p in procs:
        log, _ = p.communicate()
        if verbose and log:
            sys.stderr.write(log)
        if p.returncode != 0:
            failed.append(f"{src}:\n{log}")
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(failed))
    tmp = out.with_suffix(".so.tmp")
    link = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", str(tmp), "-lcusolver",
            "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
    os.replace(tmp, out)
    for o in objs:
        Path(o).unlink(missing_ok=True)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
