"""In-tree build of the sm_100a shared library (nvcc, no JIT cache).

    python -m paper_2602_22625_b200.build
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
SOURCES = ["pf_bin.cu", "pf_render.cu", "pf_step.cu", "pf_adam.cu", "pf_aux.cu", "pf_comm.cu"]
HEADERS = ["pf_common.cuh", "pf_bins.cuh"]
LIB = PKG / "_lib" / "libprimfit_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


LIB_DIAG = PKG / "_lib" / "libprimfit_b200_diag.so"


def build(force: bool = False, verbose: bool = False) -> Path:
    """The product library (diagnostics compiled out: -DPF_DIAG=0) and the
    diagnostics library (timeline / step profile, selected by PF_TIMELINE /
    PF_STEP_PROF in _native), every translation unit of both in parallel."""
    deps = [CSRC / s for s in SOURCES] + [CSRC / h for h in HEADERS]
    deps.append(ROOT / "include" / "primfit_b200.h")
    if not force and not _stale(LIB, deps) and not _stale(LIB_DIAG, deps):
        return LIB
    LIB.parent.mkdir(parents=True, exist_ok=True)
    libs = {LIB: ["-DPF_DIAG=0"], LIB_DIAG: ["-DPF_DIAG=1"]}
    objs, procs = {lib: [] for lib in libs}, []
    for lib, defs in libs.items():
        for s in SOURCES:  # one nvcc per translation unit, concurrently
            obj = LIB.parent / (Path(s).stem + ("_diag" if lib == LIB_DIAG else "") + ".o")
            cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-I", str(ROOT / "include"), *defs, "-c", str(CSRC / s), "-o", str(obj)]
            # diagnostics only: extra -D switches for A/B builds (e.g. -DPF_NBUF=3)
            cmd += os.environ.get("PF_NVCC_DEFS", "").split()
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), file=sys.stderr)
            procs.append((subprocess.Popen(cmd), cmd))
            objs[lib].append(str(obj))
    failed = [cmd for p, cmd in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    for lib, lo in objs.items():
        tmp = lib.with_suffix(".so.tmp")
        subprocess.run([nvcc(), *ARCH, "-shared", "-o", str(tmp), *lo], check=True)
        os.replace(tmp, lib)
        for o in lo:
            Path(o).unlink(missing_ok=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
