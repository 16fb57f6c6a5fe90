"""Build the in-tree device library libsketchpress_b200.so (sm_100a only).

    python -m paper_2105_01271_b200.build [--force]

Plain nvcc, one translation unit per .cu, linked into a shared library with
an extern "C" surface (include/sketchpress_b200.h).  The .so is written next
to this file so it travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libsketchpress_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", str(ROOT / "include")]


def sources():
    return sorted(CSRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + [ROOT / "include" / "sketchpress_b200.h"]
    return any(p.stat().st_mtime > t for p in deps)


def _compile(src: Path) -> Path:
    obj = BUILD / (src.stem + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    if os.environ.get("SPB_PTXAS_V"):
        cmd += ["-Xptxas", "-v"]
    if os.environ.get("SPB_NVCC_EXTRA"):  # e.g. -DSPB_JACOBI_TRACE for diagnostic builds
        cmd += os.environ["SPB_NVCC_EXTRA"].split()
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
    if res.stderr.strip() and os.environ.get("SPB_PTXAS_V"):
        sys.stderr.write(res.stderr)
    return obj


def build(force: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    if not shutil.which(NVCC) and not Path(NVCC).exists():
        raise RuntimeError(f"nvcc not found at {NVCC}")
    BUILD.mkdir(exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(_compile, sources()))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
