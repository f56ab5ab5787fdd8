"""In-tree build of libgvo_b200.so (sm_100a) with nvcc.

Every .cu under csrc/ is compiled with
  -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false
(--fmad=false keeps the float assembly bit-identical to the Python
reference: no contracted multiply-adds) and linked into one shared library
next to this file.  Incremental: objects are rebuilt only when a source or
header is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
# GVO_BUILD_VARIANT=prof: same sources with the set kernel's per-CTA phase
# counters compiled in (tools/unit_profile.py), as a separate library; other
# variant names take extra -D flags from GVO_BUILD_DEFS (A/B experiments)
VARIANT = os.environ.get("GVO_BUILD_VARIANT", "")
OBJ = HERE / "build" / ("obj_" + VARIANT if VARIANT else "obj")
LIB = HERE / ("libgvo_b200_" + VARIANT + ".so" if VARIANT else "libgvo_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                "-Xptxas", "-warn-spills", "--expt-relaxed-constexpr"] + (
                    ["-DGVO_PHASE_STATS=1"] if VARIANT == "prof" else []) + os.environ.get("GVO_BUILD_DEFS", "").split()


def _headers():
    return list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(CSRC.glob("*.inc")) + [
        HERE.parent / "include" / "gvo_b200.h"]


def _included_sources(src: Path) -> list:
    """.cu files a translation unit #includes (k_sets1.cu includes k_sets.cu)."""
    out = []
    for line in src.read_text().splitlines():
        line = line.strip()
        if line.startswith("#include") and line.endswith('.cu"'):
            dep = CSRC / line.split('"')[1]
            if dep.exists():
                out.append(dep)
    return out


def _compile(src: Path, verbose: bool) -> Path:
    obj = OBJ / (src.stem + ".o")
    newest = max([src.stat().st_mtime] + [h.stat().st_mtime for h in _headers() + _included_sources(src)])
    if obj.exists() and obj.stat().st_mtime >= newest:
        return obj
    cmd = [NVCC, *FLAGS, "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if verbose and (r.stderr.strip() or r.stdout.strip()):
        print(r.stdout, r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    sources = sorted(CSRC.glob("*.cu"))
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), sources))
    if LIB.exists() and LIB.stat().st_mtime >= max(o.stat().st_mtime for o in objs):
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
