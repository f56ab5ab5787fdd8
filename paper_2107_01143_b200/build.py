"""In-tree build of libgvo_b200.so (sm_100a) with nvcc.

Every .cu under csrc/ is compiled with
  -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false
(--fmad=false keeps the float assembly bit-identical to the Python
reference: no contracted multiply-adds) and linked into one shared library
next to this file.

Incremental: an object is rebuilt when a source or header is newer, or when
the compile flags changed (the object directory carries a stamp of the
flag set, GVO_BUILD_DEFS included, so an A/B define can never leave stale
objects in the product library).  The library exports gvo_build_id(): a
hash of every source, header and flag, which profiles/ captures are tagged
with.
"""
from __future__ import annotations

import hashlib
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
DEFS = os.environ.get("GVO_BUILD_DEFS", "").split()
if DEFS and not VARIANT:
    raise RuntimeError("GVO_BUILD_DEFS needs a GVO_BUILD_VARIANT name (the product library takes no A/B defines)")
OBJ = HERE / "build" / ("obj_" + VARIANT if VARIANT else "obj")
LIB = HERE / ("libgvo_b200_" + VARIANT + ".so" if VARIANT else "libgvo_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                "-Xptxas", "-warn-spills", "--expt-relaxed-constexpr"] + (
                    ["-DGVO_PHASE_STATS=1"] if VARIANT == "prof" else []) + DEFS


def _headers():
    return sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.inc")) + [
        HERE.parent / "include" / "gvo_b200.h"]


def build_id() -> str:
    """Hash of every source, header and compile flag of this build."""
    h = hashlib.sha256(" ".join(FLAGS).encode())
    for p in sorted(CSRC.glob("*.cu")) + _headers():
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()[:16]


def _flags_stamp() -> str:
    return hashlib.sha256(" ".join(FLAGS).encode()).hexdigest()[:16]


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


def _compile(src: Path, verbose: bool, bid: str, fresh: bool) -> Path:
    obj = OBJ / (src.stem + ".o")
    newest = max([src.stat().st_mtime] + [h.stat().st_mtime for h in _headers() + _included_sources(src)])
    extra = []
    if src.name == "capi.cu":  # the id changes with every source: only the ABI unit carries it
        extra = [f'-DGVO_BUILD_ID="{bid}"']
        stamp = OBJ / "capi.id"
        if obj.exists() and not fresh and stamp.exists() and stamp.read_text() == bid and obj.stat().st_mtime >= newest:
            return obj
    elif obj.exists() and not fresh and obj.stat().st_mtime >= newest:
        return obj
    cmd = [NVCC, *FLAGS, *extra, "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if verbose and (r.stderr.strip() or r.stdout.strip()):
        print(r.stdout, r.stderr, file=sys.stderr)
    if src.name == "capi.cu":
        (OBJ / "capi.id").write_text(bid)
    return obj


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    stamp = OBJ / "flags.stamp"
    fresh = not stamp.exists() or stamp.read_text() != _flags_stamp()
    bid = build_id()
    sources = sorted(CSRC.glob("*.cu"))
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, bid, fresh), sources))
    stamp.write_text(_flags_stamp())
    if LIB.exists() and not fresh and LIB.stat().st_mtime >= max(o.stat().st_mtime for o in objs):
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
