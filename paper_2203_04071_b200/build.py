"""Ahead-of-time build of libaxq.so (sm_100a) -- in-tree so the .so travels with the repo."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libaxq.so"
SOURCES = [CSRC / "axq_api.cu", CSRC / "mm_delta8.cu", CSRC / "mm_i16.cu", CSRC / "mm_i32.cu", CSRC / "mm_i32h.cu", CSRC / "mm_p4.cu", CSRC / "mm_lstm.cu", CSRC / "mm_gconv.cu", CSRC / "mm_wide.cu", CSRC / "mm_ste.cu"]
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [ROOT / "include" / "axq.h"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-I", str(ROOT / "include"),
]


def _local_deps(src: Path, seen=None) -> set:
    """The source and every repo header it includes, transitively (for incremental builds)."""
    import re
    seen = set() if seen is None else seen
    if src in seen or not src.exists():
        return seen
    seen.add(src)
    for inc in re.findall(r'#include\s+"([^"]+)"', src.read_text()):
        for base in (src.parent, ROOT / "include"):
            if (base / inc).exists():
                _local_deps((base / inc).resolve(), seen)
                break
    return seen


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(d.stat().st_mtime > t for d in DEPS if d.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile each translation unit in parallel (-c), then link the shared library."""
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    comp = [f for f in NVCC_FLAGS if f != "-shared"]

    def cc(src: Path) -> Path:
        obj = objdir / (src.stem + ".o")
        if not force and obj.exists() and all(
                d.stat().st_mtime <= obj.stat().st_mtime for d in _local_deps(src)):
            return obj
        cmd = [NVCC, *comp, *(["-Xptxas", "-v"] if verbose else []), "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError("nvcc failed on %s" % src)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(cc, SOURCES))
    tmp = LIB.with_name("libaxq.so.tmp%d" % os.getpid())
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           *map(str, objs), "-o", str(tmp)])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
