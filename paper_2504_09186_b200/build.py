"""Build the CUDA C-ABI library ``libtnc_b200.so`` in-tree for sm_100a.

Every translation unit is compiled with
``nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` (the explicit
``a`` target is required for tcgen05 / TMA instructions) and linked into one
shared library with a static CUDA runtime, so the .so travels to the GPU box
with the repo snapshot.  ``python -m paper_2504_09186_b200.build`` rebuilds
when any source is newer than the library.
"""

from __future__ import annotations

import os
import re
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "libtnc_b200.so"
OBJ = PKG.parent / "build" / "obj"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA extension cannot be built")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


_INCLUDE_RE = re.compile(r'^\s*#\s*include\s*"([^"]+)"', re.M)


def _deps(src: Path, seen: set[Path] | None = None) -> set[Path]:
    """The source plus every local header it includes (transitively)."""
    seen = set() if seen is None else seen
    if src in seen or not src.exists():
        return seen
    seen.add(src)
    for name in _INCLUDE_RE.findall(src.read_text(errors="ignore")):
        _deps((src.parent / name).resolve(), seen)
    return seen


def _stale() -> bool:
    if not LIB.exists():
        return True
    lib_t = LIB.stat().st_mtime
    deps = set().union(*(_deps(s) for s in sources()))
    return any(p.stat().st_mtime > lib_t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    OBJ.mkdir(parents=True, exist_ok=True)
    cc = nvcc()
    def compile_one(src: Path) -> Path:
        obj = OBJ / (src.stem + ".o")
        deps_t = max(p.stat().st_mtime for p in _deps(src))
        if not force and obj.exists() and obj.stat().st_mtime > deps_t:
            return obj
        cmd = [cc, *ARCH, *NVCC_FLAGS, f"-I{INCLUDE}", "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stdout}\n{res.stderr}")
        if verbose and res.stderr.strip():
            print(res.stderr, flush=True)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as pool:
        objs = list(pool.map(compile_one, sources()))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    tmp.replace(LIB)
    return LIB


if __name__ == "__main__":
    out = build(force="--force" in sys.argv, verbose=True)
    print(out)
