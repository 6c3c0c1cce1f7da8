"""Build librichgpu.so (sm_100a) in-tree with nvcc.

Every csrc/*.cu is compiled in parallel to an object file and linked into
paper_2412_08076_b200/librichgpu.so with the CUDA runtime linked statically,
so the library has no dependency on the runtime torch ships.  Flags:

  -gencode arch=compute_100a,code=sm_100a   B200 only, no PTX fallback
  --fmad=false                              no FMA contraction: bitwise parity
                                            with SciPy/NumPy
  -lineinfo                                 ncu source page

Usage: python -m paper_2412_08076_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import re
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OBJ = PKG / "build" / ("obj" + os.environ.get("RICHGPU_LIB_NAME", ""))
LIB = PKG / os.environ.get("RICHGPU_LIB_NAME", "librichgpu.so")
EXTRA = os.environ.get("RICHGPU_NVCC_FLAGS", "").split()
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC",
          "-Xptxas", "-v", f"-I{INCLUDE}"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build librichgpu")


def _deps_mtime() -> float:
    files = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return max(f.stat().st_mtime for f in files)


def _includes(path: Path, seen=None) -> set:
    """Local headers a source includes, transitively (#include "...")."""
    seen = set() if seen is None else seen
    for line in path.read_text().splitlines():
        m = re.match(r'\s*#include\s+"([^"]+)"', line)
        if m:
            h = (path.parent / m.group(1)).resolve()
            if h.exists() and h not in seen:
                seen.add(h)
                _includes(h, seen)
    return seen


def _stale(src: Path) -> bool:
    """Object missing or older than its source or any header it includes."""
    obj = OBJ / (src.stem + ".o")
    if not obj.exists() or not obj.with_suffix(".log").exists():
        return True
    newest = max([src.stat().st_mtime] + [h.stat().st_mtime for h in _includes(src)])
    return obj.stat().st_mtime < newest


def _compile(src: Path, force: bool) -> tuple[Path, str]:
    """Compile one source unless its object is up to date; returns (object,
    ptxas log of that object)."""
    obj = OBJ / (src.stem + ".o")
    if not force and not _stale(src):
        return obj, obj.with_suffix(".log").read_text()
    cmd = [nvcc(), *ARCH, *CFLAGS, *EXTRA, "-c", str(src), "-o", str(obj)]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{p.stderr}")
    obj.with_suffix(".log").write_text(p.stderr)
    return obj, p.stderr


def ptxas_summary(log: str) -> list[tuple[str, int, int]]:
    """(kernel, registers, spill bytes) per entry function in a -Xptxas -v log."""
    out, name = [], None
    for line in log.splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            name = m.group(1)
            spill = 0
            continue
        m = re.search(r"(\d+) bytes spill stores", line)
        if m and name:
            spill = int(m.group(1))
        m = re.search(r"Used (\d+) registers", line)
        if m and name:
            out.append((name, int(m.group(1)), spill))
            name = None
    return out


def build(force: bool = False, verbose: bool = False) -> Path:
    if LIB.exists() and not force and LIB.stat().st_mtime >= _deps_mtime():
        return LIB
    OBJ.mkdir(parents=True, exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu"))
    flags = OBJ / ".flags"
    force = force or not flags.exists() or flags.read_text() != " ".join(EXTRA)
    logs = []
    with cf.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = []
        for obj, log in ex.map(lambda s: _compile(s, force), srcs):
            objs.append(obj)
            logs.append(log)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-cudart", "static",
           *map(str, objs), "-o", str(tmp)]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"link failed:\n{p.stderr}")
    os.replace(tmp, LIB)
    flags.write_text(" ".join(EXTRA))
    log = "\n".join(logs)
    (PKG / "build" / "ptxas.log").write_text(log)
    if verbose:
        for name, regs, spill in ptxas_summary(log):
            print(f"{regs:4d} regs {spill:5d} B spill  {name}")
    return LIB


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args(argv)
    lib = build(force=a.force, verbose=a.verbose)
    print(lib)
    return 0


if __name__ == "__main__":
    sys.exit(main())
