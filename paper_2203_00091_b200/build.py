"""Build libdfss_sm100a.so in-tree with nvcc for sm_100a (no torch JIT cache).

    python -m paper_2203_00091_b200.build [--force]

Each .cu under csrc/ is compiled to an object (in parallel, skipped when up
to date) and linked into paper_2203_00091_b200/lib/libdfss_sm100a.so.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import re
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "lib", "obj")
LIB = os.path.join(PKG, "lib", "libdfss_sm100a.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the DFSS CUDA library cannot be built")


def _headers() -> list[str]:
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))


def _includes(src: str, seen: set | None = None) -> list[str]:
    """Files `src` pulls in with #include "..." (recursively, relative to its directory): an
    object is stale when any of them changed -- flash_tc_dump.cu includes flash_tc.cu."""
    seen = set() if seen is None else seen
    out = []
    try:
        text = open(src).read()
    except OSError:
        return out
    for m in re.finditer(r'^\s*#\s*include\s+"([^"]+)"', text, re.M):
        f = os.path.normpath(os.path.join(os.path.dirname(src), m.group(1)))
        if f not in seen and os.path.exists(f):
            seen.add(f)
            out.append(f)
            out += _includes(f, seen)
    return out


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _flags_stamp(obj: str) -> str:
    return obj + ".flags"


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
    # DFSS_NVCC_EXTRA: extra nvcc flags for bring-up builds (e.g. -DDFSS_FLASH_TRACE_BUILD)
    cmd = [nvcc(), *NVCC_FLAGS, *os.environ.get("DFSS_NVCC_EXTRA", "").split(), "-c", src, "-o", obj]
    # the object records the exact command it was built with: a flag change (a trace build
    # switched on or off) rebuilds it even when no source is newer
    stamp = " ".join(cmd)
    try:
        same_flags = open(_flags_stamp(obj)).read() == stamp
    except OSError:
        same_flags = False
    if force or not same_flags or _stale(obj, [src] + _headers() + _includes(src)):
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{res.stdout}\n{res.stderr}")
        if res.stderr.strip():
            sys.stderr.write(res.stderr)
        with open(_flags_stamp(obj), "w") as f:
            f.write(stamp)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), sources))
    if force or _stale(LIB, objs):
        cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
