"""Build libnw.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import re
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libnw.so")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "-DNW_BUILD"]


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps_mtime():
    return max(os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC)) if os.listdir(CSRC) else 0


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


_INC = re.compile(r'^\s*#\s*include\s+"([^"]+)"', re.M)


def _deps(path: str, seen=None) -> set:
    """Local headers a source includes, recursively (quoted includes under csrc/ and include/)."""
    seen = set() if seen is None else seen
    for name in _INC.findall(open(path).read()):
        for d in (os.path.dirname(path), CSRC, os.path.join(os.path.dirname(HERE), "include")):
            h = os.path.normpath(os.path.join(d, name))
            if os.path.exists(h):
                if h not in seen:
                    seen.add(h)
                    _deps(h, seen)
                break
    return seen


def _stale(src: str, headers_mtime: float) -> bool:
    """An object is rebuilt when its .cu, a header it includes (recursively) or this script is
    newer than it."""
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    path = os.path.join(CSRC, src)
    newest = max([os.path.getmtime(path), os.path.getmtime(__file__)] + [os.path.getmtime(h) for h in _deps(path)])
    return newest > t


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the stale csrc/*.cu objects and link libnw.so; skipped when up to date."""
    os.makedirs(BUILD, exist_ok=True)
    hdr = os.path.join(os.path.dirname(HERE), "include", "nw.h")
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hmt = max([os.path.getmtime(h) for h in headers] + [os.path.getmtime(hdr), os.path.getmtime(__file__)])
    srcs = sources()
    todo = srcs if force else [s for s in srcs if _stale(s, hmt)]
    with cf.ThreadPoolExecutor(max_workers=max(1, min(16, len(todo)))) as ex:
        list(ex.map(lambda s: _compile(s, verbose), todo))
    objs = [os.path.join(BUILD, s.replace(".cu", ".o")) for s in srcs]
    # per-object staleness decides what compiles; the library relinks when any object is newer
    if not todo and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
