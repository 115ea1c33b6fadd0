"""Build libswings.so (all csrc/*.cu) for sm_100a with nvcc, in-tree.

The library is written next to the package (``paper_2409_07759_b200/lib/``)
so it travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libswings.so"
OBJ_DIR = PKG.parent / "build" / "obj"
# the checked variant: same sources with -DSS_CHECKED, device-side bounds /
# invariant checks (SS_DCHECK in ss_common.cuh) that trap on violation --
# the in-house stand-in for compute-sanitizer's memcheck (closed on the GPU
# pool); tests/test_gpu_checked.py runs scenes through it
VARIANTS = {"": (LIB, OBJ_DIR, []),
            "checked": (LIB_DIR / "libswings_checked.so", PKG.parent / "build" / "obj_checked",
                        ["-DSS_CHECKED"])}

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
] + os.environ.get("SS_NVCC_EXTRA", "").split()  # developer knob: extra -D for experiments


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _deps():
    return sorted(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "swings.h"]


def needs_build(variant: str = "") -> bool:
    lib = VARIANTS[variant][0]
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    return any(p.stat().st_mtime > t for p in _sources() + _deps())


def build(force: bool = False, verbose: bool = False, variant: str = "") -> Path:
    lib, obj_dir, extra = VARIANTS[variant]
    if not force and not needs_build(variant):
        return lib
    obj_dir.mkdir(parents=True, exist_ok=True)
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    cc = nvcc()
    dep_t = max(p.stat().st_mtime for p in _deps())

    def compile_one(src: Path) -> Path:
        obj = obj_dir / (src.stem + ".o")
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, dep_t):
            cmd = [cc, *NVCC_FLAGS, *extra, "-c", str(src), "-o", str(obj)]
            if verbose:
                print(" ".join(cmd))
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stdout}\n{r.stderr}")
            if verbose and (r.stdout or r.stderr):
                print(r.stdout, r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [cc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *map(str, objs),
           "-o", str(tmp), "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import sys

    print(build(force="--force" in sys.argv, verbose=True,
                variant="checked" if "--checked" in sys.argv else ""))
