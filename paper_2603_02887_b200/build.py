"""Build libnxs.so (the C-ABI CUDA library) in-tree for sm_100a.

    python -m paper_2603_02887_b200.build [--force]

Each ``csrc/*.cu`` is compiled to an object with nvcc
(``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo``; ``project.cu``
additionally with ``--fmad=false`` so its fp64 projection/binning is
reproducible bit-for-bit by ``oracle/binning_oracle.c``) and linked, with
the CUDA runtime static, into ``paper_2603_02887_b200/lib/libnxs.so``.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libnxs.so"
INCLUDE = PKG.parent / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", str(INCLUDE),
          "--expt-relaxed-constexpr", "-Xptxas", "-v"]
PER_FILE = {
    "project.cu": ["--fmad=false"],
}


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _deps():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [INCLUDE / "nxs.h"]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in _deps())


def _compile(src: Path, objdir: Path, log: list, extra=()) -> Path:
    obj = objdir / (src.stem + ".o")
    cmd = [NVCC, *ARCH, *COMMON, *PER_FILE.get(src.name, []), *extra, "-c", str(src), "-o",
           str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log.append((src.name, res.stderr))
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> Path:
    """Build lib/libnxs.so; ``variant`` builds lib/libnxs_<variant>.so with
    extra ``-D`` defines instead (kernel experiments, loaded via NXS_LIB)."""
    out = LIBDIR / f"libnxs_{variant}.so" if variant else LIB
    if not variant and not force and not _stale():
        return LIB
    objdir = PKG / ("build_obj" + (f"_{variant}" if variant else ""))
    objdir.mkdir(exist_ok=True)
    LIBDIR.mkdir(exist_ok=True)
    log: list = []
    extra = [f"-D{d}" for d in defines]
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, objdir, log, extra), _sources()))
    tmp = out.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, out)
    if verbose:
        for name, err in log:
            print(f"== {name}\n{err}")
    return out


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv, variant=var, defines=defs)
    print(p)
