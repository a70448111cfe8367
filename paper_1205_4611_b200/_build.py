"""Build libfmm2d.so in-tree with nvcc for sm_100a (no JIT cache, no torch).

The shared library travels to the GPU box with the repo snapshot; this
module is invoked by ``__graft_entry__.build()`` and by ``python -m
paper_1205_4611_b200._build``.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libfmm2d.so"
OBJ = PKG / "_obj"
SOURCES = ["scan.cu", "tree.cu", "connect.cu", "expansions.cu", "nearfield.cu", "fmm2d.cu",
           "operators.cu",
           "dist.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo",
    "-Xcompiler", "-fPIC,-O2",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libfmm2d.so")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), out: Path | None = None) -> Path:
    """Compile and link libfmm2d.so.  ``defines``/``out`` build an A/B variant
    (e.g. ``-DP2P_UNROLL=4``) into its own object directory and library."""
    nvcc = _nvcc()
    obj_dir = OBJ if not defines else PKG.parent / "build" / "ab" / ("obj_" + Path(out).stem)
    lib_out = OUT if out is None else Path(out)
    obj_dir.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [PKG.parent / "include" / "fmm2d.h"]
    jobs = []
    for src in SOURCES:
        obj = obj_dir / (Path(src).stem + ".o")
        if force or _stale(obj, [CSRC / src, *headers]):
            cmd = [nvcc, *NVCC_FLAGS, *defines, "-c", str(CSRC / src), "-o", str(obj)]
            jobs.append((src, cmd))
    with cf.ThreadPoolExecutor(max_workers=len(jobs) or 1) as pool:
        futs = {pool.submit(subprocess.run, cmd, capture_output=True, text=True): src
                for src, cmd in jobs}
        for fut in cf.as_completed(futs):
            res = fut.result()
            if verbose or res.returncode:
                sys.stderr.write(res.stdout + res.stderr)
            if res.returncode:
                raise RuntimeError(f"nvcc failed on {futs[fut]}")
    objs = [obj_dir / (Path(s).stem + ".o") for s in SOURCES]
    if force or jobs or _stale(lib_out, objs):
        lib_out.parent.mkdir(parents=True, exist_ok=True)
        tmp = lib_out.with_suffix(".so.tmp")
        cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
               "-o", str(tmp), *map(str, objs)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("link of libfmm2d.so failed")
        os.replace(tmp, lib_out)
    return lib_out


if __name__ == "__main__":
    # python -m paper_1205_4611_b200._build [-v] [-f] [--variant NAME -DX=1 ...]
    args = sys.argv[1:]
    if "--variant" in args:
        i = args.index("--variant")
        name = args[i + 1]
        defs = [a for a in args[i + 2:] if a.startswith("-D")]
        print(build(verbose="-v" in args, defines=defs,
                    out=PKG.parent / "build" / "ab" / f"libfmm2d_{name}.so"))
    else:
        print(build(verbose="-v" in args, force="-f" in args))
