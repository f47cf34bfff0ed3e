"""Build recipe of the product library (nvcc, sm_100a, in-tree).

Compiles paper_2604_03271_b200/csrc/{kernels,host}.cu into
paper_2604_03271_b200/libspecmc_b200.so with
``-gencode arch=compute_100a,code=sm_100a -lineinfo``.  The .so is
git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
LIB = Path(os.environ["SPECMC_OUT"]) if os.environ.get("SPECMC_OUT") else PKG / "libspecmc_b200.so"
DEFS = os.environ.get("SPECMC_DEFS", "").split()  # -D... tuning variants (A/B builds)
SOURCES = sorted(CSRC.glob("*.cu"))
HEADERS = [CSRC / "device.cuh", CSRC / "chain.cuh", CSRC / "launch.h", ROOT / "include" / "specmc_b200.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--use_fast_math",
         "-Xptxas", "-warn-spills", f"-I{ROOT / 'include'}"]


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    objs = []
    procs = []
    for src in SOURCES:
        obj = CSRC / (src.stem + (".v" + str(abs(hash(tuple(DEFS)))) if DEFS else "") + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *DEFS, "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True), src))
        objs.append(obj)
    failed = False
    for p, src in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out)
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed")
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.run([NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart", "-ldl"], check=True)
    os.replace(tmp, LIB)
    for o in objs:
        o.unlink(missing_ok=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
