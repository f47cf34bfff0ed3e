"""Build recipes for the parity checker (TEST INFRASTRUCTURE ONLY).

* ``build_port()``  compiles oracle/specmc_oracle.c (the C restatement of the
  reference hot path) into oracle/liboracle.so.
* ``build_ref()``   compiles the UNCHANGED reference sources from
  /root/reference/proj/src against oracle/eigen_shim plus oracle/ref_driver.cpp
  into oracle/_ref/libspecmc_ref.so.  Only possible where /root/reference
  exists (this container); the built .so travels to the GPU box with the repo
  snapshot (git-ignored, not gpurun-ignored).

Both use ``-ffp-contract=off`` so that the restatement and the reference agree
bit for bit (no compiler-chosen FMA contraction on either side).
"""
from __future__ import annotations

import os
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_ROOT = Path("/root/reference/proj")
PORT_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libspecmc_ref.so"

# reference translation units on the SMC path (+ the synthetic generators,
# model selection, and the benchmark harness with the REMC comparator it
# tabulates, used by the parity tests); config/CLI are out of scope
REF_SOURCES = ["priors", "model", "energy", "mcmc", "smc", "spectrum", "report", "synthetic", "posterior", "remc", "bench"]

COMMON = ["-O3", "-march=x86-64-v2", "-ffp-contract=off", "-fPIC", "-shared"]

# Timing builds of the same reference sources (bench.py's reference arm and
# cpu_baseline): the reference's own Release flags (proj/CMakeLists.txt:8-10,
# :33-35: -O3 -DNDEBUG -march=native, gnu++20 with GCC's default FMA
# contraction) for the two ISA levels a GPU box's host can have; bench.py picks
# the one its CPU supports (the box cannot rebuild: /root/reference is absent
# there).  The -ffp-contract=off build above stays the bit-exact parity target.
NATIVE_VARIANTS = {"x86-64-v4": HERE / "_ref" / "libspecmc_ref_v4.so",
                   "x86-64-v3": HERE / "_ref" / "libspecmc_ref_v3.so"}


def _newer(out: Path, inputs) -> bool:
    if not out.exists():
        return False
    t = out.stat().st_mtime
    return all(Path(i).stat().st_mtime <= t for i in inputs)


def build_port(force: bool = False) -> Path:
    src = HERE / "specmc_oracle.c"
    if force or not _newer(PORT_SO, [src]):
        cmd = ["gcc", "-std=gnu11", *COMMON, str(src), "-o", str(PORT_SO), "-lm"]
        subprocess.run(cmd, check=True)
    return PORT_SO


def build_ref(force: bool = False) -> Path | None:
    """Returns the .so path, or None when the reference tree is absent."""
    if not REF_ROOT.exists():
        return REF_SO if REF_SO.exists() else None
    srcs = [REF_ROOT / "src" / f"{s}.cpp" for s in REF_SOURCES] + [HERE / "ref_driver.cpp"]
    shim = HERE / "eigen_shim" / "Eigen" / "Dense"
    if force or not _newer(REF_SO, srcs + [shim]):
        REF_SO.parent.mkdir(parents=True, exist_ok=True)
        cmd = [
            "g++", "-std=c++20", *COMMON, "-pthread",
            f"-I{HERE / 'eigen_shim'}", f"-I{REF_ROOT / 'include'}",
            f'-DSPECMC_DATA_DIR="{REF_ROOT / "data"}"',
            *map(str, srcs), "-o", str(REF_SO),
        ]
        subprocess.run(cmd, check=True)
    for march, out in NATIVE_VARIANTS.items():
        if force or not _newer(out, srcs + [shim]):
            cmd = ["g++", "-std=gnu++20", "-O3", "-DNDEBUG", f"-march={march}", "-fPIC", "-shared", "-pthread",
                   f"-I{HERE / 'eigen_shim'}", f"-I{REF_ROOT / 'include'}",
                   f'-DSPECMC_DATA_DIR="{REF_ROOT / "data"}"', *map(str, srcs), "-o", str(out)]
            subprocess.run(cmd, check=True)
    return REF_SO


def timing_ref_so() -> tuple[Path, str]:
    """The reference timing build for this host's ISA (v4 needs AVX-512 F/BW/DQ/VL)."""
    flags = set()
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("flags"):
                flags = set(line.split(":", 1)[1].split())
                break
    except OSError:
        pass
    v4 = {"avx512f", "avx512bw", "avx512dq", "avx512vl"} <= flags
    v3 = {"avx2", "fma", "bmi2"} <= flags
    for march, ok in (("x86-64-v4", v4), ("x86-64-v3", v3)):
        if ok and NATIVE_VARIANTS[march].exists():
            return NATIVE_VARIANTS[march], march
    return REF_SO, "x86-64-v2 (parity build)"


if __name__ == "__main__":
    print(build_port(force=True))
    print(build_ref(force=True))
