"""Builds the reference-side adapter (integration/smc_b200.cpp) and its callers
(integration/model_select_b200.cpp; the CLI integration/specmc_b200_cli.cpp,
fit and model-select on the B200 backend) against the REFERENCE's own headers
(/root/reference/proj/include; Eigen3 is absent here, so oracle/eigen_shim
stands in) and the reference sources the caller needs (model, synthetic,
posterior, report, ...), linked to this repo's libspecmc_b200.so.  Output:
oracle/_ref/model_select_b200 and oracle/_ref/specmc_b200 (git-ignored, travels to the GPU box with the
snapshot; /root/reference does not exist there).  Never copies reference
sources: it compiles them where they lie.
"""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = Path("/root/reference/proj")
OUT = ROOT / "oracle" / "_ref" / "model_select_b200"
CLI = ROOT / "oracle" / "_ref" / "specmc_b200"
REF_SOURCES = ["priors", "model", "energy", "mcmc", "smc", "spectrum", "report", "synthetic", "posterior", "remc",
               "bench", "config"]


def _compile(out: Path, main_src: Path, force: bool) -> Path:
    lib = ROOT / "paper_2604_03271_b200" / "libspecmc_b200.so"
    srcs = [ROOT / "integration" / "smc_b200.cpp", main_src]
    refs = [REF / "src" / f"{s}.cpp" for s in REF_SOURCES]
    deps = srcs + refs + [ROOT / "integration" / "smc_b200.hpp", ROOT / "include" / "specmc_b200.h"]
    if not force and out.exists() and all(p.stat().st_mtime <= out.stat().st_mtime for p in deps):
        return out
    out.parent.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-pthread", f"-I{ROOT / 'oracle' / 'eigen_shim'}", f"-I{REF / 'include'}",
           f"-I{ROOT / 'include'}", f"-I{ROOT / 'integration'}", f'-DSPECMC_DATA_DIR="{REF / "data"}"',
           *map(str, srcs + refs), str(lib), "-Wl,-rpath,$ORIGIN/../../paper_2604_03271_b200", "-o", str(out)]
    subprocess.run(cmd, check=True)
    return out


def build(force: bool = False) -> Path | None:
    """Builds oracle/_ref/model_select_b200 and the CLI oracle/_ref/specmc_b200;
    returns the former (None when neither can be built)."""
    if not REF.exists():
        return OUT if OUT.exists() else None
    _compile(CLI, ROOT / "integration" / "specmc_b200_cli.cpp", force)
    return _compile(OUT, ROOT / "integration" / "model_select_b200.cpp", force)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
