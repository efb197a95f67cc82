"""Build libcmb200.so in-tree with nvcc for sm_100a.

    python -m paper_2105_12301_b200.build_native [--verbose]

Objects go to paper_2105_12301_b200/_build/, the shared library to
paper_2105_12301_b200/libcmb200.so (git-ignored, shipped to the GPU box by
gpurun with the rest of the tree).  ptxas resource usage is written to
_build/ptxas.log.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libcmb200.so"
SOURCES = ["knn_sweep.cu", "knn_w_a.cu", "knn_w_b.cu", "knn_w_c.cu", "knn_w_d.cu", "knn_w_e.cu",
           "knn_t_a.cu", "knn_t_b.cu", "knn_t_c.cu", "knn_t_d.cu",
           "lookup.cu", "lookup_r16_4_12.cu", "lookup_r16_13_20.cu", "lookup_r16_21_31.cu", "lookup_nr.cu", "lookup_h16.cu", "lookup_w12.cu", "lookup_w8.cu", "utils.cu", "convergence.cu", "io.cu", "cmb_api.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", f"-I{CSRC}"]
if os.environ.get("CMB_NR_WARPS"):  # A/B builds: CTA warps of the non-resident lookup
    FLAGS.append("-DCMB_NR_WARPS=" + os.environ["CMB_NR_WARPS"])
if os.environ.get("CMB_STATS") == "1":  # selection counters in diagnostics[3..5] (profiling builds only)
    FLAGS.append("-DCMB_KNN_STATS")


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src, *CSRC.glob("*.cuh"), ROOT / "include" / "cmb200.h", Path(__file__)]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    cc = nvcc()
    jobs = []
    for name in SOURCES:
        src = CSRC / name
        obj = BUILD / (src.stem + ".o")
        if force or _stale(obj, src):
            jobs.append((src, obj))

    def compile_one(job):
        src, obj = job
        cmd = [cc, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
        return src.name, r.stderr

    logs = []
    if jobs:
        with ThreadPoolExecutor(max_workers=len(jobs)) as pool:
            logs = list(pool.map(compile_one, jobs))
        with open(BUILD / "ptxas.log", "w") as fh:
            for name, text in logs:
                fh.write(f"==== {name}\n{text}\n")
                if verbose:
                    print(text)
    objs = [str(BUILD / (Path(s).stem + ".o")) for s in SOURCES]
    if jobs or not LIB.exists():
        cmd = [cc, *ARCH, "-shared", "-o", str(LIB), *objs, "-cudart", "static",
               "-Xcompiler", "-fPIC"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    p = build(verbose="--verbose" in sys.argv, force="--force" in sys.argv)
    print(p)
