"""Build the sm_100a shared library in-tree: paper_2603_20889_b200/libskinnyqr_b200.so.

nvcc cross-compiles without a GPU.  Objects go to paper_2603_20889_b200/build/ (git-ignored); the
.so stays in-tree so that it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libskinnyqr_b200.so"
OBJ = PKG / "build"
INCLUDE = PKG.parent / "include"
SOURCES = ["tsqr_thread_kernels.cu", "tsqr_fold_kernels.cu", "tsqr_mma_kernels.cu", "gram_kernels.cu", "gram_wide_kernels.cu", "gram_thread_kernels.cu", "small_kernels.cu", "matgen_kernels.cu", "capi.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-I", str(INCLUDE), "-I", str(CSRC),
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


# (8-column tiles, 8-row groups per panel, warps per CTA) instances of the DMMA TSQR kernel, one
# translation unit each (tsqr_mma_inst.cu) - keep in sync with SQB_MMA_CONFIGS in tsqr_mma_kernels.cu
MMA_CONFIGS = [(2, 16, 8), (3, 12, 8), (4, 10, 8), (5, 8, 8), (6, 6, 8), (7, 6, 8), (8, 6, 8)]


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))
    nvcc = _nvcc()
    jobs = []
    units = [(src, [], OBJ / (src[:-3] + ".o")) for src in SOURCES]
    units += [("tsqr_mma_inst.cu", [f"-DSQB_MMA_NB={nb}", f"-DSQB_MMA_RG={rg}", f"-DSQB_MMA_NW={nw}"],
               OBJ / f"tsqr_mma_{nb}_{rg}_{nw}.o") for nb, rg, nw in MMA_CONFIGS]
    for src, defs, obj in units:
        if force or _stale(obj, [CSRC / src] + headers):
            cmd = [nvcc] + NVCC_FLAGS + defs + (["-Xptxas", "-v"] if verbose else []) + ["-c", str(CSRC / src), "-o", str(obj)]
            jobs.append(cmd)
    if jobs:
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            for res in ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs):
                if verbose or res.returncode != 0:
                    sys.stderr.write(res.stdout + res.stderr)
                if res.returncode != 0:
                    raise RuntimeError("nvcc failed: " + " ".join(res.args))
    objs = [str(obj) for _, _, obj in units]
    if force or jobs or _stale(OUT, objs):
        cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(OUT)] + objs + ["-ldl"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("link failed")
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
