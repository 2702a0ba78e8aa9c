"""Build libmdb200.so in-tree with nvcc for sm_100a (B200) only.

Used by __graft_entry__.build() and by `python -m paper_1711_00705_b200._build`.
The shared library is written next to this file so it travels with the repo
snapshot to the GPU box (gpurun copies built .so files).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libmdb200.so"
SOURCES = ["md_elementwise.cu", "md_allreduce.cu", "md_ar_tree.cu", "md_ar_direct.cu", "md_ar_push.cu",
           "md_dimd.cu", "md_toy.cu"]
HEADERS = ["md_common.cuh", "md_allreduce.cuh", "../../include/mdb200.h"]

NVCC_FLAGS = [
    "-std=c++17",
    "-O3",
    "-gencode",
    "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    # never contract a*b+c into an FMA: the reference rounds every op
    # (pkg/setup.py:31-32, -ffp-contract=off); kernels also use __f*_rn
    "-fmad=false",
    "-Xcompiler",
    "-fPIC",
    "-Xptxas",
    "-v",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not LIB.exists():
        return True
    lib_t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + [CSRC / h for h in HEADERS]
    return any(p.stat().st_mtime > lib_t for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    # one nvcc per translation unit, in parallel, then a host link
    procs = []
    for s in SOURCES:
        obj = objdir / (Path(s).stem + ".o")
        cmd = [_nvcc(), *NVCC_FLAGS, "-c", "-o", str(obj), str(CSRC / s)]
        procs.append((obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                            text=True)))
    log_text, failed = "", False
    for obj, p in procs:
        out, _ = p.communicate()
        log_text += out
        failed |= p.returncode != 0
    log = PKG / "build_ptxas.log"
    if not failed:
        res = subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                              "-o", str(tmp), *[str(o) for o, _ in procs]],
                             capture_output=True, text=True)
        log_text += res.stdout + res.stderr
        failed = res.returncode != 0
    log.write_text(log_text)
    if failed:
        sys.stderr.write(log_text)
        raise RuntimeError(f"nvcc failed; see {log}")
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
