"""Build libsgpu.so (the CUDA engine) in-tree for sm_100a with nvcc.

    python -m paper_1712_04495_b200.build [--force]

The shared library lands next to this file so it travels with the repo
snapshot to the GPU box; no JIT cache, no torch extension machinery.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB_NAME = "libsgpu.so"
LIB_PATH = os.path.join(HERE, LIB_NAME)

SOURCES = ["sgpu_sim.cu", "sgpu_lane.cu", "sgpu_octet.cu", "sgpu_lane256.cu", "sgpu_proglane.cu", "sgpu_aux.cu",
           "sgpu_abi.cu"]
DEPS = SOURCES + ["sgpu_common.cuh", "sgpu_internal.h", "sgpu_tracesim.cuh", "sgpu_lanesim.cuh",
                  "sgpu_proglanesim.cuh", "sgpu_warpsort.cuh", "sgpu_stage256.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",          # no FMA contraction: float results follow the reference's op order
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-Xcompiler", "-pthread",
    "-shared", "--threads", "0",
]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libsgpu.so")


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(INCLUDE, "sgpu.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB_PATH,
          defines: tuple[str, ...] = ()) -> str:
    if not force and out == LIB_PATH and not _stale():
        return LIB_PATH
    tmp = out + f".tmp{os.getpid()}"
    cmd = [nvcc_path(), *NVCC_FLAGS, "-I", INCLUDE, *[f"-D{d}" for d in defines], "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES]]
    t0 = time.time()
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)
    if verbose:
        print(f"built {out} in {time.time() - t0:.1f}s", file=sys.stderr)
    return out


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--out", default=LIB_PATH)
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    build(force=a.force, verbose=True, out=a.out, defines=tuple(a.defines))
