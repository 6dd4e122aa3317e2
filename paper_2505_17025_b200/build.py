"""Build the CUDA extension (C-ABI shared library) in-tree for sm_100a.

    python -m paper_2505_17025_b200.build

produces paper_2505_17025_b200/_lib/libnhswe_b200.so.  nvcc cross-compiles
without a GPU, so this runs in the CPU container too.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libnhswe_b200.so")
SOURCES = ["capi.cu", "step_kernel.cu", "aux_kernels.cu", "stream_kernels.cu", "stream_kp.cu",
           "pm_kernels.cu"]
HEADERS = ["nh_common.cuh", "bathy.cuh", "physics.cuh", "tree.cuh", "step_kernel.cuh",
           "stream_kernels.cuh", "stream_kp.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "--extended-lambda", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
# default build: reference-faithful arithmetic (NH_STRICT=1, no implicit FMA contraction);
# "fast" builds drop both (see csrc/nh_common.cuh)
STRICT_FLAGS = ["-DNH_STRICT=1"]
FAST_FLAGS = ["-DNH_STRICT=0", "-fmad=true"]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "nhswe_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = (), fast: bool = False) -> str:
    lib = out or LIB
    if not force and out is None and not _stale():
        return LIB
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:   # one nvcc per source, concurrently
        obj = os.path.join(os.path.dirname(lib), src.replace(".cu", ".o"))
        cmd = [_nvcc(), *NVCC_FLAGS, *(FAST_FLAGS if fast else STRICT_FLAGS),
               *[f"-D{d}" for d in defines], "-c",
               os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                            text=True)))
        objs.append(obj)
    for src, p in procs:
        out, err = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out}\n{err}")
        if verbose:
            sys.stderr.write(err)
    tmp = lib + ".tmp"
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           *objs, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
