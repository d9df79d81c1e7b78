"""Build the in-tree sm_100a shared library ``_lib/libblreg_b200.so``.

Compiles every ``csrc/*.cu`` with nvcc for ``sm_100a`` (``-lineinfo`` for ncu
source mapping), links cuFFT and a static CUDA runtime.  Runs on a CPU-only
box (nvcc cross-compiles).  Usage: ``python -m paper_1807_05117_b200.build``.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# experiments: BLR_OUT_DIR builds a variant library elsewhere (e.g. _lib/var_u6),
# loaded at run time through BLR_LIB_PATH (see _lib.py)
OUT_DIR = os.environ.get("BLR_OUT_DIR") or os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libblreg_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
                # the fp64 transforms are latency-bound: registers buy ILP (A/B: -0.7% HVP time)
                "-Xptxas", "--register-usage-level=10"]
# experiments: extra ptxas options, e.g. BLR_PTXAS="--register-usage-level=10"
if os.environ.get("BLR_PTXAS"):
    for _opt in os.environ["BLR_PTXAS"].split():
        FLAGS += ["-Xptxas", _opt]
# experiments: compile-time tuning macros, e.g. BLR_DEFINES="BLR_EPI_U=6 BLR_KPW=2"
if os.environ.get("BLR_DEFINES"):
    FLAGS += [f"-D{_d}" for _d in os.environ["BLR_DEFINES"].split()]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _newest_input():
    files = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    files.append(os.path.join(os.path.dirname(HERE), "include", "blreg_b200.h"))
    return max(os.path.getmtime(f) for f in files)


def up_to_date():
    return os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_input()


def build(force=False, verbose=True):
    if not force and up_to_date():
        return LIB
    if not os.path.exists(NVCC):
        raise RuntimeError(f"nvcc not found at {NVCC}")
    obj_dir = os.path.join(OUT_DIR, "obj")
    os.makedirs(obj_dir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
        cmd = [NVCC, *FLAGS, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        if verbose and r.stderr.strip():
            print(r.stderr.strip(), file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
           f"-L{CUDA}/lib64", "-lcufft", "-Xlinker", f"-rpath={CUDA}/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    shutil.rmtree(obj_dir, ignore_errors=True)
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
