"""Build recipe for libivhd_b200.so (sm_100a only).

    python -m paper_2303_05455_b200.build [--force]

nvcc compiles csrc/ivhd_capi.cu (which includes the kernels in
csrc/ivhd_step.cuh) into an in-tree shared library; the .so travels with the
repository snapshot to the GPU box.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "ivhd_capi.cu"), os.path.join(HERE, "csrc", "ivhd_knn.cu"),
       os.path.join(HERE, "csrc", "ivhd_metrics.cu")]
DEPS = SRC + [os.path.join(HERE, "csrc", "ivhd_step.cuh"), os.path.join(HERE, "csrc", "ivhd_rng.cuh"), os.path.join(ROOT, "include", "ivhd_b200.h")]
OUT = os.path.join(HERE, "libivhd_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include")]


def stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force=False, verbose=False):
    if not force and not stale():
        return OUT
    cmd = [NVCC, *FLAGS, *(["-Xptxas", "-v"] if verbose else []), "-o", OUT + ".tmp", *SRC]
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
