"""Build recipe for libivhd_b200.so (sm_100a only).

    python -m paper_2303_05455_b200.build [--force]

nvcc compiles csrc/ivhd_capi.cu (which includes the kernels in
csrc/ivhd_step.cuh) into an in-tree shared library; the .so travels with the
repository snapshot to the GPU box.
"""

import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", f) for f in
       ("ivhd_capi.cu", "ivhd_kern_d2.cu", "ivhd_kern_d3.cu", "ivhd_knn.cu", "ivhd_metrics.cu")]
DEPS = SRC + [os.path.join(HERE, "csrc", f) for f in
              ("ivhd_step.cuh", "ivhd_step_f64.cuh", "ivhd_kernels.h", "ivhd_rng.cuh")] + [
    os.path.join(ROOT, "include", "ivhd_b200.h")]
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
    """Compile every translation unit in parallel (the step-kernel
    instantiations are split by target_dim), then link the shared library."""
    if not force and not stale():
        return OUT
    cflags = [f for f in FLAGS if f != "-shared"]
    with tempfile.TemporaryDirectory(prefix="ivhd_build_") as tmp:
        jobs = []
        for src in SRC:
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            cmd = [NVCC, *cflags, *(["-Xptxas", "-v"] if verbose else []), "-c", "-o", obj, src]
            jobs.append((subprocess.Popen(cmd), obj, src))
        failed = [src for proc, _, src in jobs if proc.wait() != 0]
        if failed:
            raise subprocess.CalledProcessError(1, f"nvcc {failed}")
        subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT + ".tmp",
                        *(obj for _, obj, _ in jobs)], check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
