"""Build a variant of the library for tools/kernel_sweep.py.
    python tools/build_variant.py NAME [-DFOO=1 ...]   ->  sweep/lib_NAME.so"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_05455_b200 import build as B
os.makedirs(os.path.join(B.ROOT, "sweep"), exist_ok=True)
out = os.path.join(B.ROOT, "sweep", f"lib_{sys.argv[1]}.so")
subprocess.run([B.NVCC, *B.FLAGS, *sys.argv[2:], "-o", out, *B.SRC], check=True)
print(out)
