"""Time the GPU rank-curve pass (evaluate_embedding) at C1 / C2 shapes.

    python tools/curves_bench.py [m] [n]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2303_05455_b200 import metrics  # noqa: E402


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 784
    rng = np.random.default_rng(0)
    c = rng.standard_normal((10, n))
    lab = rng.integers(0, 10, m)
    X = c[lab] + 1.5 * rng.standard_normal((m, n))
    Y = X[:, :2] + 0.5 * rng.standard_normal((m, 2))
    metrics.evaluate_embedding(X[:2000], Y[:2000], labels=lab[:2000])  # warm-up (context, module load)
    for _ in range(2):
        t = time.perf_counter()
        cur = metrics.evaluate_embedding(X, Y, labels=lab)
        dt = time.perf_counter() - t
        print(f"m={m} n={n} k_max={len(cur.k)} evaluate_embedding {dt:.3f} s  {cur.summary()}", flush=True)


if __name__ == "__main__":
    main()
