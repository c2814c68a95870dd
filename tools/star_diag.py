import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2303_05455_b200 as P
import oracle as O
from oracle.ivhd_oracle import OracleRun
for m in (2000, 20000):
    nb = np.zeros((m, 2), dtype=np.int32); nb[:, 1] = (np.arange(m) + 1) % m; nb[0] = [1, 2]
    cfg = dict(nn=2, rn=1, c=0.01, seed=3)
    r0 = P.run_embedding(graph=P.KnnGraph(nb), config=P.EmbeddingConfig(iterations=0, **cfg))
    ref = OracleRun(nb, iterations=1, **cfg)
    print(m, "y0 diff", np.abs(r0.embedding.points - ref.Y).max(), "rn equal", np.array_equal(r0.state.rn_assignments, ref.rn_assign))
    f = P.compute_forces(ref.Y, P.ConnectionSet(np.column_stack([ref.full.src, ref.full.dst]), ref.full.target, ref.full.rand), 0.01)
    fr = O.forces(ref.Y, ref.full, 0.01)
    err = np.abs(f - fr).max() / np.abs(fr).max()
    print(m, "force normwise", err, "worst row", np.abs(f - fr).max(axis=1).argmax(), "hub f", f[0], fr[0])
    for it in (1, 2, 3):
        r = P.run_embedding(graph=P.KnnGraph(nb), config=P.EmbeddingConfig(iterations=it, **cfg))
        rr = OracleRun(nb, iterations=it, **cfg); rr.run()
        print("  it", it, np.abs(r.embedding.points - rr.Y).max() / np.abs(rr.Y).max(), r.trace.step_size, rr.trace_b)
