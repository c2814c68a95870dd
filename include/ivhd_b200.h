/*
 * ivhd_b200.h — C ABI of the B200-native IVHD embedding loop.
 *
 * One context = one embedding run on one GPU (or one rank's shard of it).
 * Plain pointers and sizes only; every host pointer is read/written
 * synchronously before the call returns.  All functions return an
 * ivhd_status; on failure ivhd_last_error(ctx) (or ivhd_global_error() when
 * no context exists yet) holds a one-line message.
 *
 * The reference interface each entry point replaces (paths relative to
 * /root/reference/pkg/src/ivhd/):
 *
 *   ivhd_create / ivhd_destroy      _Run.__init__ device state       engine.py:162-221
 *   ivhd_set_graph                  _Run._build_edges (binary)       engine.py:225-262
 *   ivhd_set_graph_sampled          sample_random_neighbors + above  engine.py:132-146,225-262
 *   ivhd_init_positions             init_layout (same PCG64 stream)  engine.py:124-129
 *   ivhd_set_connections            ConnectionSet(...)               forces.py:20-50
 *   ivhd_set_positions              init_layout result / observer    engine.py:124-129,214
 *   ivhd_get_positions              RunResult.embedding.points       engine.py:413
 *   ivhd_set_optimizer              make_optimizer                   optim.py:249-256
 *   ivhd_set_step_size              _apply_mutation("b")             engine.py:424-432
 *   ivhd_run                        the loop body, n times           engine.py:346-384
 *   ivhd_compute_forces             compute_forces(..., with_stress) forces.py:139-181
 *   ivhd_stress                     stress                           forces.py:78-83
 *   ivhd_get_deltas                 EmbeddingState.deltas            engine.py:379
 *   ivhd_snapshot / ivhd_restore    (new) device-side checkpoint     SURVEY.md §5 checkpoint row
 *   ivhd_shard_* / ivhd_step_*      (new) vertex-range sharding
 *   ivhd_peer_*                     (new) fused NVLink P2P exchange
 *   ivhd_knn_build                  knng.build_exact_knn             knng.py:158-194
 *                                   (euclidean / cosine)
 *   ivhd_neighbor_hit               metrics.neighbor_hit (points)    metrics.py:254-294
 *   ivhd_curve_pass                 metrics._curve_pass (rnx/gnn/    metrics.py:149-182
 *                                   trust/continuity/evaluate)
 *   ivhd_rank_matrix                metrics.compute_ranks            metrics.py:103-146
 *   ivhd_pair_ranks                 metrics._pair_ranks (shepard_    metrics.py:335-352
 *                                   and_corank)
 *
 */
#ifndef IVHD_B200_H
#define IVHD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IVHD_ABI_VERSION 3

enum ivhd_status {
  IVHD_OK = 0,
  IVHD_ERR_INVALID_ARG = 1, /* -> InvalidArgumentError / DimensionMismatchError */
  IVHD_ERR_CUDA = 2,        /* CUDA runtime failure (message has the CUDA error) */
  IVHD_ERR_DIVERGED = 3,    /* -> NumericalDivergenceError(iteration, state)    */
  IVHD_ERR_STATE = 4,       /* call order violated (e.g. run before set_graph)  */
  IVHD_ERR_PEER = 5,        /* peer exchange: a rank did not arrive in time      */
  IVHD_PAUSED_DEGENERATE = 6 /* not an error: see ivhd_degenerate_pending         */
};

enum ivhd_norm { IVHD_NORM_L2 = 0, IVHD_NORM_L1 = 1 };

enum ivhd_optimizer_kind {
  IVHD_OPT_FORCE_DIRECTED = 0,
  IVHD_OPT_SGD = 1,
  IVHD_OPT_MOMENTUM = 2,
  IVHD_OPT_NESTEROV = 3,
  IVHD_OPT_ADAM = 4,
  IVHD_OPT_ADADELTA = 5
};

/* Mirrors IntegratorParams (optim.py:15-56) + OptimizerParams (optim.py:59-68).
 * step = b for force-directed, alpha for sgd/momentum/nesterov/adam,
 * scale for adadelta (optim.py:71-77 defaults already resolved by the host). */
typedef struct ivhd_optimizer_params {
  int32_t kind;        /* ivhd_optimizer_kind */
  int32_t auto_adapt;  /* force-directed: self-adapting b with rollback  */
  double step;         /* b / alpha / scale                               */
  double a;            /* friction retention                              */
  double tau;          /* adaption threshold (already tau_for(M))        */
  double gamma1, gamma2;
  double beta, gamma_v, gamma_s, rho, eps;
} ivhd_optimizer_params;

typedef struct ivhd_ctx ivhd_ctx;

int ivhd_abi_version(void);
const char* ivhd_global_error(void);

/* stream: a cudaStream_t (as integer) to launch on, or 0 for a private one. */
int ivhd_create(ivhd_ctx** out, int device, int64_t m, int dim, uint64_t stream);
int ivhd_destroy(ivhd_ctx* ctx);
const char* ivhd_last_error(const ivhd_ctx* ctx);

/* Binary-mode connections of slot (0 = main set, 1 = RNN-filtered set):
 * nn block (i, nn_ids[i*nn_stride + c]) for c < ncols, then rn block
 * (i, rn_ids[i*rn + r]); nn pairs target 0 weight 1, rn pairs target 1
 * weight c.  Builds the symmetrised CSR on the device. */
int ivhd_set_graph(ivhd_ctx* ctx, int slot, const int32_t* nn_ids, int64_t nn_stride,
                   int ncols, const int32_t* rn_ids, int rn);

/* numpy's default bit generator (PCG64) on the device.  rng[6] =
 * {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger} of the caller's
 * numpy PCG64 state; it is read and advanced in place exactly as the
 * reference's numpy draws advance it, so the caller's Generator can continue.
 *
 * init_positions: positions = gen.uniform(lo, hi, size=(m, dim)).
 * set_graph_sampled: rn partners per vertex = gen.integers(0, m, (m, rn)) with
 * the reference's row-major re-draw of picks equal to the row or one of its
 * nn ids, then the binary connection set of ivhd_set_graph.  picks_out
 * (m*rn, may be NULL) receives the partners. */
int ivhd_init_positions(ivhd_ctx* ctx, uint64_t* rng, double lo, double hi);
int ivhd_set_graph_sampled(ivhd_ctx* ctx, int slot, const int32_t* nn_ids, int64_t nn_stride,
                           int ncols, int rn, uint64_t* rng, int32_t* picks_out);

/* Generic connection set (edges (L,2) row-major).  targets/scale may be NULL
 * (NULL targets = binary: 0 for nn, 1 for random pairs). */
int ivhd_set_connections(ivhd_ctx* ctx, int slot, const int32_t* edges,
                         const uint8_t* is_random, const double* targets,
                         const double* scale, int64_t n_conn);

int ivhd_set_positions(ivhd_ctx* ctx, const double* y);      /* (m, dim) */
int ivhd_get_positions(ivhd_ctx* ctx, double* y_out);        /* (m, dim) */
int ivhd_get_deltas(ivhd_ctx* ctx, double* d_out);           /* (m, dim) */
/* Page-locked host buffers (cudaHostAlloc, portable) for result arrays: the
 * positions / deltas copies above run at full PCIe/C2C rate into them and need
 * no first-touch page faults.  No reference counterpart (host memory of the
 * arrays engine.py:379-413 returns). */
int ivhd_host_alloc(int device, uint64_t bytes, void** out);
int ivhd_host_free(void* p);
int ivhd_set_optimizer(ivhd_ctx* ctx, const ivhd_optimizer_params* p); /* resets state */
int ivhd_set_step_size(ivhd_ctx* ctx, double step);
int ivhd_get_step_size(ivhd_ctx* ctx, double* step_out);

/* Run n_iter loop iterations on slot with norm and random-pair weight c.
 * stress_out/step_out (length n_iter, may be NULL) receive the trace
 * (stress at the pre-step positions, step size after the step).
 * *done_out = iterations completed.  On IVHD_ERR_DIVERGED the positions are
 * the last finite ones and stress_out[*done_out] holds the diverging
 * iteration's stress (engine.py:373-377). */
int ivhd_run(ivhd_ctx* ctx, int slot, int norm, double c, int64_t n_iter,
             double* stress_out, double* step_out, int64_t* done_out);

/* Operator level: forces (m, dim) and stress at y (host array) on slot. */
int ivhd_compute_forces(ivhd_ctx* ctx, int slot, int norm, double c, const double* y,
                        double* forces_out, double* stress_out);
int ivhd_stress(ivhd_ctx* ctx, int slot, int norm, double c, const double* y,
                double* stress_out);

int ivhd_synchronize(ivhd_ctx* ctx);

/* Degenerate random pairs (forces.py:158-174: d == 0, t != 0 get a unit
 * direction drawn from run.rng, in connection order, magnitude w * t).  The
 * kernel looks each one up in a host-filled table; when an iteration meets
 * one without an entry, ivhd_run stops before committing it and returns
 * IVHD_PAUSED_DEGENERATE with *done_out = iterations completed (their trace
 * filled); ivhd_compute_forces returns it likewise.  The caller reads the
 * entries, draws the directions from the run's generator and resumes:
 *   ivhd_degenerate_pending(ctx, cap, &n, rows, entries)   row (caller's ids),
 *       entry index in that row: out-halves in connection order, then
 *       in-halves in connection order
 *   ivhd_set_degenerate(ctx, n, rows, entries, vecs)       vecs (n, dim) =
 *       +w*t*u for the connection's source row, -w*t*u for its destination row;
 *       valid for the paused iteration (or the next forces call) only. */
int ivhd_degenerate_pending(ivhd_ctx* ctx, int64_t cap, int64_t* n_out, int32_t* rows_out,
                            int32_t* entries_out);
int ivhd_set_degenerate(ivhd_ctx* ctx, int64_t n, const int32_t* rows, const int32_t* entries,
                        const double* vecs);

/* Device-side checkpoint of positions + optimizer state + control block
 * (restore is asynchronous on the context stream; used to restart a run
 * from identical initial conditions without host copies). */
int ivhd_snapshot(ivhd_ctx* ctx);
int ivhd_restore(ivhd_ctx* ctx);

/* ---- vertex-range sharding (one context per rank, full graph replicated) ----
 * A rank updates vertices [v_begin, v_end) (tile aligned, see
 * ivhd_tile_vertices), then the caller all-gathers the positions slice and
 * the tile partials (device pointers from ivhd_shard_buffers) and calls
 * ivhd_step_finalize, which reduces all tiles in a fixed order so every
 * rank takes the same commit/rollback decision. */
int ivhd_tile_vertices(ivhd_ctx* ctx, int64_t* tile_v_out, int64_t* n_tiles_out);
int ivhd_shard_set_range(ivhd_ctx* ctx, int64_t v_begin, int64_t v_end);
/* ybuf[2] = the two position buffers; floats_per_vertex = their row stride;
 * partials = double4 per tile; cur_out = index of the buffer holding the
 * current positions (the next step writes the other one). */
int ivhd_shard_buffers(ivhd_ctx* ctx, uint64_t* ybuf0, uint64_t* ybuf1,
                       int64_t* floats_per_vertex, uint64_t* partials, int* cur_out);
int ivhd_step_local(ivhd_ctx* ctx, int slot, int norm, double c);
int ivhd_step_finalize(ivhd_ctx* ctx, double* stress_out, double* step_out,
                       int* committed_out);

/* Asynchronous sharded loop (no host round trip per iteration; the caller
 * all-gathers between step and finalize on the context's stream):
 *   ivhd_shard_begin(ctx, slot, c, n, &cur, &ep) once per segment (syncs; cur =
 *                                                current buffer index; ep changes
 *                                                when captured launches go stale)
 *   n times: ivhd_shard_step(ctx, slot, norm, &buf)   local update -> buf
 *            <all-gather buf slices and the unit partials>
 *            ivhd_shard_finalize(ctx)                decision on the device
 *   ivhd_shard_end(ctx, stress[n], step[n], &done)   syncs; DIVERGED like ivhd_run
 * buf (device pointer, m_cap*floats_per_vertex floats) alternates by parity. */
int ivhd_shard_begin(ivhd_ctx* ctx, int slot, double c, int64_t n_iter, int* cur_out,
                     int64_t* epoch_out);
int ivhd_shard_step(ivhd_ctx* ctx, int slot, int norm, uint64_t* exchange_out);
int ivhd_shard_finalize(ivhd_ctx* ctx);
int ivhd_shard_end(ivhd_ctx* ctx, double* stress_out, double* step_out, int64_t* done_out);

/* Fused peer exchange over NVLink (sharded mode, one process per GPU on one
 * node, up to 8 ranks).  Replaces the per-iteration NCCL
 * all-gather: the step kernel stores every updated position straight into
 * the replica of each peer that gathers it (P2P stores overlap the update
 * tile by tile); the last block of each rank's step kernel reduces its
 * blocks' partials, stores the rank partial into every rank's partial array,
 * raises its arrival flag on every rank, waits for all ranks' flags and takes
 * the same decision on every rank (one launch per iteration).  Set-up, after ivhd_shard_set_range:
 *   ivhd_peer_export(ctx, world, rank, h)   moves the exchanged buffers to
 *       cudaMalloc memory and writes their CUDA IPC handles
 *       (IVHD_PEER_HANDLE_BYTES bytes) into h;
 *   every rank gathers all handles in rank order (e.g. all_gather_object);
 *   ivhd_peer_import(ctx, all)              opens the peers' buffers.
 * In-process (several contexts of one process, tests): ivhd_peer_export on
 * each, then ivhd_peer_import_local(ctx, ctxs) with the contexts in rank order.
 * Afterwards ivhd_run drives the whole exchange on the device (CUDA graphs of
 * one step launch per iteration, no host work per iteration).  In-process
 * peers (ivhd_peer_import_local) decide in a separate finalizer kernel instead:
 * ivhd_shard_step / ivhd_shard_finalize launch the two one at a time, so the
 * emulation can run every rank's step before any finalizer.  A rank that
 * does not arrive within 60 s makes the others fail with IVHD_ERR_PEER
 * instead of hanging. */
#define IVHD_PEER_HANDLE_BYTES 256
int ivhd_peer_export(ivhd_ctx* ctx, int world, int rank, uint8_t* handle_out);
int ivhd_peer_import(ivhd_ctx* ctx, const uint8_t* all_handles);
int ivhd_peer_import_local(ivhd_ctx* ctx, ivhd_ctx* const* ctxs);
/* The step kernel stores a position only into the replicas of the ranks that
 * gather it (halo masks from the connection sets).  At the end of a segment
 * ivhd_run completes the local replica (both position buffers) with every
 * peer's own range and then waits for all ranks (barrier = 1), so positions /
 * deltas read back on any rank are complete.  ivhd_peer_pull does the same
 * on demand; barrier = 0 skips the all-rank wait (in-process emulation, where
 * the ranks' kernels run one after another). */
int ivhd_peer_pull(ivhd_ctx* ctx, int barrier);
/* Position records this rank stores into peers per iteration (sum over its
 * vertices of the ranks that gather them) and their bytes. */
int ivhd_peer_halo(ivhd_ctx* ctx, int64_t* records_out, int64_t* bytes_out);
/* Peer failure detection: how long a rank waits for the others' arrival
 * flags (each iteration and at the segment-end barrier) before it gives up
 * with IVHD_ERR_PEER; default 60 s.  Call after ivhd_peer_import*. */
int ivhd_peer_set_timeout(ivhd_ctx* ctx, double seconds);

/* ---- diagnostics (new; no reference counterpart) ----------------------
 * Gather floor of a connection set: a pass that streams the slot's column
 * ids and gathers every neighbour position (the step kernel's only random
 * traffic) with nothing else — no arithmetic, no update, no decision — in
 * three sweep orders (per-block slices at 8 and 3 blocks per SM, the whole
 * grid front to back).  The best device time per pass (CUDA events, warm L2,
 * `reps` passes of each) is the memory-system floor of one iteration on this
 * graph; bench.py reports the step kernel's time against it. */
int ivhd_gather_floor(ivhd_ctx* ctx, int slot, int reps, double* us_out);

/* Exact kNN graph of the rows of a host (m, n) float64 matrix, computed on
 * `device` (knng.build_exact_knn, knng.py:158-194): row i lists its k nearest
 * other rows by (distance, index); metric 0 = euclidean (distance), 1 =
 * cosine (1 - cos, rows normalised first; a zero row is IVHD_ERR_INVALID_ARG
 * with "zero-norm vector" in the message), 2 = precomputed (x is an (m, m)
 * distance matrix, n == m; k <= 128).  1 <= k < m, k <= 64 otherwise.
 * nbr_out (m, k) int32 and dist_out (m, k) float64 are host buffers.
 * stats_out (optional, 8 doubles): tensor-core pass seconds, re-rank seconds,
 * rows re-scanned exactly (uncertified), total seconds, setup seconds (H2D +
 * pack), exact re-scan seconds, D2H seconds, 0.  Errors: message in
 * ivhd_knn_last_error(). */
int ivhd_knn_build(int device, const double* x, int64_t m, int32_t n, int32_t k, int32_t metric,
                   int32_t* nbr_out, double* dist_out, double* stats_out);
const char* ivhd_knn_last_error(void);

/* Label neighbour hit of an embedding (metrics.neighbor_hit, metrics.py:254-294)
 * computed on `device`: y (m, dim) float64 host points (1 <= dim <= 3), labels
 * (m) int32; cf_nn_out[j] (nn_max doubles) = fraction of same-label points
 * among the j+1 nearest other points, averaged over all points.  Exact grid
 * kNN, (distance, index) order.  1 <= nn_max < m, nn_max <= 512.  nbr_out:
 * optional (m, nn_max) int32 neighbour ids.  Errors: ivhd_metrics_last_error(). */
int ivhd_neighbor_hit(int device, const double* y, int64_t m, int32_t dim, const int32_t* labels,
                      int32_t nn_max, double* cf_nn_out, int32_t* nbr_out);
/* One rank-curve pass (metrics._curve_pass, metrics.py:149-182) on `device`:
 * x (m, n) float64 source points, or with x_precomputed an (m, m) distance
 * matrix; y (m, dim) float64 embedding (1 <= dim <= 3); labels (m) int32 or
 * NULL.  Ranks use squared distances (|a|^2 + |b|^2) - 2 a.b clamped at 0 and
 * the (distance, index) tie rule.  Outputs (integer counts, host buffers):
 * agree_out[p], p = 0..k_max: #pairs with max(rho, r) == p; same_ld_out /
 * same_hd_out[p], p < k_max: #rows whose (p+1)-th LD / HD neighbour shares the
 * label (only with labels); trust_out / cont_out[a]: summed entrant / leaver
 * rank penalties at report_ks[a] (n_report <= 8, 1 <= k < m/2).
 * 1 <= k_max <= m-2 and max(k_max, report ks) <= 1024.
 * Errors: ivhd_metrics_last_error(). */
int ivhd_curve_pass(int device, const double* x, int64_t m, int32_t n, int32_t x_precomputed, const double* y,
                    int32_t dim, const int32_t* labels, int32_t k_max, const int32_t* report_ks, int32_t n_report,
                    int64_t* agree_out, int64_t* same_ld_out, int64_t* same_hd_out, int64_t* trust_out,
                    int64_t* cont_out);
/* Exact pair ranks (metrics._pair_ranks, metrics.py:335-352): ranks_out[p] =
 * 1 + #{k != i : (d2(i,k), k) < (d2(i,j), j)} for i = i_idx[p], j = j_idx[p]
 * (i != j), squared distances (|a|^2 + |b|^2) - 2 a.b clamped at 0 over the
 * rows of z (m, n) float64.  Host buffers.  Errors: ivhd_metrics_last_error(). */
int ivhd_pair_ranks(int device, const double* z, int64_t m, int32_t n, const int64_t* i_idx, const int64_t* j_idx,
                    int64_t n_pairs, int64_t* ranks_out);
/* Full rank matrix (metrics.compute_ranks, metrics.py:103-146): ranks_out
 * (m, m) int64 host buffer, row i = rank 1..m-1 of every other point by
 * (distance, index), 0 on the diagonal.  x (m, n) float64 points (squared
 * distances (|a|^2 + |b|^2) - 2 a.b clamped at 0) or, with precomputed, an
 * (m, m) distance matrix (n == m).  Errors: ivhd_metrics_last_error(). */
int ivhd_rank_matrix(int device, const double* x, int64_t m, int32_t n, int32_t precomputed, int64_t* ranks_out);
const char* ivhd_metrics_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* IVHD_B200_H */
