// ivhd_step.cuh — the fused IVHD iteration for sm_100a.
//
// One launch = one loop iteration of engine.run_embedding
// (/root/reference/pkg/src/ivhd/engine.py:346-384):
//   forces at the evaluation positions   forces.py:86-136 (vertex-centric)
//   stress at the current positions      forces.py:78-83, 123-124
//   optimizer update                     optim.py:95-236, 259-263
//   auto-adapt decision + rollback       optim.py:80-92, 113-124
//   divergence flag                      engine.py:373-377
//
// Layout (HBM):
//   row_ptr[M+1] u32, col[2L] u32 (bit 31 = random-pair class, zero extra bytes)
//   ew[2L] float2 {target, scale} only for euclidean / RNN-filtered sets
//   positions: two buffers (Jacobi double buffering + rollback), stride
//              YS floats/vertex: 2 (dim 2), 4 (dim 2 Nesterov: y | y+beta v,
//              dim 3 padded), 8 (dim 3 Nesterov)
//   optimizer state: SS floats/vertex, 8/16-byte vector access
//   per-tile partials double4 {sum_i sum_e w(t-d)^2, sum|dnew|^2,
//              sum|dold|^2, #non-finite}: fixed tile size => the reduction
//              order is independent of grid size and of the rank count.
//
// Work mapping: persistent blocks of 8 consumer warps + 1 TMA producer warp
// run a static list of work units (one pass of a 256-vertex tile with G lanes
// per vertex; cost-balanced per block in the fused loop, round robin in the
// sharded one).  The producer stages each unit's row pointers, columns,
// positions and optimizer state with cp.async.bulk into a 3-stage ring; the G
// lanes of a row gather neighbour positions, reduce with a fixed xor
// butterfly (all lanes get the bit-identical sum) and lane 0 of the group
// applies the optimizer.  No atomics touch the data.  One GPU: every block
// adds its partials to four fixed-point sums (integer atomics, order-
// independent) and the NEXT launch decides this iteration at its start (cur
// buffer, b, trace, status; Ctrl::pend), the last block to read the control
// block persisting the decided state.
// Sharded / Adam: the last block to finish reduces the partials in fixed order
// and writes the decision that the next launch reads.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace ivhd {

#ifdef IVHD_TIMELINE
// Debug build only: %globaltimer stamps of iterations 10 and 11, per block:
// [0] entry, [1] after the dependency wait, [2+k] consumer warp 0 done with
// unit k (k < 34), [36] all warps done, [37] arrival, [38] warp 0 loop end,
// [39] finalize end (last block only).
constexpr int kTlBlocks = 1024, kTlSlots = 40;
__device__ long long g_tl[2][kTlBlocks][kTlSlots];
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define IVHD_TL(slot)                                                                      \
  do {                                                                                     \
    if (tl_rec && lane == 0 && warp == 0 && blockIdx.x < kTlBlocks) tl_rec[(slot)] = gtime(); \
  } while (0)
#else
#define IVHD_TL(slot) \
  do {                \
  } while (0)
#endif


#ifndef IVHD_BLOCK
#define IVHD_BLOCK 256
#endif
constexpr int kBlock = IVHD_BLOCK;  // threads per block = vertices per tile

// Block barrier.  __syncthreads() lowers to the *aligned* bar.sync, which
// assumes every warp arrives converged; after the data-dependent merge-path
// walk, lanes of one warp can arrive separately (independent thread
// scheduling) and the aligned barrier then let early lanes through (observed
// on B200 / CUDA 12.9).  The non-aligned barrier.sync counts threads.
__device__ __forceinline__ void block_sync() { asm volatile("barrier.sync 0;" ::: "memory"); }
// Barrier over the first kBlock threads only (reductions run without the producer warp).
__device__ __forceinline__ void group_sync() { asm volatile("barrier.sync 1, %0;" ::"n"(IVHD_BLOCK) : "memory"); }

constexpr uint32_t kRandBit = 0x80000000u;
constexpr uint32_t kIdMask = 0x7fffffffu;

enum Opt { OPT_FD = 0, OPT_SGD = 1, OPT_MOM = 2, OPT_NEST = 3, OPT_ADAM = 4, OPT_ADADELTA = 5, OPT_NONE = 6 };

// Device-resident control block: everything a CUDA-graph replay must pick up
// without re-capture.
struct Ctrl {
  int cur;              // buffer index holding the current positions
  int status;           // 0 running, 1 diverged
  int last_commit;      // did the last iteration move the positions
  int pad0;
  long long iter;       // trace slot of the next iteration (reset per run call)
  long long gstep;      // global iteration counter (degenerate-pair RNG)
  long long diverged_at;
  long long adam_t;     // Adam step counter (optim.py:190,200)
  double step;          // b (force-directed) / alpha / scale
  double c;             // random-pair weight
  unsigned int arrive;  // blocks finished this launch
  unsigned int next_tile;
  unsigned int parrive; // peer mode: blocks that published this launch
  int need;             // a degenerate random pair had no direction in the table (forces.py:167-174)
  int scur;             // optimizer-state buffer holding the current state (double buffered)
  int dg_n;             // directions in the degenerate-pair table ...
  long long dg_gstep;   // ... valid for this global iteration only
  // deferred decisions (single-GPU loop): launch t+1 decides iteration t from
  // t's partial sums before its own work; the last block to read persists the decision
  int pend;             // the partial sums in slot `pslot` await their decision
  int pslot;
  int needw[2];         // per slot: a degenerate pair had no direction
  unsigned int readers; // blocks of this launch that have read the control block
  int fnf[2];           // per slot: bit 2q component q was +-inf / out of range, bit 2q+1 NaN
  unsigned long long facc[2][4];  // per slot: the launch's partials in fixed point (2^-20), summed by atomics
};

constexpr int kMaxPeers = 7;  // up to 8 ranks (one node)

// Fused peer exchange (sharded mode over NVLink P2P, one process per GPU):
// the step kernel stores each updated position into every peer's replica and
// its tile partials into every peer's partial array, then raises its arrival
// flag on every peer; finalize_peer_kernel waits for all ranks' flags and
// takes the (identical) decision.  Buffers below are the peers' (CUDA IPC).
struct PeerArgs {
  int on;                         // 1: peer mode
  int n_peers, rank, world;
  int t0, t1;                     // this rank's tiles
  float* y0[kMaxPeers];           // peers' position buffers 0 / 1
  float* y1[kMaxPeers];
  double4* tp[kMaxPeers];         // peers' tile partials [2][n_tiles_cap] (by stamp parity)
  unsigned long long* fl[kMaxPeers];  // peers' arrival flags [world]
  double4* tp_local;              // own tile partials [2][n_tiles_cap]
  unsigned long long* fl_local;   // own arrival flags [world]
  unsigned long long* stamp;      // iterations exchanged so far (device word; survives ivhd_restore)
  int n_tiles_cap;
  int decide_here;                // 1: the step kernel's last block waits for the peers and decides
                                  // (one process per GPU); 0: finalize_peer_kernel does (emulation)
  long long timeout_ns;           // finalizer wait limit before it reports a peer failure
  int prank[kMaxPeers];           // rank of peer slot k
  const uint8_t* mask;            // halo: bit r of mask[v] = rank r has a row that gathers v
};

struct Hyper {
  float a;               // force-directed friction (per-vertex fp32 update)
  float beta, gv, gs, rho, eps;
  double g1, g2;         // step-size factors: b is kept in fp64 like the reference
  double tau;
  double gv_d, gs_d, eps_d;  // Adam moments in fp64 (ivhd_step_f64.cuh)
  int adapt;
};

struct StepArgs {
  const uint32_t* row_ptr;
  const uint32_t* col;
  const float2* ew;       // nullptr in binary mode
  float* ybuf0;
  float* ybuf1;
  float* state;           // two buffers of sstride floats: ctrl->scur holds the current state
  long long sstride;
  const int2* dg_key;     // degenerate-pair table: (row, entry index in the row) -> direction
  const float4* dg_vec;   //   x, y, z = w * t * unit direction drawn by the host from run.rng
  int* miss_n;            // pairs with no table entry this iteration ...
  int2* miss;             // ... (row, entry index), up to miss_cap of them
  int miss_cap;
  int stream_hint;        // evict-first L2 policy on the streamed graph data (working set > L2)
  double4* partial;       // per work unit (sharded / operator calls)
  double4* tpart;         // per tile: sharded mode's exchanged partials
  const int* unit_base;   // first unit of each tile
  double4* bpart;         // fused mode: one partial per block (its units, in order)
  double2* trace;
  Ctrl* ctrl;
  double* force_out;      // OPT_NONE only: (M, DIM) float64
  const uint8_t* tile_g;  // lanes per vertex of every (global) tile
  const int* units;       // work unit -> tile << 12 | pass << 7 | min(slots,15) << 3 | log2 G
  const int* boff;        // fused mode: block b runs units[boff[b] .. boff[b+1]) (cost-balanced
                          // static schedule); nullptr: round robin u = b + k * grid
  long long v_begin, v_end;
  int tile_v;
  int n_tiles;            // work units this launch processes
  int tile0;              // global index of its first work unit
  int n_tiles_global;     // work-unit partials reduced by the finalizer
  int norm;               // 0 = L2, 1 = L1
  int fuse_finalize;      // single GPU: running sums, one partial per block (decided by the last block or deferred)
  int defer;              // fuse_finalize with deferred decisions (Ctrl::pend): the next launch decides
  int fixed_io;           // sharded async mode: read ybuf0, write ybuf1 (host-chosen parity)
  int out_index;          // fixed_io: which context buffer ybuf1 is (becomes ctrl->cur)
  long long v_cap_floats; // fixed_io: floats per position buffer (rollback copy)
  Hyper h;
  PeerArgs pe;
};

// ------------------------------------------------------------------ layout

template <int DIM, int OPT> struct Layout {
  static constexpr int YS = (OPT == OPT_NEST) ? (DIM == 2 ? 4 : 8) : (DIM == 2 ? 2 : 4);
  static constexpr int NV = (OPT == OPT_FD || OPT == OPT_MOM || OPT == OPT_NEST) ? 1
                            : (OPT == OPT_ADAM || OPT == OPT_ADADELTA) ? 2 : 0;
  static constexpr int SS = NV == 0 ? 0 : (DIM == 2 ? 2 * NV : 4 * NV);
};

template <int DIM>
__device__ __forceinline__ void ld_vec(const float* p, float (&v)[DIM]) {
  if constexpr (DIM == 2) {
    float2 t = *reinterpret_cast<const float2*>(p);
    v[0] = t.x; v[1] = t.y;
  } else {
    float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z;
  }
}

template <int DIM>
__device__ __forceinline__ void st_vec(float* p, const float (&v)[DIM]) {
  if constexpr (DIM == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], 0.f);
  }
}

// Gather of a neighbour's position (and Nesterov look-ahead) in one access.
template <int DIM, bool NEST>
__device__ __forceinline__ void gather(const float* __restrict__ Y, uint32_t j, float (&y)[DIM],
                                       float (&l)[DIM]) {
  if constexpr (DIM == 2 && !NEST) {
    float2 t = __ldg(reinterpret_cast<const float2*>(Y) + j);
    y[0] = l[0] = t.x; y[1] = l[1] = t.y;
  } else if constexpr (DIM == 2 && NEST) {
    float4 t = __ldg(reinterpret_cast<const float4*>(Y) + j);
    y[0] = t.x; y[1] = t.y; l[0] = t.z; l[1] = t.w;
  } else if constexpr (DIM == 3 && !NEST) {
    float4 t = __ldg(reinterpret_cast<const float4*>(Y) + j);
    y[0] = l[0] = t.x; y[1] = l[1] = t.y; y[2] = l[2] = t.z;
  } else {
    float4 t = __ldg(reinterpret_cast<const float4*>(Y) + 2 * (size_t)j);
    float4 u = __ldg(reinterpret_cast<const float4*>(Y) + 2 * (size_t)j + 1);
    y[0] = t.x; y[1] = t.y; y[2] = t.z; l[0] = u.x; l[1] = u.y; l[2] = u.z;
  }
}

// ---------------------------------------------------- degenerate directions
// forces.py:167-174: a random pair at exactly zero distance gets a unit
// direction drawn from run.rng (standard normals, in connection order,
// magnitude w * t).  The draw needs the reference's generator, so it is made
// on the host: the kernel looks the pair up in a small table the host filled
// for this iteration (keyed by row and entry index, so both endpoint rows of
// the connection get the same direction with opposite signs); a pair without
// an entry is recorded and flags the iteration, which the decision then
// turns into a pause (status 2, nothing committed, state not advanced).  The
// host draws the directions in connection order, fills the table and the
// iteration is re-run.  Measure-zero: after a random init it never happens.
__device__ __forceinline__ void record_degenerate(int* need, int* miss_n, int2* miss, int miss_cap, uint32_t v, int e) {
  const int slot = atomicAdd(miss_n, 1);
  if (slot < miss_cap) miss[slot] = make_int2((int)v, e);
  atomicExch(need, 1);
}

// (out of line, rare path: plain pointers only, so the caller keeps the
// kernel parameters in the constant bank instead of copying them to a stack)
static __device__ __noinline__ float4 degenerate_lookup(Ctrl* c, int* need, const int2* key, const float4* vec,
                                                int* miss_n, int2* miss, int miss_cap, uint32_t v, int e,
                                                long long gstep) {
  if (c->dg_gstep == gstep) {
    for (int i = 0; i < c->dg_n; ++i) {
      const int2 k = key[i];
      if (k.x == (int)v && k.y == e) return vec[i];
    }
  }
  const int slot = atomicAdd(miss_n, 1);
  if (slot < miss_cap) miss[slot] = make_int2((int)v, e);
  atomicExch(need, 1);
  return make_float4(0.f, 0.f, 0.f, 0.f);
}

template <int DIM>
__device__ __forceinline__ void degenerate_vec(const StepArgs& A, int* need, uint32_t v, int e, long long gstep,
                                               float (&u)[DIM]) {
  const float4 q = degenerate_lookup(A.ctrl, need, A.dg_key, A.dg_vec, A.miss_n, A.miss, A.miss_cap, v, e, gstep);
  u[0] = q.x;
  u[1] = q.y;
  if constexpr (DIM == 3) u[2] = q.z;
}

// ------------------------------------------------------------------ entries
// Contribution of one symmetrised-CSR entry to row i (forces.py:97-124):
//   L2: phi = -w (t == 0) | w (t - d)/d ; f += phi (y_i - y_o);  e += w (t-d)^2
//   L1: f += sign(y_i - y_o) w (t - d);                           e += w (t-d)^2
// The L2 form is branch-free: with rs = rsqrt(d^2), w (t - d)/d = w (t rs - 1)
// and d = d^2 rs (guarded at 0 and inf).  Random pairs at exactly zero
// distance (t != 0, d == 0) take the rare degenerate branch (forces.py:167-174).
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Adds the entry's force and stress contribution when `valid`; returns true
// for a degenerate random pair (t != 0 at zero distance), whose force the
// caller adds separately (rare path).  Branch-free.
template <int DIM, bool NEST, int NORM>
__device__ __forceinline__ bool entry(const float (&yi)[DIM], const float (&li)[DIM],
                                      const float (&yo)[DIM], const float (&lo)[DIM],
                                      uint32_t cw, bool weighted, float2 tw, float c, bool valid,
                                      float (&f)[DIM], float& e) {
  const bool rn = cw & kRandBit;
  float t, w;
  if (!weighted) {
    t = rn ? 1.f : 0.f;
    w = rn ? c : 1.f;
  } else {
    t = tw.x;
    w = (rn ? c : 1.f) * tw.y;
  }
  float df[DIM];
  float d2 = 0.f, d1 = 0.f;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    df[d] = li[d] - lo[d];
    d2 = fmaf(df[d], df[d], d2);
    d1 += fabsf(df[d]);
  }
  bool degen = false;
  if constexpr (NORM == 0) {
    const float rs = rsqrt_ftz(d2);
    float phi = (t == 0.f) ? -w : w * fmaf(t, rs, -1.f);
    degen = (t != 0.f) && (d2 == 0.f);
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const float inc = phi * df[d];
      f[d] += (valid && !degen) ? inc : 0.f;
    }
    float q2 = d2, qs = rs;
    if constexpr (NEST) {  // stress at the current (not look-ahead) positions: engine.py:370
      q2 = 0.f;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        const float q = yi[d] - yo[d];
        q2 = fmaf(q, q, q2);
      }
      qs = rsqrt_ftz(q2);
    }
    float de = q2 * qs;
    de = (q2 == 0.f) ? 0.f : de;
    de = (q2 == INFINITY) ? INFINITY : de;
    const float r = t - de;
    const float inc = w * r * r;
    e += valid ? inc : 0.f;
  } else {
    const float s = w * (t - d1);
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const float sg = df[d] > 0.f ? 1.f : (df[d] < 0.f ? -1.f : (df[d] == 0.f ? 0.f : df[d]));
      const float inc = sg * s;
      f[d] += valid ? inc : 0.f;
    }
    float de = d1;
    if constexpr (NEST) {
      de = 0.f;
#pragma unroll
      for (int d = 0; d < DIM; ++d) de += fabsf(yi[d] - yo[d]);
    }
    const float r = t - de;
    const float inc = w * r * r;
    e += valid ? inc : 0.f;
  }
  return valid && degen;
}

__device__ __forceinline__ bool all_finite(const float* v, int n) {
  bool ok = true;
  for (int d = 0; d < n; ++d) ok &= isfinite(v[d]);
  return ok;
}

// ------------------------------------------------------------ block reduce
// Fixed-shape reduction of 4 doubles over the block (deterministic).
__device__ __forceinline__ double warp_dsum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ double4 block_sum4(double4 v, double4* sm /*[kBlock/32]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v.x = warp_dsum(v.x); v.y = warp_dsum(v.y); v.z = warp_dsum(v.z); v.w = warp_dsum(v.w);
  if (lane == 0) sm[warp] = v;
  group_sync();
  double4 r = make_double4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int w = 0; w < kBlock / 32; ++w) {
      r.x += sm[w].x; r.y += sm[w].y; r.z += sm[w].z; r.w += sm[w].w;
    }
  }
  group_sync();
  return r;  // valid in thread 0
}

// The iteration decision from the reduced partials {stress, sum|dnew|^2,
// sum|dold|^2, #non-finite} (optim.py:80-92 + engine.py:373-384); one thread.
constexpr double kMissUnit = 4294967296.0;  // sharded partials: .w = #non-finite + 2^32 * (rank had misses)

// The decided part of the control block.
struct DState {
  int cur, status, last_commit, scur;
  long long iter, gstep, diverged_at, adam_t;
  double step;
};
__device__ __forceinline__ DState dstate_load(const Ctrl* c) {
  DState d;
  d.cur = c->cur; d.status = c->status; d.last_commit = c->last_commit; d.scur = c->scur;
  d.iter = c->iter; d.gstep = c->gstep; d.diverged_at = c->diverged_at; d.adam_t = c->adam_t;
  d.step = c->step;
  return d;
}
__device__ __forceinline__ void dstate_store(Ctrl* c, const DState& d) {
  c->cur = d.cur; c->status = d.status; c->last_commit = d.last_commit; c->scur = d.scur;
  c->iter = d.iter; c->gstep = d.gstep; c->diverged_at = d.diverged_at; c->adam_t = d.adam_t;
  c->step = d.step;
}

// Decide on d (no memory writes): returns true with the trace entry `tr` for
// slot d.iter (before the update), false when the iteration pauses.
template <int OPT>
__device__ __forceinline__ bool decide_core(const StepArgs& A, double4 s, int need, DState& d, double2& tr) {
  const double misses = floor(s.w / kMissUnit);
  s.w -= misses * kMissUnit;
  if (need || misses > 0.0) {  // degenerate pairs without directions: pause, redo after the host draw
    d.status = 2;
    return false;
  }
  const double E = 0.5 * s.x;
  double step = d.step;
  bool commit = true;
  if (OPT == OPT_FD && A.h.adapt) {
    const double dT = s.y - s.z;
    if (dT > A.h.tau) {
      step *= A.h.g2;
      commit = false;
    } else if (dT < -A.h.tau) {
      step *= A.h.g1;
      commit = false;
    }
  }
  const long long it = d.iter;
  tr = make_double2(E, step);
  if (commit && s.w > 0.0) {
    d.status = 1;
    d.diverged_at = it;
  } else {
    if (A.fixed_io) d.cur = A.out_index;  // the rollback copy (finalize_kernel) refills it
    else if (commit) d.cur ^= 1;
    d.last_commit = commit ? 1 : 0;
    d.step = step;
    d.iter = it + 1;
  }
  d.gstep += 1;
  d.scur ^= 1;  // the state written this iteration is current (FD keeps new deltas on rollback)
  if (OPT == OPT_ADAM) d.adam_t += 1;
  return true;
}

template <int OPT>
__device__ __forceinline__ void decide(const StepArgs& A, double4 s) {
  Ctrl* ctrl = A.ctrl;
  DState d = dstate_load(ctrl);
  double2 tr;
  if (decide_core<OPT>(A, s, ctrl->need, d, tr) && A.trace) A.trace[ctrl->iter] = tr;
  dstate_store(ctrl, d);
  ctrl->need = 0;
  ctrl->next_tile = 0;
  ctrl->arrive = 0;  // the next launch is ordered after this grid completes
}

// Deferred decisions: every block adds its partial to the launch's slot in
// fixed point (2^-20) with integer atomics — order-independent, so the sum is
// the same bit pattern whatever order the blocks finish in — and the next
// launch reads the four sums back.  A block partial beyond 2^63 / 2^11 (so that
// the sum of up to 2048 blocks cannot wrap) or non-finite is flagged and read
// back as inf / NaN.
constexpr double kFixScale = 1048576.0;  // 2^20: per-block rounding <= 5e-7
constexpr double kFixMax = 4.5e15;       // ~2^63 / 2048
__device__ __forceinline__ void fix_add(Ctrl* c, int slot, double4 t) {
  const double v[4] = {t.x, t.y, t.z, t.w};
  int nf = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double x = v[q] * kFixScale;
    if (isnan(x)) {
      nf |= 2 << (2 * q);
    } else if (!(fabs(x) < kFixMax)) {
      nf |= 1 << (2 * q);
    } else {
      atomicAdd(&c->facc[slot][q], (unsigned long long)llrint(x));
    }
  }
  if (nf) atomicOr(&c->fnf[slot], nf);
}
__device__ __forceinline__ double4 fix_read(const Ctrl* c, int slot) {
  double r[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) r[q] = (double)(long long)__ldcg(&c->facc[slot][q]) / kFixScale;
  const int nf = __ldcg(&c->fnf[slot]);
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // as the fp64 sum of the partials would read (all are >= 0)
    if ((nf >> (2 * q)) & 2) r[q] = NAN;
    else if ((nf >> (2 * q)) & 1) r[q] = INFINITY;
  }
  return make_double4(r[0], r[1], r[2], r[3]);
}

// ---------------------------------------------------------------- finalize
// Reduce n partials in a fixed order and take the iteration decision
// (optim.py:80-92 + engine.py:373-384).  Executed by ONE whole block; each
// thread keeps 8 partials in flight.  Fused single-GPU mode reduces the
// per-block partials (one per resident block); sharded mode reduces the
// all-gathered per-unit partials, whose order does not depend on the rank
// count.
template <int OPT>
__device__ void finalize_block(const StepArgs& A, double4* sm, const double4* src, int n) {
  const double2* p2 = reinterpret_cast<const double2*>(src);
  double4 s = make_double4(0, 0, 0, 0);
  for (int t0 = threadIdx.x; t0 < n; t0 += 8 * kBlock) {
    double2 a[8], b[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int t = t0 + u * kBlock;
      if (t < n) {
        a[u] = __ldcg(p2 + 2 * t);
        b[u] = __ldcg(p2 + 2 * t + 1);
      } else {
        a[u] = b[u] = make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s.x += a[u].x; s.y += a[u].y; s.z += b[u].x; s.w += b[u].y;
    }
  }
  s = block_sum4(s, sm);
  if (threadIdx.x == 0) decide<OPT>(A, s);
}

// Fused single-GPU finalizer: ONE warp reduces the n per-block partials
// (lane l sums l, l+32, ... in order, then a fixed butterfly) and lane 0
// decides.  The caller (lane 0) has acquired every block's arrival.
template <int OPT>
__device__ void finalize_warp(const StepArgs& A, const double4* src, int n) {
  const int lane = threadIdx.x & 31;
  const double2* p2 = reinterpret_cast<const double2*>(src);
  double4 s = make_double4(0, 0, 0, 0);
  constexpr int kBatch = 16;  // loads in flight per lane (L2, bypassing L1): 444 block partials in one round trip
  for (int t0 = lane; t0 < n; t0 += 32 * kBatch) {
    double2 a[kBatch], b[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int t = t0 + 32 * j;
      a[j] = b[j] = make_double2(0.0, 0.0);
      if (t < n) {
        a[j] = __ldcg(p2 + 2 * t);
        b[j] = __ldcg(p2 + 2 * t + 1);
      }
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      s.x += a[j].x; s.y += a[j].y; s.z += b[j].x; s.w += b[j].y;
    }
  }
  s.x = warp_dsum(s.x); s.y = warp_dsum(s.y); s.z = warp_dsum(s.z); s.w = warp_dsum(s.w);
  if (lane == 0) decide<OPT>(A, s);
}

template <int SS>
__device__ __forceinline__ void ld_state(const float* p, float (&s)[SS > 0 ? SS : 1]) {
  if constexpr (SS == 2) {
    const float2 t = *reinterpret_cast<const float2*>(p);
    s[0] = t.x; s[1] = t.y;
  } else if constexpr (SS == 4) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    s[0] = t.x; s[1] = t.y; s[2] = t.z; s[3] = t.w;
  } else if constexpr (SS == 8) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    const float4 u = *reinterpret_cast<const float4*>(p + 4);
    s[0] = t.x; s[1] = t.y; s[2] = t.z; s[3] = t.w; s[4] = u.x; s[5] = u.y; s[6] = u.z; s[7] = u.w;
  }
}

template <int SS>
__device__ __forceinline__ void st_state(float* p, const float (&s)[SS > 0 ? SS : 1]) {
  if constexpr (SS == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(s[0], s[1]);
  } else if constexpr (SS == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(s[0], s[1], s[2], s[3]);
  } else if constexpr (SS == 8) {
    *reinterpret_cast<float4*>(p) = make_float4(s[0], s[1], s[2], s[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(s[4], s[5], s[6], s[7]);
  }
}

// Optimizer update of one vertex (optim.py:95-236 with step_optimizer's
// grad = -2 force, optim.py:259-263).  State vectors live in sv: FD delta /
// momentum velocity at [0, DIM); Adam (v, s) and Adadelta (E[g^2], E[d^2])
// at [0, DIM) and [V, V+DIM) with V = 2 (dim 2) or 4 (dim 3).
// Store one vertex's new position record (YS floats) at base + v * YS.
template <int DIM, int OPT>
__device__ __forceinline__ void store_pos(float* base, long long v, const float (&yn)[DIM], const float (&la)[DIM]) {
  if constexpr (OPT == OPT_NEST) {
    if constexpr (DIM == 2) {
      *reinterpret_cast<float4*>(base + (size_t)v * 4) = make_float4(yn[0], yn[1], la[0], la[1]);
    } else {
      *reinterpret_cast<float4*>(base + (size_t)v * 8) = make_float4(yn[0], yn[1], yn[2], 0.f);
      *reinterpret_cast<float4*>(base + (size_t)v * 8 + 4) = make_float4(la[0], la[1], la[2], 0.f);
    }
  } else {
    st_vec<DIM>(base + (size_t)v * Layout<DIM, OPT>::YS, yn);
  }
}

template <int DIM, int OPT, bool PEER>
__device__ __forceinline__ void apply_update(const StepArgs& A, float* __restrict__ Yout, float* __restrict__ Sout,
                                             long long v,
                                             const float (&yi)[DIM], float (&sv)[Layout<DIM, OPT>::SS > 0 ? Layout<DIM, OPT>::SS : 1],
                                             const float (&f)[DIM], float step, float bc1, float bc2,
                                             float& acc_n, float& acc_o, float& acc_bad) {
  using L = Layout<DIM, OPT>;
  constexpr int V = DIM == 2 ? 2 : 4;
  float yn[DIM];
  if constexpr (OPT == OPT_FD) {
    float so = 0.f, sn = 0.f;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const float dn = fmaf(A.h.a, sv[d], step * f[d]);
      so = fmaf(sv[d], sv[d], so);
      sn = fmaf(dn, dn, sn);
      sv[d] = dn;
      yn[d] = yi[d] + dn;
    }
    acc_o += so;
    acc_n += sn;
  } else if constexpr (OPT == OPT_SGD) {
#pragma unroll
    for (int d = 0; d < DIM; ++d) yn[d] = yi[d] - step * (-2.f * f[d]);
  } else if constexpr (OPT == OPT_MOM || OPT == OPT_NEST) {
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      sv[d] = A.h.beta * sv[d] - step * (-2.f * f[d]);
      yn[d] = yi[d] + sv[d];
    }
  } else if constexpr (OPT == OPT_ADAM) {
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const float g = -2.f * f[d];
      sv[d] = A.h.gv * sv[d] + (1.f - A.h.gv) * g;
      sv[V + d] = A.h.gs * sv[V + d] + (1.f - A.h.gs) * g * g;
      yn[d] = yi[d] - step * (sv[d] * bc1) / (A.h.eps + sqrtf(sv[V + d] * bc2));
    }
  } else if constexpr (OPT == OPT_ADADELTA) {
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const float g = -2.f * f[d];
      sv[d] = A.h.rho * sv[d] + (1.f - A.h.rho) * g * g;
      const float dl = -step * sqrtf(sv[V + d] + A.h.eps) / sqrtf(sv[d] + A.h.eps) * g;
      sv[V + d] = A.h.rho * sv[V + d] + (1.f - A.h.rho) * dl * dl;
      yn[d] = yi[d] + dl;
    }
  }
  if constexpr (L::SS > 0) st_state<L::SS>(Sout + (size_t)v * L::SS, sv);
  float la[DIM];
#pragma unroll
  for (int d = 0; d < DIM; ++d) la[d] = OPT == OPT_NEST ? yn[d] + A.h.beta * sv[d] : yn[d];  // optim.py:174-175
  store_pos<DIM, OPT>(Yout, v, yn, la);
  if constexpr (PEER) {  // fused exchange: the same record into the replica of every peer that gathers it
    if (A.pe.n_peers > 0) {
      const bool out1 = Yout == A.ybuf1;
      const unsigned mk = A.pe.mask[v];
      for (int q = 0; q < A.pe.n_peers; ++q)
        if ((mk >> A.pe.prank[q]) & 1u) store_pos<DIM, OPT>(out1 ? A.pe.y1[q] : A.pe.y0[q], v, yn, la);
    }
  }
  acc_bad += all_finite(yn, DIM) ? 0.f : 1.f;
}

// ------------------------------------------------------------------ kernel
// Vertices are relabelled by degree at setup (ivhd_capi.cu), so the 256
// consecutive vertices of a tile have near-equal degree.  Each tile carries
// G = lanes per vertex (1, 2, 4, ..., 32; G * kUnroll >= its max degree
// except for hubs): G lanes walk one CSR row with kUnroll independent column
// loads and position gathers in flight each, reduce with a fixed xor
// butterfly, and lane 0 applies the optimizer.  The only block barrier is
// the per-tile partial reduction.
#ifndef IVHD_UNROLL
#define IVHD_UNROLL 8
#endif
#ifndef IVHD_MINBLOCKS
#define IVHD_MINBLOCKS 3
#endif
constexpr int kUnroll = IVHD_UNROLL;
#ifndef IVHD_STAGES
#define IVHD_STAGES 3
#endif
constexpr int kStages = IVHD_STAGES;  // TMA ring depth (units in flight per block)

// ------------------------------------------------------------- TMA helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// programmatic dependent launch (griddepcontrol): the next iteration's grid
// may start once every block has signalled; it waits before reading data the
// previous grid writes.  No-ops when the launch carries no PDL attribute.
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// non-blocking probe of a phase (the producer polls two barrier kinds)
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// global -> shared bulk copy (TMA, non-tensor); 16-byte aligned, size % 16 == 0
// L2 eviction policy for the streamed graph data (row pointers, columns) when
// the working set exceeds L2 (A.stream_hint): first out, so the randomly
// gathered positions stay (planted 10^7: 263 -> 252 µs; C3 fits L2 and runs
// without it, profiles/r02_kernel_experiments.md)
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

#ifndef IVHD_COLCAP
#define IVHD_COLCAP 2048
#endif
constexpr int kColCap = IVHD_COLCAP;  // staged column entries per unit (larger units read global)

// column ids read straight from global: streamed, never allocated in L1 (L1
// is kept for the neighbour-position gathers)
__device__ __forceinline__ uint32_t ld_col(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
// neighbour-position gather through the non-coherent path, allocating in L1
// (hub positions are re-read by many rows of a block)
__device__ __forceinline__ float2 ld_pos(const float2* p) { return __ldg(p); }
#ifndef IVHD_UNIT_CACHE
#define IVHD_UNIT_CACHE 256
#endif
constexpr int kUnitCache = IVHD_UNIT_CACHE;  // unit words cached per block

// Fast path for the dominant case (2-D, binary, L2, positions without look-ahead):
// a lane handles the entries cb[0], cb[G], ... (deg of them; G lanes per row);
// the slot count D <= 8 is a template constant, all D column reads and gathers
// are issued first, then ~20 instructions per entry.  Slots past the lane's
// last entry are self pairs (zero contribution).
template <int D, bool GCOL>
__device__ __forceinline__ void fast_row(const StepArgs& A, int* need, const uint32_t* __restrict__ cb, int G, int deg,
                                         int ebase, const float* __restrict__ Yin, uint32_t v, float y0, float y1,
                                         float c, long long gstep, float (&f)[2], float& e) {
  uint32_t cw[D];
  float2 p[D];
#pragma unroll
  for (int q = 0; q < D; ++q) cw[q] = q < deg ? (GCOL ? ld_col(cb + q * G) : cb[q * G]) : v;
#pragma unroll
  for (int q = 0; q < D; ++q) {
    p[q] = make_float2(y0, y1);
    if (q < deg) p[q] = ld_pos(reinterpret_cast<const float2*>(Yin) + (cw[q] & kIdMask));
  }
  float fx = f[0], fy = f[1], ee = e;
  unsigned dmask = 0;
#pragma unroll
  for (int q = 0; q < D; ++q) {
    const float dx = y0 - p[q].x, dy = y1 - p[q].y;
    const float d2 = fmaf(dx, dx, dy * dy);
    const float rs = rsqrt_ftz(d2);
    const bool rn = (int)cw[q] < 0, z = d2 == 0.f;
    const float phi_rn = z ? 0.f : c * (rs - 1.f);   // c (1 - d) / d
    const float de = z ? 0.f : d2 * rs;
    const float r = 1.f - de;
    const float phi = rn ? phi_rn : -1.f;
    fx = fmaf(phi, dx, fx);
    fy = fmaf(phi, dy, fy);
    ee += rn ? c * r * r : d2;
    dmask |= (unsigned)(rn && z) << q;
  }
  if (dmask) {  // degenerate random pairs (forces.py:167-174): slot q is entry ebase + q * G.
    // Only recorded here (the iteration pauses); the re-run with the host's
    // directions launches the weighted instantiation, whose general path
    // applies them (ivhd_capi.cu resume_degenerate).
#pragma unroll
    for (int q = 0; q < D; ++q)
      if ((dmask >> q) & 1u) record_degenerate(need, A.miss_n, A.miss, A.miss_cap, v, ebase + q * G);
  }
  f[0] = fx;
  f[1] = fy;
  e = ee;
}

// Shared-memory layout of one ring stage.
template <int DIM, int OPT>
struct StageLayout {
  static constexpr int STAGES = kStages;
  static constexpr int YS = Layout<DIM, OPT>::YS, SS = Layout<DIM, OPT>::SS;
  static constexpr int RP_BYTES = ((kBlock + 1) * 4 + 15) / 16 * 16 + 16;
  static constexpr int COL_BYTES = kColCap * 4 + 32;
  static constexpr int Y_BYTES = kBlock * YS * 4;
  static constexpr int S_BYTES = kBlock * (SS > 0 ? SS : 1) * 4;
  static constexpr int RP_OFF = 0, COL_OFF = RP_BYTES, Y_OFF = COL_OFF + COL_BYTES, S_OFF = Y_OFF + Y_BYTES;
  static constexpr int BYTES = S_OFF + S_BYTES;
};

template <int DIM, int OPT, bool WEIGHTED, int NORM>
__host__ __device__ constexpr int step_smem_bytes() {
  using SL = StageLayout<DIM, OPT>;
  return SL::STAGES * SL::BYTES;
}

template <int DIM, int OPT, bool WEIGHTED, int NORM>
__host__ __device__ constexpr int step_min_blocks() {
  return IVHD_MINBLOCKS;
}

// Per-stage metadata written by the producer before it arrives on the
// stage's barriers (release) and read by consumers after the wait (acquire).
struct StageMeta {
  int packed;       // unit word: tile << 12 | pass << 7 | min(slots,15) << 3 | log2 G
  int col_off;      // entries skipped at the front of the staged columns (alignment)
  int staged;       // 1 if the unit's columns are in shared memory
  int va;           // first vertex of the unit (vertex ids < 2^31)
  int nv;           // vertices in the unit
  int pad[3];
};

// ------------------------------------------------------------ peer mode
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// release fence at system scope (orders this thread's earlier stores, P2P
// ones included, before its later flag stores; lighter than fence.sc.sys)
__device__ __forceinline__ void fence_release_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ double4 ldcg4(const double4* p) {  // L2 (coherent) load of a double4
  const double2 a = __ldcg(reinterpret_cast<const double2*>(p)), b = __ldcg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// Peer mode, last block of a rank, one warp: the rank's partial (its block
// partials reduced in block order, plus 2^32 if it met degenerate pairs
// without directions) goes into slot `rank` of every rank's partial array
// (half = stamp parity), then flag[rank] = stamp is raised on every rank
// (system-scope release: every block fenced its P2P stores before arriving).
// The ranks' partials are reduced in rank order — deterministic for a given
// rank count; positions and decisions do not depend on it.
__device__ __forceinline__ void peer_rank_publish(const StepArgs& A, int n_blocks) {
  const int lane = threadIdx.x & 31;
  double4 s = make_double4(0, 0, 0, 0);
  for (int t0 = lane; t0 < n_blocks; t0 += 32 * 16) {
    double4 a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = t0 + 32 * j < n_blocks ? ldcg4(A.bpart + t0 + 32 * j) : make_double4(0, 0, 0, 0);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      s.x += a[j].x; s.y += a[j].y; s.z += a[j].z; s.w += a[j].w;
    }
  }
  s.x = warp_dsum(s.x); s.y = warp_dsum(s.y); s.z = warp_dsum(s.z); s.w = warp_dsum(s.w);
  if (lane == 0) {
    if (A.ctrl->need) {
      s.w += kMissUnit;
      A.ctrl->need = 0;
    }
    const unsigned long long stamp = *A.pe.stamp + 1;
    const size_t slot = (size_t)(stamp & 1) * A.pe.world + A.pe.rank;
    A.pe.tp_local[slot] = s;
    for (int q = 0; q < A.pe.n_peers; ++q) A.pe.tp[q][slot] = s;
    if (A.pe.n_peers > 0) {
      fence_release_sys();
      st_release_sys(A.pe.fl_local + A.pe.rank, stamp);
      for (int q = 0; q < A.pe.n_peers; ++q) st_release_sys(A.pe.fl[q] + A.pe.rank, stamp);
    } else {  // one rank: nothing leaves this GPU, GPU scope is enough
      __threadfence();
      *reinterpret_cast<volatile unsigned long long*>(A.pe.fl_local + A.pe.rank) = stamp;
    }
  }
  __syncwarp();
}

// Wait until every rank raised its flag for this iteration (system-scope
// acquire), then reduce the ranks' partials in rank order and decide.  One
// warp (lanes < world wait).  A rank that does not arrive within
// pe.timeout_ns sets status 3 (peer failure) instead of hanging.
template <int OPT>
__device__ __forceinline__ void peer_decide(const StepArgs& A) {
  const int lane = threadIdx.x & 31;
  const unsigned long long stamp = *A.pe.stamp + 1;
  int fail = 0;
  if (lane < A.pe.world) {
    const unsigned long long* f = A.pe.fl_local + lane;
    long long t0 = 0, t1 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    // own flag: written by this GPU (GPU scope); the peers' over NVLink (system)
    while ((lane == A.pe.rank ? ld_acquire_gpu(f) : ld_acquire_sys(f)) < stamp) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > A.pe.timeout_ns) {
        fail = 1;
        break;
      }
      __nanosleep(64);
    }
  }
  fail = __any_sync(0xffffffffu, fail);
  if (lane != 0) return;
  if (fail) {
    A.ctrl->status = 3;
    return;
  }
  __threadfence();
  const double4* tp = A.pe.tp_local + (size_t)(stamp & 1) * A.pe.world;
  double4 s = make_double4(0, 0, 0, 0);
  for (int r = 0; r < A.pe.world; ++r) {
    const double4 q = ldcg4(tp + r);
    s.x += q.x; s.y += q.y; s.z += q.z; s.w += q.w;
  }
  decide<OPT>(A, s);
  *A.pe.stamp = stamp;
}

// ------------------------------------------------------------------ kernel
// Persistent blocks take work units statically (u = blockIdx.x + k*grid;
// heavy tiles first in unit order).  Thread 0 is also the TMA producer: for
// unit k+2 it bulk-copies the row pointers, positions and optimizer state
// into ring stage (k+2)%3, and once unit k+1's row pointers have landed it
// bulk-copies that unit's contiguous column segment.  The block computes
// unit k from shared memory; only the neighbour-position gathers go to
// global memory (L2).  Tiles hold 256 vertices relabelled by degree; a unit
// is one pass of a tile: 256/G vertices with G lanes each.
constexpr int kThreads = kBlock + 32;  // 8 consumer warps + 1 TMA producer warp
constexpr int kConsumerWarps = kBlock / 32;

// PEER: sharded mode with the fused NVLink exchange (separate instantiation,
// so the single-GPU kernel carries none of its code).
template <int DIM, int OPT, bool WEIGHTED, int NORM, bool PEER>
__global__ void __launch_bounds__(kThreads, step_min_blocks<DIM, OPT, WEIGHTED, NORM>()) step_kernel(StepArgs A) {
  using L = Layout<DIM, OPT>;
  using SL = StageLayout<DIM, OPT>;
  constexpr int kStages = SL::STAGES;
  constexpr bool NEST = (OPT == OPT_NEST);
  constexpr int SSX = L::SS > 0 ? L::SS : 1;
  constexpr int YS = L::YS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar_r[kStages], bar_a[kStages], bar_b[kStages], bar_e[kStages];
  __shared__ StageMeta meta[kStages];
  __shared__ double4 sm_wp[kStages][kConsumerWarps];
  __shared__ int sm_cnt[kStages];
  __shared__ int sm_units[kUnitCache];  // this block's unit words (static schedule)

  Ctrl* ctrl = A.ctrl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef IVHD_TIMELINE
  const long long tl_entry = gtime();
  long long* tl_rec = nullptr;
#endif
  const int n_units = A.n_tiles;
  const int grid = gridDim.x;
  // this block's unit list: a cost-balanced contiguous range (fused mode) or
  // round robin over the heavy-first unit order (sharded mode)
  const int* ulist = A.units + A.tile0 + blockIdx.x;
  int ustride = grid;
  int my_units = blockIdx.x < n_units ? (n_units - 1 - blockIdx.x) / grid + 1 : 0;
  if (A.boff) {
    const int b0 = __ldg(A.boff + blockIdx.x);
    my_units = __ldg(A.boff + blockIdx.x + 1) - b0;
    ulist = A.units + b0;
    ustride = 1;
  }

  // ---- before the dependency wait: only graph constants (unit list, row
  // pointers, columns) are read, so this overlaps the previous iteration's tail.
  for (int k = tid; k < min(my_units, kUnitCache); k += kThreads)
    sm_units[k] = __ldg(ulist + k * ustride);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bar_r[s], 1);
      mbar_init(&bar_a[s], 1);
      mbar_init(&bar_b[s], 1);
      mbar_init(&bar_e[s], kConsumerWarps);
      sm_cnt[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    griddep_launch_dependents();
  }
  block_sync();

  auto unit_range = [&](int packed, long long& va, int& nv) {
    const int tile = packed >> 12, pass = (packed >> 7) & 31, lgG = packed & 7;
    const int groups = kBlock >> lgG;
    va = (long long)tile * kBlock + (long long)pass * groups;
    nv = (int)max(0LL, min((long long)groups, A.v_end - va));
  };

  // fused mode: this thread's running partials in fp32 over at most 64 units,
  // then folded (fixed fp64 warp butterfly) into its warp's fp64 sums — the
  // auto-adapt test compares the cancelling difference sum|dnew|^2 -
  // sum|dold|^2 with tau, so long sums (C4/C5: ~900 vertices per thread) stay
  // fp64 without fp64 registers in the unit loop
  float te = 0.f, tn = 0.f, to = 0.f, tb = 0.f;
  __shared__ double4 sm_wacc[kConsumerWarps];
  if (tid < kConsumerWarps) sm_wacc[tid] = make_double4(0, 0, 0, 0);

  // deferred decisions (A.defer): consumer warp 0 decides the pending launch's
  // iteration right after the dependency wait; every warp then reads the
  // decided state from shared memory.  sm_df: 0 write slot, 1 decided (trace
  // entry valid), 2 pending slot consumed, 3 its index, 4 stopped before this launch
  __shared__ DState sm_dec;
  __shared__ int sm_df[5];
  __shared__ double2 sm_tr;
  __shared__ long long sm_trit;
  auto defer_decide = [&]() {  // one thread
    DState d = dstate_load(ctrl);
    const int pend = ctrl->pend, pslot = ctrl->pslot, pre = d.status;
    int decided = 0;
    double2 tr = make_double2(0.0, 0.0);
    const long long trit = d.iter;
    if (pre == 0 && pend) decided = decide_core<OPT>(A, fix_read(ctrl, pslot), ctrl->needw[pslot], d, tr) ? 1 : 0;
    if (lane == 0) {
      sm_dec = d;
      sm_df[0] = pend ? (pslot ^ 1) : 0;
      sm_df[1] = decided;
      sm_df[2] = pend;
      sm_df[3] = pslot;
      sm_df[4] = pre != 0;
      sm_tr = tr;
      sm_trit = trit;
    }
  };
  // the block that reads the control block last (its reader count says every
  // other block has read it), one thread: the decided state, the trace entry,
  // this launch's partials pending — no block waits for another
  auto defer_persist = [&]() {
    dstate_store(ctrl, sm_dec);
    if (sm_df[1] && A.trace) A.trace[sm_trit] = sm_tr;
    if (sm_df[2]) {  // consumed: free for the launch after next
      ctrl->needw[sm_df[3]] = 0;
      ctrl->fnf[sm_df[3]] = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) ctrl->facc[sm_df[3]][q] = 0ull;
    }
    ctrl->pend = sm_dec.status == 0 ? 1 : 0;
    ctrl->pslot = sm_df[0];
    ctrl->readers = 0;
    ctrl->next_tile = 0;
    ctrl->arrive = 0;
  };
  auto flush_partials = [&]() {
    double a = te, b = tn, c2 = to, d = tb;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      c2 += __shfl_xor_sync(0xffffffffu, c2, o);
      d += __shfl_xor_sync(0xffffffffu, d, o);
    }
    if (lane == 0) {
      double4 w = sm_wacc[warp];
      w.x += a; w.y += b; w.z += c2; w.w += d;
      sm_wacc[warp] = w;
    }
    te = tn = to = tb = 0.f;
  };
  if (warp == kConsumerWarps) {
    // ---------------------------------------------------- TMA producer warp
    // Lane 0 issues the bulk copies (the whole warp runs the loop).
      auto issue_rp = [&](int k) {  // row pointers of local unit k (graph constant)
        const int s = k % kStages;
        unsigned char* st = smem_raw + s * SL::BYTES;
        const int packed = k < kUnitCache ? sm_units[k] : __ldg(ulist + k * ustride);
        long long va;
        int nv;
        unit_range(packed, va, nv);
        meta[s].packed = packed;
        meta[s].va = (int)va;
        meta[s].nv = nv;
        const uint32_t rp_bytes = (uint32_t)((nv + 1) * 4 + 15) / 16 * 16;
        mbar_expect_tx(&bar_r[s], rp_bytes);
        if (A.stream_hint) bulk_g2s_hint(st + SL::RP_OFF, A.row_ptr + va, rp_bytes, &bar_r[s], policy_evict_first());
        else bulk_g2s(st + SL::RP_OFF, A.row_ptr + va, rp_bytes, &bar_r[s]);
      };
      auto issue_cols = [&](int k) {  // column segment of local unit k (its row pointers have landed)
        const int s = k % kStages;
        unsigned char* st = smem_raw + s * SL::BYTES;
        long long va;
        int nv;
        unit_range(meta[s].packed, va, nv);
        const uint32_t* rp = reinterpret_cast<const uint32_t*>(st + SL::RP_OFF);
        const uint32_t e0 = rp[0], e1 = rp[nv];
        const uint32_t a0 = e0 & ~3u, a1 = (e1 + 3u) & ~3u;  // 16-byte aligned cover
        if (kColCap > 0 && nv > 0 && e1 > e0 && a1 - a0 <= (uint32_t)kColCap + 4) {
          meta[s].col_off = (int)(e0 - a0);
          meta[s].staged = 1;
          mbar_expect_tx(&bar_b[s], (a1 - a0) * 4);
          if (A.stream_hint) bulk_g2s_hint(st + SL::COL_OFF, A.col + a0, (a1 - a0) * 4, &bar_b[s], policy_evict_first());
          else bulk_g2s(st + SL::COL_OFF, A.col + a0, (a1 - a0) * 4, &bar_b[s]);
        } else {
          meta[s].col_off = 0;
          meta[s].staged = 0;
          mbar_arrive(&bar_b[s]);
        }
      };
      const float* Sin = nullptr;  // current optimizer state (set after the dependency wait)
      auto issue_ys = [&](int k, const float* Yin) {  // positions + optimizer state of unit k
        const int s = k % kStages;
        unsigned char* st = smem_raw + s * SL::BYTES;
        long long va;
        int nv;
        unit_range(meta[s].packed, va, nv);
        const uint32_t y_copy = ((uint32_t)nv * YS * 4 + 15) / 16 * 16;
        uint32_t s_copy = 0;
        if constexpr (L::SS > 0) s_copy = ((uint32_t)nv * L::SS * 4 + 15) / 16 * 16;
        mbar_expect_tx(&bar_a[s], y_copy + s_copy);
        bulk_g2s(st + SL::Y_OFF, Yin + va * YS, y_copy, &bar_a[s]);
        if constexpr (L::SS > 0) bulk_g2s(st + SL::S_OFF, Sin + va * L::SS, s_copy, &bar_a[s]);
      };
      const int pre = min(my_units, kStages);
      int nf = pre, nc = pre;
      if (lane == 0) {
        for (int k = 0; k < pre; ++k) issue_rp(k);
        for (int k = 0; k < pre; ++k) {
          mbar_wait(&bar_r[k], 0);
          issue_cols(k);
        }
      }
      __syncwarp();
      griddep_wait();  // the previous iteration (positions, state, ctrl) is complete
      if (A.defer) block_sync();  // consumer warp 0 has decided the pending iteration
      const int p_status = A.defer ? sm_dec.status : ctrl->status;
      if (p_status != 0) {  // diverged / paused: drain the prefetch and leave
        for (int k = 0; k < pre; ++k) mbar_wait(&bar_b[k], 0);
      } else {
        const int p_cur = A.defer ? sm_dec.cur : ctrl->cur, p_scur = A.defer ? sm_dec.scur : ctrl->scur;
        const float* Yin = (A.fixed_io || !p_cur) ? A.ybuf0 : A.ybuf1;
        Sin = A.state + (p_scur ? A.sstride : 0);
        if (lane == 0)
          for (int k = 0; k < pre; ++k) issue_ys(k, Yin);
        // Event loop: stages are claimed as consumers free them; a unit's
        // columns are requested the moment its row pointers land.
        while (nc < my_units) {
          int ok = 0;
          if (lane == 0) {
            if (nf < my_units && nf < nc + kStages && mbar_test(&bar_e[nf % kStages], (uint32_t)(nf / kStages - 1) & 1))
              ok |= 1;
            if (nc < nf && mbar_test(&bar_r[nc % kStages], (uint32_t)(nc / kStages) & 1)) ok |= 2;
            if (ok & 1) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              issue_rp(nf);
              issue_ys(nf, Yin);
            }
            if (ok & 2) issue_cols(nc);
          }
          ok = __shfl_sync(0xffffffffu, ok, 0);
          nf += ok & 1;
          nc += (ok >> 1) & 1;
        }
      }
    if (p_status != 0) return;
  } else {
    // ----------------------------------------------------- consumer warps
    griddep_wait();
    if (A.defer) {
      if (warp == 0 && lane == 0) defer_decide();
      block_sync();
      if (sm_dec.status != 0) {  // stopped: before this launch (nothing to do) or by this decision
        if (!sm_df[4] && warp == 0 && lane == 0 && atomicAdd(&ctrl->readers, 1u) == gridDim.x - 1) defer_persist();
        return;
      }
      if (warp == 0 && lane == 0 && atomicAdd(&ctrl->readers, 1u) == gridDim.x - 1) defer_persist();
    } else if (ctrl->status != 0) {
      return;  // diverged earlier: later iterations are no-ops
    }
#ifdef IVHD_TIMELINE
    if (A.fuse_finalize && (ctrl->iter == 10 || ctrl->iter == 11) && blockIdx.x < kTlBlocks) {
      tl_rec = g_tl[ctrl->iter - 10][blockIdx.x];
      if (warp == 0 && lane == 0) tl_rec[0] = tl_entry;
    }
    IVHD_TL(1);
#endif
    const int ycur = A.fixed_io ? 0 : (A.defer ? sm_dec.cur : ctrl->cur);
    const float c = (float)ctrl->c;
    const float step = (float)(A.defer ? sm_dec.step : ctrl->step);
    const long long gstep = A.defer ? sm_dec.gstep : ctrl->gstep;
    const float* __restrict__ Yin = ycur ? A.ybuf1 : A.ybuf0;
    float* __restrict__ Yout = ycur ? A.ybuf0 : A.ybuf1;
    float* __restrict__ Sout = A.state + ((A.defer ? sm_dec.scur : ctrl->scur) ? 0 : A.sstride);
    // degenerate pairs without a direction: flagged per partial slot when deferred
    int* const needp = A.defer ? &ctrl->needw[sm_df[0]] : &ctrl->need;
    float bc1 = 1.f, bc2 = 1.f;  // Adam bias corrections (optim.py:203-204)
    if constexpr (OPT == OPT_ADAM) {
      const double tt = (double)((A.defer ? sm_dec.adam_t : ctrl->adam_t) + 1);
      bc1 = (float)(1.0 / (1.0 - pow((double)A.h.gv, tt)));
      bc2 = (float)(1.0 / (1.0 - pow((double)A.h.gs, tt)));
    }
    for (int k = 0; k < my_units; ++k) {
      const int u = blockIdx.x + k * grid;
      const int s = k % kStages;
      unsigned char* st = smem_raw + s * SL::BYTES;
      const uint32_t par = (uint32_t)(k / kStages) & 1;
      mbar_wait(&bar_r[s], par);
      mbar_wait(&bar_a[s], par);
      mbar_wait(&bar_b[s], par);
    const int packed = meta[s].packed;
      const int lgG = packed & 7, G = 1 << lgG;
      const int lg = tid & (G - 1), grp = tid >> lgG;
      const int va = meta[s].va, nv = meta[s].nv;
      const uint32_t* rp = reinterpret_cast<const uint32_t*>(st + SL::RP_OFF);
      const uint32_t* colst = reinterpret_cast<const uint32_t*>(st + SL::COL_OFF);
      const float* ys = reinterpret_cast<const float*>(st + SL::Y_OFF);
      const float* ss = reinterpret_cast<const float*>(st + SL::S_OFF);
      const bool staged = meta[s].staged != 0;
      const uint32_t e0 = rp[0];
      const int coff = meta[s].col_off;

      float acc_e = 0.f, acc_n = 0.f, acc_o = 0.f, acc_bad = 0.f;
      const bool active = grp < nv;
      if (active) {
        const long long v = va + grp;
        const uint32_t beg = rp[grp], end = rp[grp + 1];
        float yi[DIM], li[DIM];
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          yi[d] = ys[grp * YS + d];
          li[d] = NEST ? ys[grp * YS + (DIM == 2 ? 2 : 4) + d] : yi[d];
        }
        float f[DIM];
#pragma unroll
        for (int d = 0; d < DIM; ++d) f[d] = 0.f;
        float e = 0.f;
        constexpr bool kFast = DIM == 2 && !WEIGHTED && NORM == 0 && !NEST;
        const int slots = (packed >> 3) & 15;  // per lane: ceil(tile max degree / G), 15 = more
        bool fast = false;
        if constexpr (kFast) fast = true;
        if (fast) {
          if constexpr (kFast) {
            const int deg = (int)(end - beg);
            const int nl = deg > lg ? (deg - lg + G - 1) >> lgG : 0;  // this lane's entries
            float ff[2] = {0.f, 0.f};
            auto run = [&](auto gcol_tag, const uint32_t* cb) {
              constexpr bool GC = decltype(gcol_tag)::value;
              if (slots <= 8) {
                switch (slots) {
#define IVHD_FAST_CASE(D) \
  case D: fast_row<D, GC>(A, needp, cb, G, nl, lg, Yin, (uint32_t)v, yi[0], yi[1], c, gstep, ff, e); break;
                  IVHD_FAST_CASE(1) IVHD_FAST_CASE(2) IVHD_FAST_CASE(3) IVHD_FAST_CASE(4)
                  IVHD_FAST_CASE(5) IVHD_FAST_CASE(6) IVHD_FAST_CASE(7) IVHD_FAST_CASE(8)
#undef IVHD_FAST_CASE
                  default: break;
                }
              } else {
                for (int c0 = 0; c0 < nl; c0 += 8)
                  fast_row<8, GC>(A, needp, cb + c0 * G, G, nl - c0, lg + c0 * G, Yin, (uint32_t)v, yi[0], yi[1], c,
                                  gstep, ff, e);
              }
            };
            if (staged) run(std::false_type{}, colst + (beg - e0 + coff) + lg);
            else run(std::true_type{}, A.col + beg + lg);
            f[0] = ff[0];
            f[1] = ff[1];
          }
        } else
        for (uint32_t k0 = beg + lg; k0 < end; k0 += (uint32_t)G * kUnroll) {
          uint32_t cw[kUnroll];
          float2 tw[WEIGHTED ? kUnroll : 1];
          float gy[kUnroll][DIM], gl[kUnroll][DIM];
          // A slot past the row end becomes a zero-target pair with the vertex
          // itself: zero distance, zero force, zero stress — no masking needed.
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            const uint32_t kk = k0 + (uint32_t)(q * G);
            cw[q] = (uint32_t)v;
            if (kk < end) cw[q] = staged ? colst[kk - e0 + coff] : ld_col(A.col + kk);
          }
          if constexpr (WEIGHTED) {
#pragma unroll
            for (int q = 0; q < kUnroll; ++q) {
              const uint32_t kk = k0 + (uint32_t)(q * G);
              tw[q] = make_float2(0.f, 1.f);
              if (kk < end) tw[q] = __ldg(A.ew + kk);
            }
          }
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
#pragma unroll
            for (int d = 0; d < DIM; ++d) {
              gy[q][d] = yi[d];
              gl[q][d] = li[d];
            }
            if (k0 + (uint32_t)(q * G) < end) gather<DIM, NEST>(Yin, cw[q] & kIdMask, gy[q], gl[q]);
          }
          unsigned dmask = 0;
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            float2 twq = make_float2(0.f, 0.f);
            if constexpr (WEIGHTED) twq = tw[q];
            if (entry<DIM, NEST, NORM>(yi, li, gy[q], gl[q], cw[q], WEIGHTED, twq, c, true, f, e)) dmask |= 1u << q;
          }
          if (dmask) {  // degenerate random pairs (forces.py:167-174): measure-zero path
#pragma unroll
            for (int q = 0; q < kUnroll; ++q) {
              if ((dmask >> q) & 1u) {
                float uvec[DIM];
                degenerate_vec<DIM>(A, needp, (uint32_t)v, (int)(k0 + (uint32_t)(q * G) - beg), gstep, uvec);
#pragma unroll
                for (int d = 0; d < DIM; ++d) f[d] += uvec[d];
              }
            }
          }
        }
        // fixed xor butterfly over the G lanes of the group (G uniform per unit);
        // the mask names exactly this group's lanes (the walk leaves the warp diverged)
        if (G > 1) {
          const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << ((tid & 31) & ~(G - 1));
          for (int o = G >> 1; o > 0; o >>= 1) {
#pragma unroll
            for (int d = 0; d < DIM; ++d) f[d] += __shfl_xor_sync(gmask, f[d], o);
            e += __shfl_xor_sync(gmask, e, o);
          }
        }
        if (lg == 0) {
          acc_e = e;
          if constexpr (OPT == OPT_NONE) {
#pragma unroll
            for (int d = 0; d < DIM; ++d) A.force_out[(size_t)v * DIM + d] = (double)f[d];
          } else {
            float sv[SSX];
#pragma unroll
            for (int q = 0; q < SSX; ++q) sv[q] = L::SS > 0 ? ss[grp * SSX + q] : 0.f;
            apply_update<DIM, OPT, PEER>(A, Yout, Sout, v, yi, sv, f, step, bc1, bc2, acc_n, acc_o, acc_bad);
          }
        }
      }
      if (A.fuse_finalize) {
        // single GPU: running per-thread sums (fixed vertex order); the block
        // reduces them once after its last unit
        te += acc_e; tn += acc_n; to += acc_o; tb += acc_bad;
        if ((k & 63) == 63) flush_partials();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_e[s]);  // this warp is done with stage s
        if (k < 34) IVHD_TL(2 + k);
        continue;
      }
      // sharded: per-unit partials (rank-count independent order).  Warp
      // partial by a fixed butterfly; the warp that completes the unit sums
      // the 8 warp partials in warp order into the unit partial.
      double pe = acc_e, pn = acc_n, po = acc_o, pb = acc_bad;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        pe += __shfl_xor_sync(0xffffffffu, pe, o);
        pn += __shfl_xor_sync(0xffffffffu, pn, o);
        po += __shfl_xor_sync(0xffffffffu, po, o);
        pb += __shfl_xor_sync(0xffffffffu, pb, o);
      }
      if (lane == 0) {
        sm_wp[s][warp] = make_double4(pe, pn, po, pb);
        __threadfence_block();
        if (atomicAdd(&sm_cnt[s], 1) == kConsumerWarps - 1) {
          __threadfence_block();
          double4 t = make_double4(0, 0, 0, 0);
#pragma unroll
          for (int w = 0; w < kConsumerWarps; ++w) {
            const double4 q = sm_wp[s][w];
            t.x += q.x; t.y += q.y; t.z += q.z; t.w += q.w;
          }
          A.partial[A.tile0 + u] = t;
          sm_cnt[s] = 0;
          __threadfence_block();
        }
        mbar_arrive(&bar_e[s]);  // this warp is done with stage s
      }
      __syncwarp();
    }
  }

  if (!A.fuse_finalize) return;
  IVHD_TL(38);
  // block partial: warp sums in a fixed butterfly, then warps in order
  block_sync();
  IVHD_TL(36);
  if (warp < kConsumerWarps) flush_partials();  // the last (partial) group of units
  block_sync();
  if (warp != 0) return;
  if (A.defer) {  // the block partial into this launch's slot; the next launch decides
    if (lane == 0) {
      double4 t = make_double4(0, 0, 0, 0);
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) {
        t.x += sm_wacc[w].x; t.y += sm_wacc[w].y; t.z += sm_wacc[w].z; t.w += sm_wacc[w].w;
      }
      fix_add(ctrl, sm_df[0], t);
    }
    return;
  }
  // last-block-done: lane 0 publishes the block partial with a release
  // arrival; the block that arrives last (acquire) reduces and decides
  int last = 0;
  if (lane == 0) {
    double4 t = make_double4(0, 0, 0, 0);
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) {
      t.x += sm_wacc[w].x; t.y += sm_wacc[w].y; t.z += sm_wacc[w].z; t.w += sm_wacc[w].w;
    }
    A.bpart[blockIdx.x] = t;
    if constexpr (PEER) {  // this block's P2P position stores first (none with one rank)
      if (A.pe.n_peers > 0) fence_release_sys();
    }
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(&ctrl->arrive) : "memory");
    last = old == gridDim.x - 1;
  }
  IVHD_TL(37);
  if (!__shfl_sync(0xffffffffu, last, 0)) return;
  __syncwarp();
  if constexpr (PEER) {
    peer_rank_publish(A, (int)gridDim.x);
    if (A.pe.decide_here) peer_decide<OPT>(A);  // ranks on separate GPUs: no finalizer launch
    else if (lane == 0) ctrl->arrive = 0;       // the finalizer kernel decides (in-process emulation)
    IVHD_TL(39);
    return;
  }
  finalize_warp<OPT>(A, A.bpart, (int)gridDim.x);
  IVHD_TL(39);
}

// Peer-mode finalizer for ranks that share one GPU (in-process emulation:
// every rank's step kernel runs before any finalizer, so nothing waits on a
// kernel that has not run).  One warp: peer_decide.
template <int OPT>
__global__ void __launch_bounds__(32) finalize_peer_kernel(StepArgs A) {
  if (threadIdx.x == 0) griddep_launch_dependents();  // the next step may stage its graph constants
  griddep_wait();
  if (A.ctrl->status != 0) return;
  peer_decide<OPT>(A);
}

// Standalone finalizer (sharded mode, after the exchange): one block.
template <int OPT>
__global__ void __launch_bounds__(kBlock) finalize_kernel(StepArgs A) {
  __shared__ double4 sm_red[kBlock / 32];
  if (A.ctrl->status != 0) return;
  finalize_block<OPT>(A, sm_red, A.tpart, A.n_tiles_global);
  if (!A.fixed_io) return;
  // async sharded mode: the buffer just written becomes current; after a
  // rollback (rare) it is refilled with the unchanged positions
  block_sync();  // CTA-scope ordering after thread 0's decision
  const volatile Ctrl* vc = A.ctrl;
  if (vc->status != 0 || vc->last_commit) return;
  const float4* src = reinterpret_cast<const float4*>(A.ybuf0);
  float4* dst = reinterpret_cast<float4*>(A.ybuf1);
  const long long n4 = (A.v_cap_floats + 3) / 4;
  for (long long i = threadIdx.x; i < n4; i += kBlock) dst[i] = src[i];
}

}  // namespace ivhd
