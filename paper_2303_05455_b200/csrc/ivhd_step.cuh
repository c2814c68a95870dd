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
// Work mapping: a block of 256 threads takes fixed-size vertex tiles from a
// dynamic tile counter; inside a tile G lanes cooperate on one vertex (its
// symmetrised CSR row), reduce with a fixed xor-butterfly (all lanes get the
// bit-identical sum), and lane 0 of the group applies the optimizer.  No
// atomics touch the data; the last block to finish reduces the tile partials
// in fixed order and writes the decision (cur buffer, b, trace, status) that
// the next launch reads.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ivhd {


constexpr int kBlock = 256;

// Block barrier.  __syncthreads() lowers to the *aligned* bar.sync, which
// assumes every warp arrives converged; after the data-dependent merge-path
// walk, lanes of one warp can arrive separately (independent thread
// scheduling) and the aligned barrier then let early lanes through (observed
// on B200 / CUDA 12.9).  The non-aligned barrier.sync counts threads.
__device__ __forceinline__ void block_sync() { asm volatile("barrier.sync 0;" ::: "memory"); }

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
};

struct Hyper {
  float a, g1, g2;       // force-directed
  float beta, gv, gs, rho, eps;
  double tau;
  int adapt;
};

struct StepArgs {
  const uint32_t* row_ptr;
  const uint32_t* col;
  const float2* ew;       // nullptr in binary mode
  float* ybuf0;
  float* ybuf1;
  float* state;
  double4* partial;
  double2* trace;
  Ctrl* ctrl;
  double* force_out;      // OPT_NONE only: (M, DIM) float64
  long long v_begin, v_end;
  int tile_v;
  int n_tiles;            // tiles this launch processes
  int tile0;              // global index of its first tile
  int n_tiles_global;     // tiles reduced by the finalizer
  int norm;               // 0 = L2, 1 = L1
  int fuse_finalize;      // last block reduces + decides (single GPU)
  Hyper h;
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
// forces.py:167-174 draws a random unit direction (magnitude w*t) for random
// pairs at exactly zero distance.  On the device the direction comes from a
// counter-based hash of (min id, max id, global step) so both endpoint rows
// of the pair see the same direction with opposite signs (measure-zero path).
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27; x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

template <int DIM>
__device__ __noinline__ void degenerate_dir(uint32_t i, uint32_t j, long long step, float (&u)[DIM]) {
  const uint32_t lo = min(i, j), hi = max(i, j);
  uint64_t h = mix64(((uint64_t)lo << 32 | hi) ^ mix64((uint64_t)step + 0x9e3779b97f4a7c15ull));
  const float r0 = (float)(h >> 40) * (1.0f / 16777216.0f);
  const float r1 = (float)((h >> 16) & 0xffffff) * (1.0f / 16777216.0f);
  const float sgn = (i == lo) ? 1.f : -1.f;
  float s, c;
  sincospif(2.f * r0, &s, &c);
  if constexpr (DIM == 2) {
    u[0] = sgn * c; u[1] = sgn * s;
  } else {
    const float z = 2.f * r1 - 1.f, rho = sqrtf(fmaxf(0.f, 1.f - z * z));
    u[0] = sgn * rho * c; u[1] = sgn * rho * s; u[2] = sgn * z;
  }
  if (i == j) {
    for (int d = 0; d < DIM; ++d) u[d] = 0.f;  // self pair: +comp and -comp cancel
  }
}

// ------------------------------------------------------------------ entries
// Contribution of one symmetrised-CSR entry to row i (forces.py:97-124):
//   L2: phi = -w (t == 0) | w (t - d)/d ; f += phi (y_i - y_o);  e += w (t-d)^2
//   L1: f += sign(y_i - y_o) w (t - d);                           e += w (t-d)^2
template <int DIM, bool NEST>
__device__ __forceinline__ void entry(const float (&yi)[DIM], const float (&li)[DIM],
                                      const float (&yo)[DIM], const float (&lo)[DIM],
                                      uint32_t cw, bool weighted, float2 tw,
                                      float c, int norm, uint32_t i, long long step,
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
  if (norm == 0) {
    const float dist = sqrtf(d2);
    if (t == 0.f) {
#pragma unroll
      for (int d = 0; d < DIM; ++d) f[d] = fmaf(-w, df[d], f[d]);
    } else if (dist > 0.f) {
      const float phi = w * (t - dist) / dist;
#pragma unroll
      for (int d = 0; d < DIM; ++d) f[d] = fmaf(phi, df[d], f[d]);
    } else if (dist == 0.f) {
      float u[DIM];
      degenerate_dir<DIM>(i, cw & kIdMask, step, u);
#pragma unroll
      for (int d = 0; d < DIM; ++d) f[d] = fmaf(w * t, u[d], f[d]);
    } else {  // NaN distance: propagate like the reference's factor
#pragma unroll
      for (int d = 0; d < DIM; ++d) f[d] += dist;
    }
  } else {
    const float s = w * (t - d1);
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const float sg = df[d] > 0.f ? 1.f : (df[d] < 0.f ? -1.f : (df[d] == 0.f ? 0.f : df[d]));
      f[d] = fmaf(sg, s, f[d]);
    }
  }
  // stress at the current (not look-ahead) positions: engine.py:370
  float dist_e;
  if constexpr (NEST) {
    float q2 = 0.f, q1 = 0.f;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const float q = yi[d] - yo[d];
      q2 = fmaf(q, q, q2);
      q1 += fabsf(q);
    }
    dist_e = norm == 0 ? sqrtf(q2) : q1;
  } else {
    dist_e = norm == 0 ? sqrtf(d2) : d1;
  }
  const float r = t - dist_e;
  e = fmaf(w * r, r, e);
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
  block_sync();
  double4 r = make_double4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int w = 0; w < kBlock / 32; ++w) {
      r.x += sm[w].x; r.y += sm[w].y; r.z += sm[w].z; r.w += sm[w].w;
    }
  }
  block_sync();
  return r;  // valid in thread 0
}

// ---------------------------------------------------------------- finalize
// Reduce all tile partials in a fixed order and take the iteration decision
// (optim.py:80-92 + engine.py:373-384).  Executed by ONE whole block; each
// thread keeps 8 tiles in flight so the tail is ~one memory round trip.
template <int OPT>
__device__ void finalize_block(const StepArgs& A, double4* sm) {
  Ctrl* ctrl = A.ctrl;
  const double2* p2 = reinterpret_cast<const double2*>(A.partial);
  double4 s = make_double4(0, 0, 0, 0);
  for (int t0 = threadIdx.x; t0 < A.n_tiles_global; t0 += 8 * kBlock) {
    double2 a[8], b[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int t = t0 + u * kBlock;
      if (t < A.n_tiles_global) {
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
  if (threadIdx.x == 0) {
    const double E = 0.5 * s.x;
    double step = ctrl->step;
    bool commit = true;
    if (OPT == OPT_FD && A.h.adapt) {
      const double dT = s.y - s.z;
      if (dT > A.h.tau) {
        step *= (double)A.h.g2;
        commit = false;
      } else if (dT < -A.h.tau) {
        step *= (double)A.h.g1;
        commit = false;
      }
    }
    const long long it = ctrl->iter;
    if (A.trace) A.trace[it] = make_double2(E, step);
    if (commit && s.w > 0.0) {
      ctrl->status = 1;
      ctrl->diverged_at = it;
    } else {
      if (commit) ctrl->cur ^= 1;
      ctrl->last_commit = commit ? 1 : 0;
      ctrl->step = step;
      ctrl->iter = it + 1;
    }
    ctrl->gstep += 1;
    if (OPT == OPT_ADAM) ctrl->adam_t += 1;
    ctrl->next_tile = 0;
    __threadfence();
    ctrl->arrive = 0;
  }
}

// ---------------------------------------------------------- merge path
// Tile-local merge path of row ends (s_re[r] = end of row r, local entry
// index) and entries: row-end r sits at diagonal s_re[r] + r.  Returns the
// number of rows whose end item lies before diagonal d.
__device__ __forceinline__ int merge_search(const uint32_t* s_re, int nrows, int d) {
  int lo = 0, hi = nrows;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((int)s_re[mid] + mid < d) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
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
template <int DIM, int OPT>
__device__ __forceinline__ void apply_update(const StepArgs& A, float* __restrict__ Yout, long long v,
                                             const float (&yi)[DIM], float (&sv)[Layout<DIM, OPT>::SS > 0 ? Layout<DIM, OPT>::SS : 1],
                                             const float (&f)[DIM], float step, float bc1, float bc2,
                                             double& acc_n, double& acc_o, double& acc_bad) {
  using L = Layout<DIM, OPT>;
  constexpr int V = DIM == 2 ? 2 : 4;
  float yn[DIM];
  if constexpr (OPT == OPT_FD) {
    double so = 0.0, sn = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const float dn = fmaf(A.h.a, sv[d], step * f[d]);
      so += (double)sv[d] * (double)sv[d];
      sn += (double)dn * (double)dn;
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
  if constexpr (L::SS > 0) st_state<L::SS>(A.state + (size_t)v * L::SS, sv);
  if constexpr (OPT == OPT_NEST) {
    float la[DIM];
#pragma unroll
    for (int d = 0; d < DIM; ++d) la[d] = yn[d] + A.h.beta * sv[d];  // optim.py:174-175
    if constexpr (DIM == 2) {
      *reinterpret_cast<float4*>(Yout + (size_t)v * 4) = make_float4(yn[0], yn[1], la[0], la[1]);
    } else {
      *reinterpret_cast<float4*>(Yout + (size_t)v * 8) = make_float4(yn[0], yn[1], yn[2], 0.f);
      *reinterpret_cast<float4*>(Yout + (size_t)v * 8 + 4) = make_float4(la[0], la[1], la[2], 0.f);
    }
  } else {
    st_vec<DIM>(Yout + (size_t)v * L::YS, yn);
  }
  acc_bad += all_finite(yn, DIM) ? 0.0 : 1.0;
}

// Store one row partial produced by a thread walking entries [js, je):
// complete rows go to s_row[r]; a row that starts here and continues goes to
// s_tail[tid]; a row continued from an earlier thread goes to s_head[tid].
template <int DIM>
__device__ __forceinline__ void emit_row(int r, const float (&f)[DIM], float e, int js, int je,
                                         const uint32_t* s_re, float4* s_row, float4* s_head,
                                         float4* s_tail) {
  const int rs = r > 0 ? (int)s_re[r - 1] : 0;
  const int re = (int)s_re[r];
  const bool started = rs >= js;
  float4* dst = started ? (re <= je ? &s_row[r] : &s_tail[threadIdx.x]) : &s_head[threadIdx.x];
  if constexpr (DIM == 2) *dst = make_float4(f[0], f[1], e, 0.f);
  else *dst = make_float4(f[0], f[1], f[2], e);
}

// ------------------------------------------------------------------ kernel
// Tile = TV = 256*RPT consecutive vertices.  Its rows' entries are walked as
// one merge path of (row ends + entries); each thread owns P consecutive
// items, so its column loads and position gathers are issued as one batch
// and hub rows are split evenly across threads.  A row touching several
// threads is summed as tail(first thread) + head(next) + ... in thread
// order (deterministic); rows spanning a round of 256*P items carry over in
// s_carry.  The thread owning row r (r mod 256) applies the optimizer.
template <int DIM, int OPT, int RPT, int P, bool WEIGHTED>
__global__ void __launch_bounds__(kBlock, 2) step_kernel(StepArgs A) {
  using L = Layout<DIM, OPT>;
  constexpr bool NEST = (OPT == OPT_NEST);
  constexpr int TV = kBlock * RPT;
  constexpr int ITEMS = kBlock * P;
  constexpr int YS = L::YS;
  constexpr int SSX = L::SS > 0 ? L::SS : 1;

  __shared__ __align__(16) float s_y[TV * YS];
  __shared__ float4 s_row[TV];
  __shared__ float4 s_head[kBlock];
  __shared__ float4 s_tail[kBlock];
  __shared__ uint32_t s_re[TV];
  __shared__ float4 s_carry[2];  // double-buffered by round parity
  __shared__ double4 sm_red[kBlock / 32];
  __shared__ int sm_tile;

  Ctrl* ctrl = A.ctrl;
  if (ctrl->status != 0) return;  // diverged earlier: later iterations are no-ops
  const int cur = ctrl->cur;
  const float c = (float)ctrl->c;
  const float step = (float)ctrl->step;
  const long long gstep = ctrl->gstep;
  const float* __restrict__ Yin = cur ? A.ybuf1 : A.ybuf0;
  float* __restrict__ Yout = cur ? A.ybuf0 : A.ybuf1;
  const int tid = threadIdx.x;

  float bc1 = 1.f, bc2 = 1.f;  // Adam bias corrections (optim.py:203-204)
  if constexpr (OPT == OPT_ADAM) {
    const double tt = (double)(ctrl->adam_t + 1);
    bc1 = (float)(1.0 / (1.0 - pow((double)A.h.gv, tt)));
    bc2 = (float)(1.0 / (1.0 - pow((double)A.h.gs, tt)));
  }

  while (true) {
    if (tid == 0) sm_tile = (int)atomicAdd(&ctrl->next_tile, 1u);
    block_sync();
    const int tile = sm_tile;
    if (tile >= A.n_tiles) break;
    const long long v0 = A.v_begin + (long long)tile * TV;
    const int nrows = (int)max(0LL, min((long long)TV, A.v_end - v0));
    double acc_e = 0.0, acc_n = 0.0, acc_o = 0.0, acc_bad = 0.0;

    if (nrows > 0) {
      // ---- round trip 1: row ends, the tile's positions, owners' state
      const uint32_t e0 = __ldg(A.row_ptr + v0);
      for (int r = tid; r < nrows; r += kBlock) s_re[r] = __ldg(A.row_ptr + v0 + r + 1) - e0;
      if constexpr (YS % 4 == 0) {
        const float4* src = reinterpret_cast<const float4*>(Yin + (size_t)v0 * YS);
        for (int q = tid; q < nrows * YS / 4; q += kBlock) reinterpret_cast<float4*>(s_y)[q] = __ldg(src + q);
      } else {
        const float2* src = reinterpret_cast<const float2*>(Yin + (size_t)v0 * YS);
        for (int q = tid; q < nrows * YS / 2; q += kBlock) reinterpret_cast<float2*>(s_y)[q] = __ldg(src + q);
      }
      float sv[RPT][SSX];
#pragma unroll
      for (int kk = 0; kk < RPT; ++kk) {
        const int r = tid + kk * kBlock;
        if constexpr (L::SS > 0) {
          if (r < nrows) ld_state<L::SS>(A.state + (size_t)(v0 + r) * L::SS, sv[kk]);
        }
      }
      block_sync();
      const int E = (int)s_re[nrows - 1];
      const int total = nrows + E;

      for (int base = 0, round = 0; base < total; base += ITEMS, ++round) {
        const float4* carry_in = &s_carry[round & 1];
        const int d0 = min(base + tid * P, total), d1 = min(d0 + P, total);
        const int i0 = merge_search(s_re, nrows, d0);
        const int i1 = merge_search(s_re, nrows, d1);
        const int js = d0 - i0, ne = (d1 - i1) - js;
        const int je = js + ne;
        // ---- round trip 2 + 3: this thread's entries, then their positions
        uint32_t cw[P];
        float2 tw[WEIGHTED ? P : 1];
        float gy[P][DIM], gl[P][DIM];
#pragma unroll
        for (int q = 0; q < P; ++q)
          if (q < ne) cw[q] = __ldg(A.col + e0 + js + q);
        if constexpr (WEIGHTED) {
#pragma unroll
          for (int q = 0; q < P; ++q)
            if (q < ne) tw[q] = __ldg(A.ew + e0 + js + q);
        }
#pragma unroll
        for (int q = 0; q < P; ++q)
          if (q < ne) gather<DIM, NEST>(Yin, cw[q] & kIdMask, gy[q], gl[q]);
        // ---- walk: accumulate per row, emit at row changes
        int cr = i0;
        bool open = false;
        float f[DIM];
        float e = 0.f;
#pragma unroll
        for (int d = 0; d < DIM; ++d) f[d] = 0.f;
#ifdef IVHD_NOUNROLL_WALK
#pragma unroll 1
#else
#pragma unroll
#endif
        for (int q = 0; q < P; ++q) {
          if (q < ne) {
            const int j = js + q;
            int r = cr;
            while ((int)s_re[r] <= j) ++r;
            if (open && r != cr) {
              emit_row<DIM>(cr, f, e, js, je, s_re, s_row, s_head, s_tail);
#pragma unroll
              for (int d = 0; d < DIM; ++d) f[d] = 0.f;
              e = 0.f;
            }
            cr = r;
            open = true;
            float yi[DIM], li[DIM];
            const float* ys = s_y + r * YS;
#pragma unroll
            for (int d = 0; d < DIM; ++d) {
              yi[d] = ys[d];
              li[d] = NEST ? ys[(DIM == 2 ? 2 : 4) + d] : ys[d];
            }
            float2 twq = make_float2(0.f, 0.f);
            if constexpr (WEIGHTED) twq = tw[q];
            entry<DIM, NEST>(yi, li, gy[q], gl[q], cw[q], WEIGHTED, twq,
                             c, A.norm, (uint32_t)(v0 + r), gstep, f, e);
          }
        }
        if (open) emit_row<DIM>(cr, f, e, js, je, s_re, s_row, s_head, s_tail);
        block_sync();

        // ---- resolve the rows whose end item lies in this round
        auto chain = [&](int r, int tlast) {
          const int rs = r > 0 ? (int)s_re[r - 1] : 0;
          const int da = rs + r;
          int t;
          float4 sum;
          if (da >= base) {
            t = (da - base) / P;
            sum = s_tail[t];
          } else {
            t = -1;
            sum = *carry_in;
          }
          for (++t; t <= tlast; ++t) sum = f4add(sum, s_head[t]);
          return sum;
        };
#pragma unroll
        for (int kk = 0; kk < RPT; ++kk) {
          const int r = tid + kk * kBlock;
          if (r >= nrows) continue;
          const int pe = (int)s_re[r] + r;
          if (pe < base || pe >= base + ITEMS) continue;
          const int rs = r > 0 ? (int)s_re[r - 1] : 0;
          const int re = (int)s_re[r];
          float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
          if (re > rs) {
            const int da = rs + r, db = re - 1 + r;
            if (da / P == db / P) sum = s_row[r];
            else sum = chain(r, db >= base ? (db - base) / P : -1);
          }
          float fr[DIM];
          fr[0] = sum.x;
          fr[1] = sum.y;
          if constexpr (DIM == 3) fr[2] = sum.z;
          acc_e += (double)(DIM == 2 ? sum.z : sum.w);
          const long long v = v0 + r;
          if constexpr (OPT == OPT_NONE) {
#pragma unroll
            for (int d = 0; d < DIM; ++d) A.force_out[(size_t)v * DIM + d] = (double)fr[d];
          } else {
            float yi[DIM];
#pragma unroll
            for (int d = 0; d < DIM; ++d) yi[d] = s_y[r * YS + d];
            apply_update<DIM, OPT>(A, Yout, v, yi, sv[kk], fr, step, bc1, bc2, acc_n, acc_o, acc_bad);
          }
        }
        // ---- carry the row that is still open at the round boundary
        if (tid == 0 && base + ITEMS < total) {
          const int ib = merge_search(s_re, nrows, base + ITEMS);
          const int jb = base + ITEMS - ib;
          const int rs = ib > 0 ? (int)s_re[ib - 1] : 0;
          if (ib < nrows && jb > rs) {
            const int da = rs + ib, db = (int)s_re[ib] - 1 + ib;
            if (da / P != db / P) s_carry[(round + 1) & 1] = chain(ib, (jb - 1 + ib - base) / P);
          }
        }
        block_sync();
      }
    }
    const double4 tot = block_sum4(make_double4(acc_e, acc_n, acc_o, acc_bad), sm_red);
    if (tid == 0) A.partial[A.tile0 + tile] = tot;
  }

  if (!A.fuse_finalize) return;
  // last-block-done: the block that retires last reduces and decides
  __shared__ bool sm_last;
  __threadfence();
  block_sync();
  if (tid == 0) sm_last = (atomicAdd(&ctrl->arrive, 1u) == gridDim.x - 1);
  block_sync();
  if (!sm_last) return;
  __threadfence();
  finalize_block<OPT>(A, sm_red);
}

// Standalone finalizer (sharded mode, after the exchange): one block.
template <int OPT>
__global__ void __launch_bounds__(kBlock) finalize_kernel(StepArgs A) {
  __shared__ double4 sm_red[kBlock / 32];
  if (A.ctrl->status != 0) return;
  finalize_block<OPT>(A, sm_red);
}

// Items per thread: sized so the batched gathers fit in registers.
template <int DIM, int OPT> struct ItemsPerThread {
  static constexpr int value = (OPT == OPT_NEST) ? (DIM == 2 ? 6 : 4) : (DIM == 2 ? 12 : 6);
};

}  // namespace ivhd
