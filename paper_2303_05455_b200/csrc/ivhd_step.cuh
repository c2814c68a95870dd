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
  const uint8_t* tile_g;  // lanes per vertex of every (global) tile
  const int* units;       // work unit -> (tile << 6) | pass, global unit order
  long long v_begin, v_end;
  int tile_v;
  int n_tiles;            // work units this launch processes
  int tile0;              // global index of its first work unit
  int n_tiles_global;     // work-unit partials reduced by the finalizer
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

// ------------------------------------------------------------------ kernel
// Vertices are relabelled by degree at setup (ivhd_capi.cu), so the 256
// consecutive vertices of a tile have near-equal degree.  Each tile carries
// G = lanes per vertex (1, 2, 4, ..., 32; G * kUnroll >= its max degree
// except for hubs): G lanes walk one CSR row with kUnroll independent column
// loads and position gathers in flight each, reduce with a fixed xor
// butterfly, and lane 0 applies the optimizer.  The only block barrier is
// the per-tile partial reduction.
constexpr int kUnroll = 8;

template <int DIM, int OPT, bool WEIGHTED>
__global__ void __launch_bounds__(kBlock, 3) step_kernel(StepArgs A) {
  using L = Layout<DIM, OPT>;
  constexpr bool NEST = (OPT == OPT_NEST);
  constexpr int SSX = L::SS > 0 ? L::SS : 1;
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

  // Work unit = one pass of a tile: 256/G vertices with G lanes each.  Heavy
  // tiles (large G) thus spread over many blocks instead of serialising G
  // passes in one; each unit writes its own partial (fixed unit order).
  while (true) {
    if (tid == 0) sm_tile = (int)atomicAdd(&ctrl->next_tile, 1u);
    block_sync();
    const int unit = sm_tile;
    if (unit >= A.n_tiles) break;
    const int packed = __ldg(A.units + A.tile0 + unit);
    const int tile = packed >> 6, pass = packed & 63;
    const long long v0 = (long long)tile * kBlock;
    const int G = A.tile_g[tile];
    const int lgG = __ffs(G) - 1;
    const int lg = tid & (G - 1);
    const int grp = tid >> lgG;
    const int groups = kBlock >> lgG;
    double acc_e = 0.0, acc_n = 0.0, acc_o = 0.0, acc_bad = 0.0;

    {
      const long long v = v0 + (long long)pass * groups + grp;
      const bool active = v < A.v_end;
      uint32_t beg = 0, end = 0;
      float yi[DIM], li[DIM], sv[SSX];
      if (active) {
        beg = __ldg(A.row_ptr + v);
        end = __ldg(A.row_ptr + v + 1);
        gather<DIM, NEST>(Yin, (uint32_t)v, yi, li);
        if constexpr (L::SS > 0) {
          if (lg == 0) ld_state<L::SS>(A.state + (size_t)v * L::SS, sv);
        }
      } else {
#pragma unroll
        for (int d = 0; d < DIM; ++d) yi[d] = li[d] = 0.f;
      }
      float f[DIM];
#pragma unroll
      for (int d = 0; d < DIM; ++d) f[d] = 0.f;
      float e = 0.f;
      for (uint32_t k0 = beg + lg; k0 < end; k0 += (uint32_t)G * kUnroll) {
        uint32_t cw[kUnroll];
        float2 tw[WEIGHTED ? kUnroll : 1];
        float gy[kUnroll][DIM], gl[kUnroll][DIM];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint32_t k = k0 + (uint32_t)(u * G);
          if (k < end) cw[u] = __ldg(A.col + k);
        }
        if constexpr (WEIGHTED) {
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const uint32_t k = k0 + (uint32_t)(u * G);
            if (k < end) tw[u] = __ldg(A.ew + k);
          }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint32_t k = k0 + (uint32_t)(u * G);
          if (k < end) gather<DIM, NEST>(Yin, cw[u] & kIdMask, gy[u], gl[u]);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint32_t k = k0 + (uint32_t)(u * G);
          if (k < end) {
            float2 twu = make_float2(0.f, 0.f);
            if constexpr (WEIGHTED) twu = tw[u];
            entry<DIM, NEST>(yi, li, gy[u], gl[u], cw[u], WEIGHTED, twu, c, A.norm, (uint32_t)v,
                             gstep, f, e);
          }
        }
      }
      // fixed xor butterfly over the G lanes of the group (G uniform per tile)
      for (int o = G >> 1; o > 0; o >>= 1) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) f[d] += __shfl_xor_sync(0xffffffffu, f[d], o);
        e += __shfl_xor_sync(0xffffffffu, e, o);
      }
      if (active && lg == 0) {
        acc_e += (double)e;
        if constexpr (OPT == OPT_NONE) {
#pragma unroll
          for (int d = 0; d < DIM; ++d) A.force_out[(size_t)v * DIM + d] = (double)f[d];
        } else {
          apply_update<DIM, OPT>(A, Yout, v, yi, sv, f, step, bc1, bc2, acc_n, acc_o, acc_bad);
        }
      }
    }
    const double4 tot = block_sum4(make_double4(acc_e, acc_n, acc_o, acc_bad), sm_red);
    if (tid == 0) A.partial[A.tile0 + unit] = tot;
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

}  // namespace ivhd
