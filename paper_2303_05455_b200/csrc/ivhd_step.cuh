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
                                      uint32_t cw, const float2* __restrict__ ew, uint32_t k,
                                      float c, int norm, uint32_t i, long long step,
                                      float (&f)[DIM], float& e) {
  const bool rn = cw & kRandBit;
  float t, w;
  if (ew == nullptr) {
    t = rn ? 1.f : 0.f;
    w = rn ? c : 1.f;
  } else {
    const float2 tw = __ldg(ew + k);
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

template <int G>
__device__ __forceinline__ float group_sum(float x) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
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
  __syncthreads();
  double4 r = make_double4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int w = 0; w < kBlock / 32; ++w) {
      r.x += sm[w].x; r.y += sm[w].y; r.z += sm[w].z; r.w += sm[w].w;
    }
  }
  __syncthreads();
  return r;  // valid in thread 0
}

// ---------------------------------------------------------------- finalize
// Reduce all tile partials in a fixed order and take the iteration decision
// (optim.py:80-92 + engine.py:373-384).  Executed by ONE whole block.
template <int OPT>
__device__ void finalize_block(const StepArgs& A, double4* sm) {
  Ctrl* ctrl = A.ctrl;
  double4 s = make_double4(0, 0, 0, 0);
  for (int t = threadIdx.x; t < A.n_tiles_global; t += kBlock) {
    const double2 p0 = __ldcg(reinterpret_cast<const double2*>(A.partial + t));
    const double2 p1 = __ldcg(reinterpret_cast<const double2*>(A.partial + t) + 1);
    s.x += p0.x; s.y += p0.y; s.z += p1.x; s.w += p1.y;
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

// ------------------------------------------------------------------ kernel

template <int DIM, int OPT, int G>
__global__ void __launch_bounds__(kBlock) step_kernel(StepArgs A) {
  using L = Layout<DIM, OPT>;
  constexpr bool NEST = (OPT == OPT_NEST);
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

  // Adam bias corrections (optim.py:200-204), fp64 like the reference's scalars.
  float bc1 = 1.f, bc2 = 1.f;
  if constexpr (OPT == OPT_ADAM) {
    const double tt = (double)(ctrl->adam_t + 1);
    bc1 = (float)(1.0 / (1.0 - pow((double)A.h.gv, tt)));
    bc2 = (float)(1.0 / (1.0 - pow((double)A.h.gs, tt)));
  }

  const int lg = threadIdx.x % G;
  const int grp = threadIdx.x / G;
  constexpr int kGroups = kBlock / G;

  while (true) {
    if (threadIdx.x == 0) sm_tile = (int)atomicAdd(&ctrl->next_tile, 1u);
    __syncthreads();
    const int tile = sm_tile;
    __syncthreads();
    if (tile >= A.n_tiles) break;
    const long long v0 = A.v_begin + (long long)tile * A.tile_v;
    const long long v1 = min(v0 + (long long)A.tile_v, A.v_end);

    double acc_e = 0.0, acc_n = 0.0, acc_o = 0.0, acc_bad = 0.0;
    // vb advances uniformly over the block so every lane reaches the group
    // shuffles; lanes past the tile end carry an empty row.
    for (long long vb = v0; vb < v1; vb += kGroups) {
      const long long v = vb + grp;
      const bool active = v < v1;
      uint32_t beg = 0, end = 0;
      float yi[DIM], li[DIM];
      if (active) {
        beg = __ldg(A.row_ptr + v);
        end = __ldg(A.row_ptr + v + 1);
        gather<DIM, NEST>(Yin, (uint32_t)v, yi, li);
      } else {
#pragma unroll
        for (int d = 0; d < DIM; ++d) yi[d] = li[d] = 0.f;
      }
      float f[DIM];
#pragma unroll
      for (int d = 0; d < DIM; ++d) f[d] = 0.f;
      float e = 0.f;
      uint32_t k = beg + lg;
      // two entries in flight per lane
      for (; k + G < end; k += 2 * G) {
        const uint32_t c0 = __ldg(A.col + k), c1 = __ldg(A.col + k + G);
        float y0[DIM], l0[DIM], y1[DIM], l1[DIM];
        gather<DIM, NEST>(Yin, c0 & kIdMask, y0, l0);
        gather<DIM, NEST>(Yin, c1 & kIdMask, y1, l1);
        entry<DIM, NEST>(yi, li, y0, l0, c0, A.ew, k, c, A.norm, (uint32_t)v, gstep, f, e);
        entry<DIM, NEST>(yi, li, y1, l1, c1, A.ew, k + G, c, A.norm, (uint32_t)v, gstep, f, e);
      }
      if (k < end) {
        const uint32_t c0 = __ldg(A.col + k);
        float y0[DIM], l0[DIM];
        gather<DIM, NEST>(Yin, c0 & kIdMask, y0, l0);
        entry<DIM, NEST>(yi, li, y0, l0, c0, A.ew, k, c, A.norm, (uint32_t)v, gstep, f, e);
      }
#pragma unroll
      for (int d = 0; d < DIM; ++d) f[d] = group_sum<G>(f[d]);
      e = group_sum<G>(e);
      if (!active || lg != 0) continue;
      acc_e += (double)e;

      // ------------------------------------------------ optimizer update
      if constexpr (OPT == OPT_NONE) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) A.force_out[(size_t)v * DIM + d] = (double)f[d];
      } else {
        float* st = A.state + (size_t)v * L::SS;
        float yn[DIM];
        if constexpr (OPT == OPT_FD) {
          // optim.py:113-124: delta <- a*delta + b*f; y <- y + delta (maybe rolled back)
          float dl[DIM], dn[DIM];
          ld_vec<DIM>(st, dl);
          double so = 0.0, sn = 0.0;
#pragma unroll
          for (int d = 0; d < DIM; ++d) {
            dn[d] = fmaf(A.h.a, dl[d], step * f[d]);
            yn[d] = yi[d] + dn[d];
            so += (double)dl[d] * (double)dl[d];
            sn += (double)dn[d] * (double)dn[d];
          }
          st_vec<DIM>(st, dn);
          acc_o += so;
          acc_n += sn;
        } else if constexpr (OPT == OPT_SGD) {
          // optim.py:140-141 with grad = -2 f (optim.py:259-263)
#pragma unroll
          for (int d = 0; d < DIM; ++d) yn[d] = yi[d] - step * (-2.f * f[d]);
        } else if constexpr (OPT == OPT_MOM || OPT == OPT_NEST) {
          // optim.py:161-163: v <- beta v - alpha g; y <- y + v
          float vv[DIM];
          ld_vec<DIM>(st, vv);
#pragma unroll
          for (int d = 0; d < DIM; ++d) {
            vv[d] = A.h.beta * vv[d] - step * (-2.f * f[d]);
            yn[d] = yi[d] + vv[d];
          }
          st_vec<DIM>(st, vv);
          if constexpr (NEST) {
            float la[DIM];
#pragma unroll
            for (int d = 0; d < DIM; ++d) la[d] = yn[d] + A.h.beta * vv[d];  // optim.py:174-175
            if constexpr (DIM == 2) {
              *reinterpret_cast<float4*>(Yout + (size_t)v * 4) = make_float4(yn[0], yn[1], la[0], la[1]);
            } else {
              *reinterpret_cast<float4*>(Yout + (size_t)v * 8) = make_float4(yn[0], yn[1], yn[2], 0.f);
              *reinterpret_cast<float4*>(Yout + (size_t)v * 8 + 4) = make_float4(la[0], la[1], la[2], 0.f);
            }
          }
        } else if constexpr (OPT == OPT_ADAM) {
          // optim.py:199-205
          float m1[DIM], m2[DIM];
          if constexpr (DIM == 2) {
            float4 s4 = *reinterpret_cast<const float4*>(st);
            m1[0] = s4.x; m1[1] = s4.y; m2[0] = s4.z; m2[1] = s4.w;
          } else {
            ld_vec<3>(st, m1);
            ld_vec<3>(st + 4, m2);
          }
#pragma unroll
          for (int d = 0; d < DIM; ++d) {
            const float g = -2.f * f[d];
            m1[d] = A.h.gv * m1[d] + (1.f - A.h.gv) * g;
            m2[d] = A.h.gs * m2[d] + (1.f - A.h.gs) * g * g;
            yn[d] = yi[d] - step * (m1[d] * bc1) / (A.h.eps + sqrtf(m2[d] * bc2));
          }
          if constexpr (DIM == 2) {
            *reinterpret_cast<float4*>(st) = make_float4(m1[0], m1[1], m2[0], m2[1]);
          } else {
            st_vec<3>(st, m1);
            st_vec<3>(st + 4, m2);
          }
        } else if constexpr (OPT == OPT_ADADELTA) {
          // optim.py:227-236
          float sg[DIM], sd[DIM];
          if constexpr (DIM == 2) {
            float4 s4 = *reinterpret_cast<const float4*>(st);
            sg[0] = s4.x; sg[1] = s4.y; sd[0] = s4.z; sd[1] = s4.w;
          } else {
            ld_vec<3>(st, sg);
            ld_vec<3>(st + 4, sd);
          }
#pragma unroll
          for (int d = 0; d < DIM; ++d) {
            const float g = -2.f * f[d];
            sg[d] = A.h.rho * sg[d] + (1.f - A.h.rho) * g * g;
            const float dl = -step * sqrtf(sd[d] + A.h.eps) / sqrtf(sg[d] + A.h.eps) * g;
            sd[d] = A.h.rho * sd[d] + (1.f - A.h.rho) * dl * dl;
            yn[d] = yi[d] + dl;
          }
          if constexpr (DIM == 2) {
            *reinterpret_cast<float4*>(st) = make_float4(sg[0], sg[1], sd[0], sd[1]);
          } else {
            st_vec<3>(st, sg);
            st_vec<3>(st + 4, sd);
          }
        }
        if constexpr (!NEST) st_vec<DIM>(Yout + (size_t)v * L::YS, yn);
        acc_bad += all_finite(yn, DIM) ? 0.0 : 1.0;
      }
    }
    const double4 tot = block_sum4(make_double4(acc_e, acc_n, acc_o, acc_bad), sm_red);
    if (threadIdx.x == 0) A.partial[A.tile0 + tile] = tot;
  }

  if (!A.fuse_finalize) return;
  // last-block-done: the block that retires last reduces and decides
  __shared__ bool sm_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) sm_last = (atomicAdd(&ctrl->arrive, 1u) == gridDim.x - 1);
  __syncthreads();
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
