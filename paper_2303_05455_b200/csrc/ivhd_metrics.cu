// ivhd_metrics.cu — embedding quality metrics on B200.
//
// neighbor_hit (reference metrics.py:254-294): for every embedded point its
// nn_max nearest other points in the 2-D / 3-D embedding, and the fraction of
// them sharing its label, per neighbourhood size 1..nn_max:
//     cf_nn[j] = sum_i #{same label among the first j+1 neighbours of i} / ((j+1) M)
//     cf       = mean_j cf_nn[j]
//
// Exact kNN in 2-D/3-D by a uniform grid: points are binned (~2 per cell)
// and sorted by cell (CUB radix sort); one warp per query walks square
// (cubic) rings of cells outwards, keeps its nn_max nearest in registers
// distributed over the lanes (slot s = lane + 32 j, sorted by (squared
// distance, index) — the reference's tie rule, knng.py:1-6), and stops when
// the nn_max-th distance is no larger than the distance to the unvisited
// region.  The per-size hit counts are integer sums (block shared memory,
// then 64-bit global atomics): order-independent, hence deterministic.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/ivhd_b200.h"

namespace metrics {

constexpr int NH_MAX = 512;              // neighbourhood sizes supported (<= 16 slots per lane)
constexpr int QWARPS = 8;                // query warps per block

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

struct Grid {
  double lo[3];
  double h;       // cell edge
  int g[3];       // cells per axis (1 for unused axes)
  int dim;
};

__device__ __forceinline__ int cell_axis(double x, double lo, double h, int g) {
  int c = (int)floor((x - lo) / h);
  return min(max(c, 0), g - 1);
}

__global__ void k_bbox(const double* __restrict__ y, int64_t m, int dim, double* __restrict__ out /*[6]: min,max*/) {
  __shared__ double smn[3][256], smx[3][256];
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    for (int d = 0; d < dim; ++d) {
      mn[d] = fmin(mn[d], y[i * dim + d]);
      mx[d] = fmax(mx[d], y[i * dim + d]);
    }
  for (int d = 0; d < 3; ++d) {
    smn[d][threadIdx.x] = mn[d];
    smx[d][threadIdx.x] = mx[d];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int d = 0; d < dim; ++d) {
      double a = INFINITY, b = -INFINITY;
      for (int t = 0; t < (int)blockDim.x; ++t) {
        a = fmin(a, smn[d][t]);
        b = fmax(b, smx[d][t]);
      }
      out[(blockIdx.x * 3 + d) * 2] = a;
      out[(blockIdx.x * 3 + d) * 2 + 1] = b;
    }
  }
}

__global__ void k_cells(const double* __restrict__ y, int64_t m, Grid G, uint32_t* __restrict__ cell,
                        int32_t* __restrict__ ids) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  uint32_t c = 0;
  for (int d = G.dim - 1; d >= 0; --d) c = c * (uint32_t)G.g[d] + (uint32_t)cell_axis(y[i * G.dim + d], G.lo[d], G.h, G.g[d]);
  cell[i] = c;
  ids[i] = (int32_t)i;
}

// cell_start[c] = first sorted index with cell >= c (n_cells + 1 entries)
__global__ void k_cell_start(const uint32_t* __restrict__ sorted_cell, int64_t m, int64_t n_cells,
                             uint32_t* __restrict__ start) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > m) return;
  const int64_t a = i == 0 ? -1 : (int64_t)sorted_cell[i - 1];
  const int64_t b = i == m ? n_cells : (int64_t)sorted_cell[i];
  for (int64_t c = a + 1; c <= b; ++c) start[c] = (uint32_t)i;
}

__global__ void k_gather_points(const double* __restrict__ y, const int32_t* __restrict__ ids, int64_t m, int dim,
                                double* __restrict__ ys) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  for (int d = 0; d < dim; ++d) ys[i * 3 + d] = y[(int64_t)ids[i] * dim + d];
  for (int d = dim; d < 3; ++d) ys[i * 3 + d] = 0.0;
}

__device__ __forceinline__ bool lt(double da, int ia, double db, int ib) { return da < db || (da == db && ia < ib); }

// One warp per query (queries visited in cell order for cache locality);
// SPL slots per lane hold up to 32 * SPL neighbours.
template <int SPL>
__global__ void __launch_bounds__(QWARPS * 32) k_grid_knn(const double* __restrict__ ys, const int32_t* __restrict__ sid,
                                                         const uint32_t* __restrict__ start, int64_t m, Grid G, int kk,
                                                         const int32_t* __restrict__ labels,
                                                         unsigned long long* __restrict__ hits,
                                                         int32_t* __restrict__ nbr_out) {
  __shared__ unsigned int sh_hits[32 * SPL];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 32 * SPL; i += blockDim.x) sh_hits[i] = 0;
  __syncthreads();
  const int64_t nw = (int64_t)gridDim.x * QWARPS;
  for (int64_t qs = blockIdx.x * (int64_t)QWARPS + warp; qs < m; qs += nw) {
    const int q = sid[qs];
    const double qx = ys[qs * 3], qy = ys[qs * 3 + 1], qz = ys[qs * 3 + 2];
    int qc[3];
    qc[0] = cell_axis(qx, G.lo[0], G.h, G.g[0]);
    qc[1] = G.dim > 1 ? cell_axis(qy, G.lo[1], G.h, G.g[1]) : 0;
    qc[2] = G.dim > 2 ? cell_axis(qz, G.lo[2], G.h, G.g[2]) : 0;
    double ld[SPL];
    int li[SPL];
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
      ld[j] = INFINITY;
      li[j] = 0x7fffffff;
    }
    int cnt = 0;
    double thr = INFINITY;  // squared distance of the kk-th entry (when cnt == kk)
    int thr_i = 0x7fffffff;
    const int rmax = max(G.g[0], max(G.g[1], G.g[2]));
    for (int r = 0; r < rmax; ++r) {
      // visit every cell at Chebyshev distance r (clipped to the grid)
      const int z0 = G.dim > 2 ? max(qc[2] - r, 0) : 0, z1 = G.dim > 2 ? min(qc[2] + r, G.g[2] - 1) : 0;
      const int y0 = max(qc[1] - r, 0), y1 = min(qc[1] + r, G.g[1] - 1);
      const int x0 = max(qc[0] - r, 0), x1 = min(qc[0] + r, G.g[0] - 1);
      for (int cz = z0; cz <= z1; ++cz)
        for (int cy = y0; cy <= y1; ++cy) {
          const bool edge_zy = abs(cz - qc[2]) == r || abs(cy - qc[1]) == r;
          for (int cx = x0; cx <= x1; ++cx) {
            if (!edge_zy && abs(cx - qc[0]) != r) {
              cx = qc[0] + r - 1;  // jump to the ring's far x column
              continue;
            }
            const uint32_t c = ((uint32_t)cz * G.g[1] + cy) * G.g[0] + cx;
            const uint32_t a = start[c], b = start[c + 1];
            for (uint32_t p0 = a; p0 < b; p0 += 32) {
              const uint32_t p = p0 + lane;
              double d2 = INFINITY;
              int id = 0x7fffffff;
              if (p < b) {
                id = sid[p];
                const double dx = ys[p * 3] - qx, dy = ys[p * 3 + 1] - qy, dz = ys[p * 3 + 2] - qz;
                d2 = fma(dx, dx, fma(dy, dy, dz * dz));
                if (id == q) d2 = INFINITY, id = 0x7fffffff;
              }
              unsigned pass = __ballot_sync(0xffffffffu, id != 0x7fffffff && (cnt < kk || lt(d2, id, thr, thr_i)));
              while (pass) {
                const int src = __ffs(pass) - 1;
                pass &= pass - 1;
                const double nd = __shfl_sync(0xffffffffu, d2, src);
                const int ni = __shfl_sync(0xffffffffu, id, src);
                if (!(cnt < kk || lt(nd, ni, thr, thr_i))) continue;  // threshold moved
                // position = number of entries before (nd, ni)
                int before = 0;
#pragma unroll
                for (int j = 0; j < SPL; ++j) before += lt(ld[j], li[j], nd, ni) ? 1 : 0;
                const int pos = __reduce_add_sync(0xffffffffu, before);
                // shift slots >= pos up by one (slot s = lane + 32 j)
#pragma unroll
                for (int j = SPL - 1; j >= 0; --j) {
                  double pd = __shfl_up_sync(0xffffffffu, ld[j], 1);
                  int pi = __shfl_up_sync(0xffffffffu, li[j], 1);
                  const double cd = j > 0 ? __shfl_sync(0xffffffffu, ld[j > 0 ? j - 1 : 0], 31) : INFINITY;
                  const int ci = j > 0 ? __shfl_sync(0xffffffffu, li[j > 0 ? j - 1 : 0], 31) : 0x7fffffff;
                  if (lane == 0) {
                    pd = cd;
                    pi = ci;
                  }
                  const int s = lane + 32 * j;
                  if (s > pos) {
                    ld[j] = pd;
                    li[j] = pi;
                  } else if (s == pos) {
                    ld[j] = nd;
                    li[j] = ni;
                  }
                }
                cnt = min(cnt + 1, kk);
                const int ts = kk - 1;
                // slot kk-1 lives in register (kk-1)/32 of lane (kk-1)%32: select statically
                double tv = ld[0];
                int ti = li[0];
#pragma unroll
                for (int j = 1; j < SPL; ++j)
                  if ((ts >> 5) == j) {
                    tv = ld[j];
                    ti = li[j];
                  }
                thr = __shfl_sync(0xffffffffu, tv, ts & 31);
                thr_i = __shfl_sync(0xffffffffu, ti, ts & 31);
              }
            }
          }
        }
      // distance from q to the region outside the visited block of cells
      if (cnt == kk) {
        double bnd = INFINITY;
        const double qq[3] = {qx, qy, qz};
        for (int d = 0; d < G.dim; ++d) {
          if (qc[d] - r > 0) bnd = fmin(bnd, qq[d] - (G.lo[d] + (qc[d] - r) * G.h));
          if (qc[d] + r < G.g[d] - 1) bnd = fmin(bnd, G.lo[d] + (qc[d] + r + 1) * G.h - qq[d]);
        }
        if (bnd == INFINITY || thr <= bnd * bnd) break;
      }
    }
    // per-size same-label counts: inclusive scan over slots 0..kk-1
    const int lq = labels[q];
    int carry = 0;
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
      const int s = lane + 32 * j;
      int v = (s < kk && li[j] != 0x7fffffff && labels[li[j]] == lq) ? 1 : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      v += carry;
      if (s < kk) atomicAdd(&sh_hits[s], (unsigned)v);
      carry = __shfl_sync(0xffffffffu, v, 31);
      if (nbr_out && s < kk) nbr_out[(int64_t)q * kk + s] = li[j] == 0x7fffffff ? -1 : li[j];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kk; i += blockDim.x) atomicAdd(&hits[i], (unsigned long long)sh_hits[i]);
}


// ---------------------------------------------------------------------------
// Rank-curve pass (reference metrics.py:149-182 `_curve_pass`, used by
// rnx_curve 185-202, gnn_curve 217-228, trust_continuity 240-251 and
// evaluate_embedding 351-380).  For every point i the reference ranks all
// other points by (squared distance, index) in the source space X (rho) and
// in the embedding Y (r) and accumulates
//     agree[max(rho, r)] += 1                         (Q_NX counts)
//     same_hd[p] / same_ld[p] += label match of the p-th neighbour
//     trust[k] += rho - k   for j with r <= k < rho   (entrants)
//     cont[k]  += r - k     for j with rho <= k < r   (leavers)
// Only ranks <= k_max reach the curves (cumsum(agree)[1..k_max]), so the
// pass needs each row's K = max(k_max, report ks) nearest in both spaces,
// plus the exact far rank of the few entrants / leavers outside that list.
//
// Distances follow the reference formula (metrics.py:76-84):
//     d2(i, j) = max((|x_i|^2 + |x_j|^2) - 2 x_i.x_j, 0),  d2(i, i) = +inf.
// X rows come in blocks of B rows: a fp64 SIMT tile kernel writes the (B, M)
// distance block (the 126 MB L2 holds a block's working set for small M);
// Y distances (dim <= 3) are recomputed on the fly.  Per row one CTA keeps
// the best 1024 (d2, j) pairs sorted in shared memory and merges a pending
// buffer of threshold-passing candidates by bitonic sort (~k ln(M/k)
// insertions per row).  All counts are integers: deterministic.
namespace curves {

constexpr int KMAX = 1024;  // longest ranked list per row
constexpr int NT = 512;     // threads per row CTA
constexpr int NB = 2 * KMAX;
constexpr int MAX_REPORT = 8;
constexpr int DT = 64, DK = 16;  // distance tile

struct Report {
  int n;
  int k[MAX_REPORT];
  int kmax;  // max of k (0 when n == 0)
};

__global__ void k_sqnorm(const double* __restrict__ x, int64_t m, int n, double* __restrict__ sq) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  double s = 0.0;
  for (int c = 0; c < n; ++c) s = fma(x[i * n + c], x[i * n + c], s);
  sq[i] = s;
}

// out[r][j] = max((sqa[r] + sqb[j]) - 2 a_r.b_j, 0) for r < nb, j < m
__global__ void __launch_bounds__(256) k_dist_block(const double* __restrict__ a, const double* __restrict__ sqa,
                                                    const double* __restrict__ b, const double* __restrict__ sqb,
                                                    int64_t m, int n, int nb, double* __restrict__ out) {
  __shared__ double As[DK][DT + 1], Bs[DK][DT + 1];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int64_t rb = (int64_t)blockIdx.y * DT, cb = (int64_t)blockIdx.x * DT;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < n; k0 += DK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = t + 256 * q, row = e >> 4, kk = e & 15;
      const int64_t ra = rb + row, cbb = cb + row;
      As[kk][row] = (ra < nb && k0 + kk < n) ? a[ra * n + k0 + kk] : 0.0;
      Bs[kk][row] = (cbb < m && k0 + kk < n) ? b[cbb * n + k0 + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < DK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = As[kk][ty + 16 * u];
        b[u] = Bs[kk][tx + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t r = rb + ty + 16 * u;
    if (r >= nb) continue;
    const double si = sqa[r];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t c = cb + tx + 16 * v;
      if (c < m) out[r * m + c] = fmax((si + sqb[c]) - 2.0 * acc[u][v], 0.0);
    }
  }
}

struct HdRow {
  const double* p;
  __device__ __forceinline__ double operator()(int64_t j) const { return p[j]; }
};

struct LdRow {
  const double* y;
  const double* sq;
  int dim;
  double yi[3];
  double si;
  __device__ __forceinline__ double operator()(int64_t j) const {
    double dot = 0.0;
    for (int d = 0; d < dim; ++d) dot = fma(yi[d], y[j * dim + d], dot);
    return fmax((si + sq[j]) - 2.0 * dot, 0.0);
  }
};

// Bitonic sort of consecutive segments of length S (power of two) within the
// first N entries, ascending by (d, j).
__device__ void bitonic(double* d, int* jj, int N, int S) {
  for (int k = 2; k <= S; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < N / 2; t += NT) {
        const int i = 2 * t - (t & (j - 1));
        const int p = i + j;
        const bool asc = (k == S) || !(i & k);
        const bool gt = lt(d[p], jj[p], d[i], jj[i]);
        if (gt == asc) {
          const double td = d[i];
          d[i] = d[p];
          d[p] = td;
          const int tj = jj[i];
          jj[i] = jj[p];
          jj[p] = tj;
        }
      }
      __syncthreads();
    }
}

// Merge the pending half into the sorted best half.
__device__ void merge_pending(double* sd, int* sj, int* s_cnt) {
  const int cnt = *s_cnt;
  for (int t = KMAX + cnt + threadIdx.x; t < NB; t += NT) {
    sd[t] = INFINITY;
    sj[t] = 0x7fffffff;
  }
  __syncthreads();
  bitonic(sd, sj, NB, NB);
  if (threadIdx.x == 0) *s_cnt = 0;
  __syncthreads();
}

// sd[0..K) / sj[0..K) <- the K smallest (d2, j), j != self, in order.
template <class Dist>
__device__ void select_row(const Dist& dist, int64_t m, int self, int K, double* sd, int* sj, int* s_cnt) {
  for (int t = threadIdx.x; t < NB; t += NT) {
    sd[t] = INFINITY;
    sj[t] = 0x7fffffff;
  }
  if (threadIdx.x == 0) *s_cnt = 0;
  __syncthreads();
  double thr_d = INFINITY;
  int thr_j = 0x7fffffff;
  for (int64_t c = 0; c < m; c += NT) {
    if (*s_cnt > KMAX - NT) {
      merge_pending(sd, sj, s_cnt);
      thr_d = sd[K - 1];
      thr_j = sj[K - 1];
    }
    const int64_t j = c + threadIdx.x;
    if (j < m && j != self) {
      const double d = dist(j);
      if (lt(d, (int)j, thr_d, thr_j)) {
        const int p = atomicAdd(s_cnt, 1);
        sd[KMAX + p] = d;
        sj[KMAX + p] = (int)j;
      }
    }
    __syncthreads();
  }
  merge_pending(sd, sj, s_cnt);
}

// Radix select of the same K smallest (d2, j): up to three 12-bit histogram
// passes over the row's distance bits (non-negative fp64 bit patterns order
// like the values) narrow down the bucket that holds the K-th key; every key
// below that bucket and the whole bucket are then collected and sorted once.
// Returns false (nothing written) when the bucket is too crowded to collect —
// exact ties of many points — and the caller falls back to select_row.
// The histogram aliases sd, the per-thread bin sums alias sj.
__device__ __forceinline__ unsigned long long dkey(double d) {
  return (unsigned long long)__double_as_longlong(d + 0.0);  // -0 -> +0
}

template <class Dist>
__device__ bool select_radix(const Dist& dist, int64_t m, int self, int K, double* sd, int* sj, int* s_misc) {
  unsigned* hist = reinterpret_cast<unsigned*>(sd);  // 4096 bins
  int* tsum = sj;                                    // 512 per-thread sums
  unsigned long long prefix = 0;
  int sh = 64, need = K, below = 0, bucket = 0;
  for (int level = 0; level < 3; ++level) {
    const int nsh = sh - 12;
    for (int t = threadIdx.x; t < 4096; t += NT) hist[t] = 0;
    __syncthreads();
    for (int64_t j = threadIdx.x; j < m; j += NT) {
      if (j == self) continue;
      const unsigned long long k = dkey(dist(j));
      if (level == 0 || (k >> sh) == prefix) atomicAdd(&hist[(k >> nsh) & 4095], 1u);
    }
    __syncthreads();
    {
      int a = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) a += hist[threadIdx.x * 8 + b];
      tsum[threadIdx.x] = a;
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // find the bin where the running count reaches `need`
      const int lane = threadIdx.x;
      int a = 0;
      for (int t = 0; t < 16; ++t) a += tsum[lane * 16 + t];
      int incl = a;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, incl >= need);
      const int L = __ffs(hit) - 1;  // hit != 0: the row has >= need keys in this group
      if (lane == L) {
        int run = incl - a;
        int t = lane * 16;
        while (run + tsum[t] < need) run += tsum[t++];
        int b = t * 8;
        while (run + (int)hist[b] < need) run += hist[b++];
        s_misc[0] = b;
        s_misc[1] = run;
        s_misc[2] = (int)hist[b];
      }
    }
    __syncthreads();
    const int b = s_misc[0];
    need -= s_misc[1];
    below += s_misc[1];
    bucket = s_misc[2];
    prefix = (prefix << 12) | (unsigned long long)b;
    sh = nsh;
    __syncthreads();
    if (below + bucket <= NB) break;
  }
  if (below + bucket > NB) return false;
  // collect every key below the bucket and the bucket itself, then sort once
  if (threadIdx.x == 0) s_misc[3] = 0;
  __syncthreads();
  for (int64_t j = threadIdx.x; j < m; j += NT) {
    if (j == self) continue;
    const double d = dist(j);
    if ((dkey(d) >> sh) <= prefix) {
      const int p = atomicAdd(&s_misc[3], 1);
      sd[p] = d;
      sj[p] = (int)j;
    }
  }
  __syncthreads();
  const int n = s_misc[3];
  const int N = n <= KMAX ? KMAX : NB;
  for (int t = n + threadIdx.x; t < N; t += NT) {
    sd[t] = INFINITY;
    sj[t] = 0x7fffffff;
  }
  __syncthreads();
  bitonic(sd, sj, N, N);
  return true;
}

// 1-based rank of id j in a by-id sorted list (keys in kd as doubles), 0 if absent
__device__ __forceinline__ int find_rank(const double* kd, const int* kr, int K, int j) {
  int lo = 0, hi = K;
  const double key = (double)j;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (kd[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return (lo < K && kd[lo] == key) ? kr[lo] : 0;
}

// Exact 1-based ranks, among all j != self of a row, of Q query ids that lie
// outside the row's ranked list: one pass over the row.  The queries are
// sorted by (d2, id) in qd/qj; every row element lands (binary search) on the
// first query above it, diff[] counts those landings, and a query's rank is
// one plus the landings at or below its sorted position.
template <class Dist>
__device__ void far_ranks(const Dist& dist, int64_t m, int self, int Q, const int* need_j, double* qd, int* qj,
                          int* diff) {
  for (int t = threadIdx.x; t < KMAX; t += NT) {
    qd[t] = t < Q ? dist(need_j[t]) : INFINITY;
    qj[t] = t < Q ? need_j[t] : 0x7fffffff;
    diff[t] = 0;
  }
  __syncthreads();
  bitonic(qd, qj, KMAX, KMAX);
  for (int64_t j = threadIdx.x; j < m; j += NT) {
    if (j == self) continue;
    const double d = dist(j);
    int lo = 0, hi = Q;  // first query q with (d, j) < (qd[q], qj[q])
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (lt(d, (int)j, qd[mid], qj[mid])) hi = mid;
      else lo = mid + 1;
    }
    if (lo < Q) atomicAdd(&diff[lo], 1);
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // inclusive scan of diff[0..Q) by one warp
    int carry = 0;
    for (int b = 0; b < Q; b += 32) {
      const int t = b + threadIdx.x;
      int v = t < Q ? diff[t] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (threadIdx.x >= o) v += u;
      }
      if (t < Q) diff[t] = v + carry;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
}

// rank of query id jq (distance dq) after far_ranks
__device__ __forceinline__ int far_rank_of(const double* qd, const int* qj, const int* diff, int Q, double dq, int jq) {
  int lo = 0, hi = Q;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (lt(qd[mid], qj[mid], dq, jq)) lo = mid + 1;
    else hi = mid;
  }
  return diff[lo] + 1;
}

struct Shared {
  double sd[NB];
  int sj[NB];
  int hd_ids[KMAX], ld_ids[KMAX];
  unsigned agree[KMAX + 1], same_ld[KMAX], same_hd[KMAX];
  int need_hd_j[KMAX], need_hd_r[KMAX], need_ld_j[KMAX], need_ld_r[KMAX];
  int diff[KMAX];
  unsigned long long trust[MAX_REPORT], cont[MAX_REPORT];
  int cnt, n_need_hd, n_need_ld;
  int misc[4];
};

__global__ void __launch_bounds__(NT) k_curve_rows(const double* __restrict__ hd_block, int64_t r0, int nb, int64_t m,
                                                   const double* __restrict__ y, const double* __restrict__ sqy,
                                                   int dim, const int32_t* __restrict__ labels, int k_max, int K,
                                                   Report rep, unsigned long long* __restrict__ g_agree,
                                                   unsigned long long* __restrict__ g_same_ld,
                                                   unsigned long long* __restrict__ g_same_hd,
                                                   unsigned long long* __restrict__ g_trust,
                                                   unsigned long long* __restrict__ g_cont) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Shared& S = *reinterpret_cast<Shared*>(smem_raw);
  const int tid = threadIdx.x;
  for (int t = tid; t <= KMAX; t += NT) S.agree[t] = 0;
  for (int t = tid; t < KMAX; t += NT) S.same_ld[t] = S.same_hd[t] = 0;
  if (tid < MAX_REPORT) S.trust[tid] = S.cont[tid] = 0;
  if (tid == 0) S.n_need_hd = S.n_need_ld = 0;
  __syncthreads();
  for (int row = blockIdx.x; row < nb; row += gridDim.x) {
    const int i = (int)(r0 + row);
    const HdRow hd{hd_block + (int64_t)row * m};
    LdRow ld{y, sqy, dim, {0, 0, 0}, sqy[i]};
    for (int d = 0; d < dim; ++d) ld.yi[d] = y[(int64_t)i * dim + d];
    const int own = labels ? labels[i] : 0;

    if (!select_radix(hd, m, i, K, S.sd, S.sj, S.misc)) select_row(hd, m, i, K, S.sd, S.sj, &S.cnt);
    for (int t = tid; t < K; t += NT) {
      S.hd_ids[t] = S.sj[t];
      if (labels && t < k_max && labels[S.sj[t]] == own) ++S.same_hd[t];  // one writer per slot
    }
    __syncthreads();
    if (!select_radix(ld, m, i, K, S.sd, S.sj, S.misc)) select_row(ld, m, i, K, S.sd, S.sj, &S.cnt);
    for (int t = tid; t < K; t += NT) {
      S.ld_ids[t] = S.sj[t];
      if (labels && t < k_max && labels[S.sj[t]] == own) ++S.same_ld[t];
    }
    __syncthreads();
    // by-id lists: [0, KMAX) = HD (id, rank), [KMAX, NB) = LD (id, rank)
    for (int t = tid; t < KMAX; t += NT) {
      S.sd[t] = t < K ? (double)S.hd_ids[t] : INFINITY;
      S.sj[t] = t + 1;
      S.sd[KMAX + t] = t < K ? (double)S.ld_ids[t] : INFINITY;
      S.sj[KMAX + t] = t + 1;
    }
    __syncthreads();
    bitonic(S.sd, S.sj, NB, KMAX);
    for (int t = tid; t < K; t += NT) {
      {  // LD neighbour of rank rl: agreement and trustworthiness entrants
        const int rl = t + 1, rh = find_rank(S.sd, S.sj, K, S.ld_ids[t]);
        if (rh) {
          const int p = max(rh, rl);
          if (p <= k_max) atomicAdd(&S.agree[p], 1u);
        }
        if (rl <= rep.kmax) {
          if (!rh) {
            const int q = atomicAdd(&S.n_need_hd, 1);
            S.need_hd_j[q] = S.ld_ids[t];
            S.need_hd_r[q] = rl;
          } else {
            for (int a = 0; a < rep.n; ++a)
              if (rl <= rep.k[a] && rh > rep.k[a]) atomicAdd(&S.trust[a], (unsigned long long)(rh - rep.k[a]));
          }
        }
      }
      {  // HD neighbour of rank rh: continuity leavers
        const int rh = t + 1;
        if (rh <= rep.kmax) {
          const int rl = find_rank(S.sd + KMAX, S.sj + KMAX, K, S.hd_ids[t]);
          if (!rl) {
            const int q = atomicAdd(&S.n_need_ld, 1);
            S.need_ld_j[q] = S.hd_ids[t];
            S.need_ld_r[q] = rh;
          } else {
            for (int a = 0; a < rep.n; ++a)
              if (rh <= rep.k[a] && rl > rep.k[a]) atomicAdd(&S.cont[a], (unsigned long long)(rl - rep.k[a]));
          }
        }
      }
    }
    __syncthreads();
    // ranks beyond the lists: one batched counting pass over the row per space
    const int nh = S.n_need_hd, nl = S.n_need_ld;
    if (nh) {
      far_ranks(hd, m, i, nh, S.need_hd_j, S.sd, S.sj, S.diff);
      for (int q = tid; q < nh; q += NT) {
        const int jq = S.need_hd_j[q];
        const int rank = far_rank_of(S.sd, S.sj, S.diff, nh, hd(jq), jq);
        for (int a = 0; a < rep.n; ++a)
          if (S.need_hd_r[q] <= rep.k[a]) atomicAdd(&S.trust[a], (unsigned long long)(rank - rep.k[a]));
      }
      __syncthreads();
    }
    if (nl) {
      far_ranks(ld, m, i, nl, S.need_ld_j, S.sd, S.sj, S.diff);
      for (int q = tid; q < nl; q += NT) {
        const int jq = S.need_ld_j[q];
        const int rank = far_rank_of(S.sd, S.sj, S.diff, nl, ld(jq), jq);
        for (int a = 0; a < rep.n; ++a)
          if (S.need_ld_r[q] <= rep.k[a]) atomicAdd(&S.cont[a], (unsigned long long)(rank - rep.k[a]));
      }
    }
    __syncthreads();
    if (tid == 0) S.n_need_hd = S.n_need_ld = 0;
    __syncthreads();
  }
  for (int t = tid; t <= k_max; t += NT)
    if (S.agree[t]) atomicAdd(&g_agree[t], (unsigned long long)S.agree[t]);
  if (labels)
    for (int t = tid; t < k_max; t += NT) {
      if (S.same_ld[t]) atomicAdd(&g_same_ld[t], (unsigned long long)S.same_ld[t]);
      if (S.same_hd[t]) atomicAdd(&g_same_hd[t], (unsigned long long)S.same_hd[t]);
    }
  if (tid < rep.n) {
    atomicAdd(&g_trust[tid], S.trust[tid]);
    atomicAdd(&g_cont[tid], S.cont[tid]);
  }
}


// ---------------------------------------------------------------------------
// Pair ranks (reference metrics.py:335-352 `_pair_ranks`, used by
// shepard_and_corank 297-320): the exact rank of j among i's neighbours,
//     1 + #{k != i : (d2(i,k), k) < (d2(i,j), j)},
// for sampled pairs (i, j).  Rows of the distinct i are gathered, their
// distance rows computed by k_dist_block, then one CTA per pair counts.
__global__ void k_gather_rows(const double* __restrict__ z, const double* __restrict__ sq, int n,
                              const int64_t* __restrict__ rows, int nb, double* __restrict__ a,
                              double* __restrict__ sqa) {
  const int r = blockIdx.x;
  if (r >= nb) return;
  const int64_t i = rows[r];
  for (int c = threadIdx.x; c < n; c += blockDim.x) a[(int64_t)r * n + c] = z[i * n + c];
  if (threadIdx.x == 0) sqa[r] = sq[i];
}

__global__ void __launch_bounds__(256) k_pair_count(const double* __restrict__ blk, int64_t m,
                                                    const int* __restrict__ prow, const int64_t* __restrict__ pi,
                                                    const int64_t* __restrict__ pj, int np,
                                                    int64_t* __restrict__ ranks) {
  __shared__ int s_cnt;
  const int p = blockIdx.x;
  if (p >= np) return;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const double* row = blk + (int64_t)prow[p] * m;
  const int64_t i = pi[p];
  const int j = (int)pj[p];
  const double dj = row[j];
  int c = 0;
  for (int64_t k = threadIdx.x; k < m; k += blockDim.x)
    if (k != i && lt(row[k], (int)k, dj, j)) ++c;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) atomicAdd(&s_cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) ranks[p] = (int64_t)s_cnt + 1;
}

// ---------------------------------------------------------------------------
// Full rank matrix (reference metrics.py:103-146 `_rank_block` /
// `compute_ranks`): per row, a stable sort of (distance, index) with the
// diagonal at +inf, ranks 1..M-1, self 0.  Keys: order-preserving uint64 of
// the fp64 distance (-0 folded to +0, so equal values tie and the stable
// radix sort keeps index order).
__global__ void k_rank_keys(const double* __restrict__ blk, int64_t m, int64_t r0, int nb,
                            unsigned long long* __restrict__ keys, int* __restrict__ vals) {
  const int64_t n = (int64_t)nb * m;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / m, c = t - r * m;
    const double d = (c == r0 + r) ? INFINITY : blk[t] + 0.0;
    unsigned long long k = (unsigned long long)__double_as_longlong(d);
    k = (k >> 63) ? ~k : (k | 0x8000000000000000ull);
    keys[t] = k;
    vals[t] = (int)c;
  }
}

__global__ void k_rank_scatter(const int* __restrict__ order, int64_t m, int64_t r0, int nb,
                               int64_t* __restrict__ ranks) {
  const int64_t n = (int64_t)nb * m;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / m, p = t - r * m;
    const int c = order[t];
    ranks[r * m + c] = (c == r0 + r) ? 0 : p + 1;
  }
}

__global__ void k_seg_offsets(int* __restrict__ off, int nb, int64_t m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= nb) off[i] = (int)(i * m);
}
}  // namespace curves

}  // namespace metrics

using namespace metrics;

extern "C" {

const char* ivhd_metrics_last_error(void) { return g_err.c_str(); }

int ivhd_neighbor_hit(int device, const double* y, int64_t m, int32_t dim, const int32_t* labels, int32_t nn_max,
                      double* cf_nn_out, int32_t* nbr_out) {
  if (!y || !labels || !cf_nn_out) return fail(IVHD_ERR_INVALID_ARG, "null pointer");
  if (dim < 1 || dim > 3) return fail(IVHD_ERR_INVALID_ARG, "grid neighbour search needs 1 <= dim <= 3, got %d", dim);
  if (!(1 <= nn_max && nn_max < m)) return fail(IVHD_ERR_INVALID_ARG, "nn_max must be in [1, M), got %d", nn_max);
  if (nn_max > NH_MAX) return fail(IVHD_ERR_INVALID_ARG, "nn_max=%d above the supported %d", nn_max, NH_MAX);
  if (m >= 0x7fffffffLL) return fail(IVHD_ERR_INVALID_ARG, "M too large");
  if (cudaSetDevice(device) != cudaSuccess) return fail(IVHD_ERR_CUDA, "cudaSetDevice(%d) failed", device);
  {  // keep freed stream-ordered memory pooled: returning GBs to the driver
     // at every synchronisation costs seconds (as in ivhd_create)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return fail(IVHD_ERR_CUDA, "stream");
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double *dy = nullptr, *ys = nullptr, *bb = nullptr;
  int32_t *dl = nullptr, *ids = nullptr, *sid = nullptr, *dn = nullptr;
  uint32_t *cell = nullptr, *scell = nullptr, *start = nullptr;
  unsigned long long* hits = nullptr;
  void* tmp = nullptr;
  cudaError_t e = cudaSuccess;
  int rc = IVHD_OK;
  const int nbb = std::min<int64_t>(sms * 2, (m + 255) / 256);
  do {
#define MTRY(call) \
  if ((e = (call)) != cudaSuccess) break
    MTRY(cudaMallocAsync(&dy, sizeof(double) * m * dim, st));
    MTRY(cudaMallocAsync(&dl, sizeof(int32_t) * m, st));
    MTRY(cudaMallocAsync(&bb, sizeof(double) * nbb * 6, st));
    MTRY(cudaMemcpyAsync(dy, y, sizeof(double) * m * dim, cudaMemcpyHostToDevice, st));
    MTRY(cudaMemcpyAsync(dl, labels, sizeof(int32_t) * m, cudaMemcpyHostToDevice, st));
    k_bbox<<<nbb, 256, 0, st>>>(dy, m, dim, bb);
    std::vector<double> hb(nbb * 6);
    MTRY(cudaMemcpyAsync(hb.data(), bb, sizeof(double) * nbb * 6, cudaMemcpyDeviceToHost, st));
    MTRY(cudaStreamSynchronize(st));
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int d = 0; d < dim; ++d) {
      lo[d] = INFINITY;
      hi[d] = -INFINITY;
      for (int b = 0; b < nbb; ++b) {
        lo[d] = std::min(lo[d], hb[(b * 3 + d) * 2]);
        hi[d] = std::max(hi[d], hb[(b * 3 + d) * 2 + 1]);
      }
    }
    bool finite = true;
    for (int d = 0; d < dim; ++d) finite &= std::isfinite(lo[d]) && std::isfinite(hi[d]);
    if (!finite) {
      rc = fail(IVHD_ERR_INVALID_ARG, "embedding has non-finite coordinates");
      break;
    }
    // cell edge: ~2 points per cell over the bounding box, at most ~4M cells per point budget
    double vol = 1.0;
    int used = 0;
    for (int d = 0; d < dim; ++d)
      if (hi[d] > lo[d]) {
        vol *= hi[d] - lo[d];
        ++used;
      }
    Grid G{};
    G.dim = dim;
    const double target = std::max(1.0, (double)m / 2.0);
    G.h = used ? std::pow(vol / target, 1.0 / used) : 1.0;
    if (!(G.h > 0) || !std::isfinite(G.h)) G.h = 1.0;
    int64_t n_cells = 1;
    for (int d = 0; d < 3; ++d) {
      G.lo[d] = lo[d];
      G.g[d] = d < dim ? (int)std::min<double>(std::floor((hi[d] - lo[d]) / G.h) + 1, 1 << 20) : 1;
      n_cells *= G.g[d];
    }
    while (n_cells > 4 * m + 64) {  // degenerate aspect ratios: coarsen
      G.h *= 2;
      n_cells = 1;
      for (int d = 0; d < dim; ++d) {
        G.g[d] = (int)std::floor((hi[d] - lo[d]) / G.h) + 1;
        n_cells *= G.g[d];
      }
    }
    MTRY(cudaMallocAsync(&cell, sizeof(uint32_t) * m, st));
    MTRY(cudaMallocAsync(&scell, sizeof(uint32_t) * m, st));
    MTRY(cudaMallocAsync(&ids, sizeof(int32_t) * m, st));
    MTRY(cudaMallocAsync(&sid, sizeof(int32_t) * m, st));
    MTRY(cudaMallocAsync(&start, sizeof(uint32_t) * (n_cells + 1), st));
    MTRY(cudaMallocAsync(&ys, sizeof(double) * 3 * m, st));
    MTRY(cudaMallocAsync(&hits, sizeof(unsigned long long) * NH_MAX, st));
    MTRY(cudaMemsetAsync(hits, 0, sizeof(unsigned long long) * NH_MAX, st));
    k_cells<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(dy, m, G, cell, ids);
    int end_bit = 1;
    while (end_bit < 32 && ((int64_t)1 << end_bit) < n_cells) ++end_bit;
    size_t tb = 0;
    MTRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, cell, scell, ids, sid, (int)m, 0, end_bit, st));
    MTRY(cudaMallocAsync(&tmp, std::max<size_t>(tb, 16), st));
    MTRY(cub::DeviceRadixSort::SortPairs(tmp, tb, cell, scell, ids, sid, (int)m, 0, end_bit, st));
    k_cell_start<<<(unsigned)((m + 256) / 256), 256, 0, st>>>(scell, m, n_cells, start);
    k_gather_points<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(dy, sid, m, dim, ys);
    if (nbr_out) MTRY(cudaMallocAsync(&dn, sizeof(int32_t) * m * nn_max, st));
    const int blocks = (int)std::min<int64_t>((m + QWARPS - 1) / QWARPS, (int64_t)sms * 16);
    if (nn_max <= 128) k_grid_knn<4><<<blocks, QWARPS * 32, 0, st>>>(ys, sid, start, m, G, nn_max, dl, hits, dn);
    else if (nn_max <= 256) k_grid_knn<8><<<blocks, QWARPS * 32, 0, st>>>(ys, sid, start, m, G, nn_max, dl, hits, dn);
    else k_grid_knn<16><<<blocks, QWARPS * 32, 0, st>>>(ys, sid, start, m, G, nn_max, dl, hits, dn);
    MTRY(cudaGetLastError());
    std::vector<unsigned long long> hh(NH_MAX);
    MTRY(cudaMemcpyAsync(hh.data(), hits, sizeof(unsigned long long) * NH_MAX, cudaMemcpyDeviceToHost, st));
    if (nbr_out) MTRY(cudaMemcpyAsync(nbr_out, dn, sizeof(int32_t) * m * nn_max, cudaMemcpyDeviceToHost, st));
    MTRY(cudaStreamSynchronize(st));
    for (int j = 0; j < nn_max; ++j) cf_nn_out[j] = (double)hh[j] / ((double)(j + 1) * (double)m);
#undef MTRY
  } while (0);
  for (void* p : {(void*)dy, (void*)ys, (void*)bb, (void*)dl, (void*)ids, (void*)sid, (void*)dn, (void*)cell,
                  (void*)scell, (void*)start, (void*)hits, tmp})
    if (p) cudaFreeAsync(p, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (rc != IVHD_OK) return rc;
  if (e != cudaSuccess) return fail(IVHD_ERR_CUDA, "neighbor_hit: %s", cudaGetErrorString(e));
  return IVHD_OK;
}


int ivhd_curve_pass(int device, const double* x, int64_t m, int32_t n, int32_t x_precomputed, const double* y,
                    int32_t dim, const int32_t* labels, int32_t k_max, const int32_t* report_ks, int32_t n_report,
                    int64_t* agree_out, int64_t* same_ld_out, int64_t* same_hd_out, int64_t* trust_out,
                    int64_t* cont_out) {
  using namespace curves;
  if (!x || !y || !agree_out) return fail(IVHD_ERR_INVALID_ARG, "null pointer");
  if (m < 3) return fail(IVHD_ERR_INVALID_ARG, "need at least 3 points");
  if (m >= 0x7fffffffLL) return fail(IVHD_ERR_INVALID_ARG, "M too large");
  if (dim < 1 || dim > 3) return fail(IVHD_ERR_INVALID_ARG, "embedding dimension must be 1..3, got %d", dim);
  if (x_precomputed ? n != m : n < 1) return fail(IVHD_ERR_INVALID_ARG, "bad source shape (m=%lld, n=%d)", (long long)m, n);
  if (!(1 <= k_max && k_max <= m - 2)) return fail(IVHD_ERR_INVALID_ARG, "k_max must be in [1, %lld]", (long long)(m - 2));
  if (n_report < 0 || n_report > MAX_REPORT || (n_report && !report_ks))
    return fail(IVHD_ERR_INVALID_ARG, "at most %d report ks", MAX_REPORT);
  if (labels && (!same_ld_out || !same_hd_out)) return fail(IVHD_ERR_INVALID_ARG, "null label-count output");
  if (n_report && (!trust_out || !cont_out)) return fail(IVHD_ERR_INVALID_ARG, "null trust/continuity output");
  Report rep{};
  rep.n = n_report;
  for (int a = 0; a < n_report; ++a) {
    if (!(1 <= report_ks[a] && 2LL * report_ks[a] < m))
      return fail(IVHD_ERR_INVALID_ARG, "k must satisfy 1 <= k < M/2, got %d", report_ks[a]);
    rep.k[a] = report_ks[a];
    rep.kmax = std::max(rep.kmax, rep.k[a]);
  }
  const int K = (int)std::min<int64_t>(std::max(k_max, rep.kmax), m - 1);
  if (K > KMAX) return fail(IVHD_ERR_INVALID_ARG, "k_max=%d above the supported %d", K, KMAX);
  if (cudaSetDevice(device) != cudaSuccess) return fail(IVHD_ERR_CUDA, "cudaSetDevice(%d) failed", device);
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return fail(IVHD_ERR_CUDA, "stream");
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  // distance block: <= 1 GiB, at least one row
  const int64_t nb_max = std::max<int64_t>(1, std::min<int64_t>(m, ((int64_t)1 << 27) / m));
  double *dx = nullptr, *sqx = nullptr, *dy = nullptr, *sqy = nullptr, *blk = nullptr;
  int32_t* dl = nullptr;
  unsigned long long* acc = nullptr;  // agree[KMAX+1] | same_ld[KMAX] | same_hd[KMAX] | trust[8] | cont[8]
  const size_t n_acc = (KMAX + 1) + 2 * KMAX + 2 * MAX_REPORT;
  cudaError_t e = cudaSuccess;
  do {
#define MTRY(call) \
  if ((e = (call)) != cudaSuccess) break
    MTRY(cudaMallocAsync(&dy, sizeof(double) * m * dim, st));
    MTRY(cudaMallocAsync(&sqy, sizeof(double) * m, st));
    MTRY(cudaMallocAsync(&blk, sizeof(double) * nb_max * m, st));
    MTRY(cudaMallocAsync(&acc, sizeof(unsigned long long) * n_acc, st));
    MTRY(cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * n_acc, st));
    MTRY(cudaMemcpyAsync(dy, y, sizeof(double) * m * dim, cudaMemcpyHostToDevice, st));
    if (labels) {
      MTRY(cudaMallocAsync(&dl, sizeof(int32_t) * m, st));
      MTRY(cudaMemcpyAsync(dl, labels, sizeof(int32_t) * m, cudaMemcpyHostToDevice, st));
    }
    if (!x_precomputed) {
      MTRY(cudaMallocAsync(&dx, sizeof(double) * m * n, st));
      MTRY(cudaMallocAsync(&sqx, sizeof(double) * m, st));
      MTRY(cudaMemcpyAsync(dx, x, sizeof(double) * m * n, cudaMemcpyHostToDevice, st));
      k_sqnorm<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(dx, m, n, sqx);
    }
    k_sqnorm<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(dy, m, dim, sqy);
    MTRY(cudaFuncSetAttribute(k_curve_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Shared)));
    unsigned long long* g = acc;
    for (int64_t r0 = 0; r0 < m; r0 += nb_max) {
      const int nb = (int)std::min<int64_t>(nb_max, m - r0);
      if (x_precomputed) {
        MTRY(cudaMemcpyAsync(blk, x + r0 * m, sizeof(double) * nb * m, cudaMemcpyHostToDevice, st));
      } else {
        dim3 grid((unsigned)((m + DT - 1) / DT), (unsigned)((nb + DT - 1) / DT));
        k_dist_block<<<grid, 256, 0, st>>>(dx + r0 * n, sqx + r0, dx, sqx, m, n, nb, blk);
      }
      const int ctas = std::min(nb, sms * 3);
      k_curve_rows<<<ctas, NT, sizeof(Shared), st>>>(blk, r0, nb, m, dy, sqy, dim, dl, k_max, K, rep, g,
                                                     g + KMAX + 1, g + 2 * KMAX + 1, g + 3 * KMAX + 1,
                                                     g + 3 * KMAX + 1 + MAX_REPORT);
      MTRY(cudaGetLastError());
    }
    if (e != cudaSuccess) break;
    std::vector<unsigned long long> h(n_acc);
    MTRY(cudaMemcpyAsync(h.data(), acc, sizeof(unsigned long long) * n_acc, cudaMemcpyDeviceToHost, st));
    MTRY(cudaStreamSynchronize(st));
    for (int t = 0; t <= k_max; ++t) agree_out[t] = (int64_t)h[t];
    if (labels)
      for (int t = 0; t < k_max; ++t) {
        same_ld_out[t] = (int64_t)h[KMAX + 1 + t];
        same_hd_out[t] = (int64_t)h[2 * KMAX + 1 + t];
      }
    for (int a = 0; a < n_report; ++a) {
      trust_out[a] = (int64_t)h[3 * KMAX + 1 + a];
      cont_out[a] = (int64_t)h[3 * KMAX + 1 + MAX_REPORT + a];
    }
#undef MTRY
  } while (0);
  for (void* p : {(void*)dx, (void*)sqx, (void*)dy, (void*)sqy, (void*)blk, (void*)dl, (void*)acc})
    if (p) cudaFreeAsync(p, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (e != cudaSuccess) return fail(IVHD_ERR_CUDA, "curve_pass: %s", cudaGetErrorString(e));
  return IVHD_OK;
}


int ivhd_pair_ranks(int device, const double* z, int64_t m, int32_t n, const int64_t* i_idx, const int64_t* j_idx,
                    int64_t n_pairs, int64_t* ranks_out) {
  using namespace curves;
  if (!z || !i_idx || !j_idx || !ranks_out) return fail(IVHD_ERR_INVALID_ARG, "null pointer");
  if (m < 2 || m >= 0x7fffffffLL || n < 1) return fail(IVHD_ERR_INVALID_ARG, "bad shape (m=%lld, n=%d)", (long long)m, n);
  if (n_pairs < 0 || n_pairs >= 0x7fffffffLL) return fail(IVHD_ERR_INVALID_ARG, "bad pair count");
  for (int64_t p = 0; p < n_pairs; ++p)
    if (i_idx[p] < 0 || i_idx[p] >= m || j_idx[p] < 0 || j_idx[p] >= m || i_idx[p] == j_idx[p])
      return fail(IVHD_ERR_INVALID_ARG, "pair %lld out of range or self", (long long)p);
  if (n_pairs == 0) return IVHD_OK;
  // pairs grouped by i (stable), distinct rows in ascending order
  std::vector<int64_t> ord(n_pairs);
  for (int64_t p = 0; p < n_pairs; ++p) ord[p] = p;
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return i_idx[a] < i_idx[b]; });
  std::vector<int64_t> rows;
  std::vector<int> row_of(n_pairs);
  for (int64_t q = 0; q < n_pairs; ++q) {
    const int64_t p = ord[q];
    if (rows.empty() || rows.back() != i_idx[p]) rows.push_back(i_idx[p]);
    row_of[q] = (int)rows.size() - 1;
  }
  if (cudaSetDevice(device) != cudaSuccess) return fail(IVHD_ERR_CUDA, "cudaSetDevice(%d) failed", device);
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return fail(IVHD_ERR_CUDA, "stream");
  const int64_t nb_max = std::max<int64_t>(1, std::min<int64_t>((int64_t)rows.size(), ((int64_t)1 << 27) / m));
  double *dz = nullptr, *sq = nullptr, *a = nullptr, *sqa = nullptr, *blk = nullptr;
  int64_t *drows = nullptr, *dpi = nullptr, *dpj = nullptr, *dr = nullptr;
  int* dprow = nullptr;
  cudaError_t e = cudaSuccess;
  std::vector<int64_t> hpi(n_pairs), hpj(n_pairs), hr(n_pairs);
  std::vector<int> hprow(n_pairs);
  do {
#define MTRY(call) \
  if ((e = (call)) != cudaSuccess) break
    MTRY(cudaMallocAsync(&dz, sizeof(double) * m * n, st));
    MTRY(cudaMallocAsync(&sq, sizeof(double) * m, st));
    MTRY(cudaMallocAsync(&a, sizeof(double) * nb_max * n, st));
    MTRY(cudaMallocAsync(&sqa, sizeof(double) * nb_max, st));
    MTRY(cudaMallocAsync(&blk, sizeof(double) * nb_max * m, st));
    MTRY(cudaMallocAsync(&drows, sizeof(int64_t) * rows.size(), st));
    MTRY(cudaMallocAsync(&dpi, sizeof(int64_t) * n_pairs, st));
    MTRY(cudaMallocAsync(&dpj, sizeof(int64_t) * n_pairs, st));
    MTRY(cudaMallocAsync(&dr, sizeof(int64_t) * n_pairs, st));
    MTRY(cudaMallocAsync(&dprow, sizeof(int) * n_pairs, st));
    MTRY(cudaMemcpyAsync(dz, z, sizeof(double) * m * n, cudaMemcpyHostToDevice, st));
    MTRY(cudaMemcpyAsync(drows, rows.data(), sizeof(int64_t) * rows.size(), cudaMemcpyHostToDevice, st));
    k_sqnorm<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(dz, m, n, sq);
    // pair arrays in grouped order; prow = row index within its distance block
    for (int64_t q = 0; q < n_pairs; ++q) {
      hpi[q] = i_idx[ord[q]];
      hpj[q] = j_idx[ord[q]];
      hprow[q] = (int)(row_of[q] % nb_max);
    }
    MTRY(cudaMemcpyAsync(dpi, hpi.data(), sizeof(int64_t) * n_pairs, cudaMemcpyHostToDevice, st));
    MTRY(cudaMemcpyAsync(dpj, hpj.data(), sizeof(int64_t) * n_pairs, cudaMemcpyHostToDevice, st));
    MTRY(cudaMemcpyAsync(dprow, hprow.data(), sizeof(int) * n_pairs, cudaMemcpyHostToDevice, st));
    int64_t q0 = 0;
    for (int64_t r0 = 0; r0 < (int64_t)rows.size(); r0 += nb_max) {
      const int nb = (int)std::min<int64_t>(nb_max, (int64_t)rows.size() - r0);
      k_gather_rows<<<nb, 128, 0, st>>>(dz, sq, n, drows + r0, nb, a, sqa);
      dim3 grid((unsigned)((m + DT - 1) / DT), (unsigned)((nb + DT - 1) / DT));
      k_dist_block<<<grid, 256, 0, st>>>(a, sqa, dz, sq, m, n, nb, blk);
      int64_t q1 = q0;
      while (q1 < n_pairs && row_of[q1] < r0 + nb) ++q1;
      if (q1 > q0) k_pair_count<<<(unsigned)(q1 - q0), 256, 0, st>>>(blk, m, dprow + q0, dpi + q0, dpj + q0,
                                                                   (int)(q1 - q0), dr + q0);
      MTRY(cudaGetLastError());
      q0 = q1;
    }
    if (e != cudaSuccess) break;
    MTRY(cudaMemcpyAsync(hr.data(), dr, sizeof(int64_t) * n_pairs, cudaMemcpyDeviceToHost, st));
    MTRY(cudaStreamSynchronize(st));
    for (int64_t q = 0; q < n_pairs; ++q) ranks_out[ord[q]] = hr[q];
#undef MTRY
  } while (0);
  for (void* p : {(void*)dz, (void*)sq, (void*)a, (void*)sqa, (void*)blk, (void*)drows, (void*)dpi, (void*)dpj,
                  (void*)dr, (void*)dprow})
    if (p) cudaFreeAsync(p, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (e != cudaSuccess) return fail(IVHD_ERR_CUDA, "pair_ranks: %s", cudaGetErrorString(e));
  return IVHD_OK;
}


int ivhd_rank_matrix(int device, const double* x, int64_t m, int32_t n, int32_t precomputed, int64_t* ranks_out) {
  using namespace curves;
  if (!x || !ranks_out) return fail(IVHD_ERR_INVALID_ARG, "null pointer");
  if (m < 2) return fail(IVHD_ERR_INVALID_ARG, "need at least two points to rank");
  if (m >= (1LL << 31) / 2 || (precomputed ? n != m : n < 1))
    return fail(IVHD_ERR_INVALID_ARG, "bad shape (m=%lld, n=%d)", (long long)m, n);
  if (cudaSetDevice(device) != cudaSuccess) return fail(IVHD_ERR_CUDA, "cudaSetDevice(%d) failed", device);
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return fail(IVHD_ERR_CUDA, "stream");
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  // per block entry: distance 8 + keys 2x8 + vals 2x4 + ranks 8 = 40 bytes; <= 1 GiB, < 2^31 entries
  const int64_t nb_max = std::max<int64_t>(1, std::min<int64_t>(m, std::min<int64_t>(((int64_t)1 << 30) / (40 * m),
                                                                                      ((int64_t)1 << 31) / m - 1)));
  double *dx = nullptr, *sq = nullptr, *blk = nullptr;
  unsigned long long *k1 = nullptr, *k2 = nullptr;
  int *v1 = nullptr, *v2 = nullptr, *off = nullptr;
  int64_t* rk = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  cudaError_t e = cudaSuccess;
  const unsigned g = (unsigned)std::min<int64_t>((nb_max * m + 255) / 256, (int64_t)sms * 32);
  do {
#define MTRY(call) \
  if ((e = (call)) != cudaSuccess) break
    MTRY(cudaMallocAsync(&blk, sizeof(double) * nb_max * m, st));
    MTRY(cudaMallocAsync(&k1, 8 * nb_max * m, st));
    MTRY(cudaMallocAsync(&k2, 8 * nb_max * m, st));
    MTRY(cudaMallocAsync(&v1, 4 * nb_max * m, st));
    MTRY(cudaMallocAsync(&v2, 4 * nb_max * m, st));
    MTRY(cudaMallocAsync(&rk, 8 * nb_max * m, st));
    MTRY(cudaMallocAsync(&off, 4 * (nb_max + 1), st));
    if (!precomputed) {
      MTRY(cudaMallocAsync(&dx, sizeof(double) * m * n, st));
      MTRY(cudaMallocAsync(&sq, sizeof(double) * m, st));
      MTRY(cudaMemcpyAsync(dx, x, sizeof(double) * m * n, cudaMemcpyHostToDevice, st));
      k_sqnorm<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(dx, m, n, sq);
    }
    MTRY(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tb, k1, k2, v1, v2, (int)(nb_max * m), (int)nb_max, off,
                                                  off + 1, 0, 64, st));
    MTRY(cudaMallocAsync(&tmp, std::max<size_t>(tb, 16), st));
    for (int64_t r0 = 0; r0 < m; r0 += nb_max) {
      const int nb = (int)std::min<int64_t>(nb_max, m - r0);
      if (precomputed) {
        MTRY(cudaMemcpyAsync(blk, x + r0 * m, sizeof(double) * nb * m, cudaMemcpyHostToDevice, st));
      } else {
        dim3 grid((unsigned)((m + DT - 1) / DT), (unsigned)((nb + DT - 1) / DT));
        k_dist_block<<<grid, 256, 0, st>>>(dx + r0 * n, sq + r0, dx, sq, m, n, nb, blk);
      }
      k_rank_keys<<<g, 256, 0, st>>>(blk, m, r0, nb, k1, v1);
      k_seg_offsets<<<(nb + 256) / 256, 256, 0, st>>>(off, nb, m);
      size_t tb2 = tb;
      MTRY(cub::DeviceSegmentedRadixSort::SortPairs(tmp, tb2, k1, k2, v1, v2, (int)(nb * m), nb, off, off + 1, 0, 64,
                                                    st));
      k_rank_scatter<<<g, 256, 0, st>>>(v2, m, r0, nb, rk);
      MTRY(cudaGetLastError());
      MTRY(cudaMemcpyAsync(ranks_out + r0 * m, rk, 8 * nb * m, cudaMemcpyDeviceToHost, st));
    }
    if (e != cudaSuccess) break;
    MTRY(cudaStreamSynchronize(st));
#undef MTRY
  } while (0);
  for (void* p : {(void*)dx, (void*)sq, (void*)blk, (void*)k1, (void*)k2, (void*)v1, (void*)v2, (void*)off, (void*)rk, tmp})
    if (p) cudaFreeAsync(p, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (e != cudaSuccess) return fail(IVHD_ERR_CUDA, "rank_matrix: %s", cudaGetErrorString(e));
  return IVHD_OK;
}

}  // extern "C"
