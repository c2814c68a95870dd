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

constexpr int NH_MAX = 128;              // neighbourhood sizes supported (4 slots per lane)
constexpr int SPL = NH_MAX / 32;
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

// One warp per query (queries visited in cell order for cache locality).
__global__ void __launch_bounds__(QWARPS * 32) k_grid_knn(const double* __restrict__ ys, const int32_t* __restrict__ sid,
                                                         const uint32_t* __restrict__ start, int64_t m, Grid G, int kk,
                                                         const int32_t* __restrict__ labels,
                                                         unsigned long long* __restrict__ hits,
                                                         int32_t* __restrict__ nbr_out) {
  __shared__ unsigned int sh_hits[NH_MAX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < NH_MAX; i += blockDim.x) sh_hits[i] = 0;
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
    k_grid_knn<<<blocks, QWARPS * 32, 0, st>>>(ys, sid, start, m, G, nn_max, dl, hits, dn);
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

}  // extern "C"
