// ivhd_capi.cu — context, symmetrised-CSR builder, launch plumbing and the
// extern "C" entry points declared in include/ivhd_b200.h.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/ivhd_b200.h"
#include "ivhd_kernels.h"
#include "ivhd_rng.cuh"

using namespace ivhd;

namespace {

thread_local std::string g_error;

struct CsrSlot {
  uint32_t* row_ptr = nullptr;  // [M+1]
  uint32_t* col = nullptr;      // [n]
  float2* ew = nullptr;         // [n] or nullptr (binary)
  uint8_t* tile_g = nullptr;    // [n_tiles_cap] lanes per vertex of each tile
  uint32_t* tile_dm = nullptr;  // [n_tiles_cap] max row length of each tile
  int* units = nullptr;         // work units (tile << 12 | pass << 7 | min(slots per lane,15) << 3 | log2 G)
  int n_units = 0;
  std::vector<int> unit_base;   // host: first unit of each tile (n_tiles_cap + 1)
  int* d_unit_base = nullptr;   // device copy (sharded fold of unit partials into tile partials)
  std::vector<int> unit_words;  // host copy of units
  std::vector<int> unit_cost;   // host: modelled cost of each unit (slot rounds per lane)
  int sched_grid = 0;           // grid the cost-balanced schedule below was built for
  int sched_u0 = 0, sched_u1 = 0;  // ... and its unit range
  int* sched_units = nullptr;   // units regrouped per block (fused mode)
  int* sched_off = nullptr;     // [sched_grid + 1]
  int64_t n = 0;                // entries (2 * connections)
  int64_t cap = 0;
  bool valid = false;
};


struct GraphKey {
  int slot, norm, opt, G;
  bool operator<(const GraphKey& o) const {
    return std::tie(slot, norm, opt, G) < std::tie(o.slot, o.norm, o.opt, o.G);
  }
};

}  // namespace

struct ivhd_ctx {
  int device = 0;
  int64_t m = 0;
  int dim = 2;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sm_count = 148;

  int tile_v = kBlock;  // vertices per tile (fixed: reduction order independent of grid/ranks)
  int n_tiles = 0;
  int n_tiles_cap = 0;  // padded to a multiple of 8 (rank counts 1/2/4/8)
  int64_t v_cap = 0;    // vertex capacity of position/state buffers

  CsrSlot slots[2];
  // Vertex relabelling (new id -> old id and back), fixed by the first CSR
  // build: vertices sorted by descending degree so a tile's rows have
  // near-equal length.  All device vertex arrays are in the new order.
  int32_t* perm = nullptr;
  int32_t* inv = nullptr;
  bool perm_fixed = false;
  bool window_order = false;  // locality-ordered input: degree sort inside id windows, in-order schedule

  float* ybuf[2] = {nullptr, nullptr};  // 8 floats/vertex capacity
  float* state = nullptr;               // 2 buffers x state_fpv floats/vertex (ctrl.scur = current)
  int state_fpv = 8;                    // 16 for fp64 Adam in 3-D
  // degenerate random pairs (forces.py:167-174): host-drawn direction table + kernel misses
  int2* dg_key = nullptr;
  float4* dg_vec = nullptr;
  int64_t dg_cap = 0;
  int* miss_n = nullptr;
  int2* miss = nullptr;
  int miss_cap = 4096;
  bool op_paused = false;  // an operator call (not the loop) is waiting for directions
  double4* partial = nullptr;  // per work unit (sharded / operator calls)
  double4* tpart = nullptr;    // per tile [n_tiles_cap]: the array ranks exchange (sharded)
  double4* bpart = nullptr;  // one per resident block of the step kernel
  double2* trace = nullptr;
  int64_t trace_cap = 0;
  Ctrl* ctrl = nullptr;      // device
  Ctrl* ctrl_h = nullptr;    // pinned host mirror
  Ctrl* opctrl = nullptr;    // device, operator calls
  double4* red_out = nullptr;

  // scratch
  double* stage = nullptr;  // (v_cap * 4) doubles: host <-> device conversion
  float* op_y = nullptr;    // operator positions (8 floats/vertex)
  double* op_force = nullptr;
  float* snap_y = nullptr;      // snapshot: positions (8 floats/vertex)
  float* snap_state = nullptr;  // snapshot: optimizer state
  Ctrl snap_ctrl{};
  bool snap_valid = false;

  ivhd_optimizer_params opt{};
  bool opt_set = false;
  bool pos_set = false;
  Hyper hyper{};

  int64_t shard_begin = 0, shard_end = 0;  // sharded mode range (0,0 = whole)
  bool sharded = false;
  int shard_cur = 0;    // async sharded loop: host-side copy of the current buffer index
  int shard_slot = 0;   // connection slot of the last ivhd_shard_step
  int64_t graph_epoch = 0;  // bumped whenever captured launch arguments go stale

  // fused peer exchange (ivhd_peer_*): buffers peers write into are cudaMalloc'd (IPC)
  bool peer_on = false;
  int world = 1, rank = 0;
  bool ybuf_malloc = false;            // ybuf[0..1] are cudaMalloc (not pool) memory
  double4* tp2 = nullptr;              // [2][world][8 * SMs] block partials by stamp parity
  int64_t tp2_slots = 0;
  unsigned long long* flags = nullptr; // [8] arrival flags, one slot per rank
  unsigned long long* stamp = nullptr; // iterations exchanged
  PeerArgs pe{};
  uint8_t* hmask = nullptr;            // [v_cap] halo masks (ranks that gather each own vertex)
  bool masks_stale = true;
  std::vector<void*> ipc_opened;       // cudaIpcOpenMemHandle pointers to close

  std::map<GraphKey, cudaGraphExec_t> graphs;
  int graph_chunk = 64;

  std::map<KernelFn, int> occ;  // blocks per SM
  std::string err;
};

namespace {

template <class T>
inline cudaError_t dalloc(ivhd_ctx* ctx, T** p, size_t bytes) {
  return cudaMallocAsync(reinterpret_cast<void**>(p), bytes, ctx->stream);
}
template <class T>
inline void dfree(ivhd_ctx* ctx, T* p) {
  if (p) cudaFreeAsync(reinterpret_cast<void*>(const_cast<typename std::remove_const<T>::type*>(p)), ctx->stream);
}

// Pinned host mirrors of Ctrl come from a process-wide pool: cudaFreeHost
// synchronises the device and can take 100+ ms, so blocks are recycled and
// never returned to the driver (one page serves 32 live contexts).
std::mutex g_pinned_mu;
std::vector<Ctrl*> g_pinned_free;

Ctrl* pinned_ctrl_get() {
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  if (g_pinned_free.empty()) {
    constexpr int kPer = 32;
    Ctrl* page = nullptr;
    if (cudaMallocHost(&page, sizeof(Ctrl) * kPer) != cudaSuccess) return nullptr;
    for (int i = kPer - 1; i >= 0; --i) g_pinned_free.push_back(page + i);
  }
  Ctrl* c = g_pinned_free.back();
  g_pinned_free.pop_back();
  *c = Ctrl{};
  return c;
}

void pinned_ctrl_put(Ctrl* c) {
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  g_pinned_free.push_back(c);
}

int fail(ivhd_ctx* ctx, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  g_error = buf;
  return code;
}

#define CU(ctx, call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(ctx, IVHD_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                 \
  } while (0)

#define TRY(expr)               \
  do {                          \
    int r_ = (expr);            \
    if (r_ != IVHD_OK) return r_; \
  } while (0)

// Stream-ordered allocation on the context stream: no device-wide syncs,
// and the default pool keeps freed memory for the next context (see create).
template <class T>
inline cudaError_t dalloc(ivhd_ctx* ctx, T** p, size_t bytes);
template <class T>
inline void dfree(ivhd_ctx* ctx, T* p);

// floats per vertex of a position buffer: fp32 (y | y + beta v for
// Nesterov), or fp64 for Adam (ivhd_step_f64.cuh)
inline int ys_of(int dim, int opt) {
  return (opt == OPT_NEST || opt == OPT_ADAM) ? (dim == 2 ? 4 : 8) : (dim == 2 ? 2 : 4);
}
inline bool f64_of(int opt) { return opt == OPT_ADAM; }

// ------------------------------------------------------------ kernel table

KernelFn pick_finalize_peer(int opt) {
  switch (opt) {
    case OPT_FD: return finalize_peer_kernel<OPT_FD>;
    case OPT_ADAM: return finalize_peer_kernel<OPT_ADAM>;
    default: return finalize_peer_kernel<OPT_SGD>;
  }
}

KernelFn pick_finalize(int opt) {
  switch (opt) {
    case OPT_FD: return finalize_kernel<OPT_FD>;
    case OPT_ADAM: return finalize_kernel<OPT_ADAM>;
    default: return finalize_kernel<OPT_SGD>;
  }
}

int occupancy(ivhd_ctx* ctx, KernelInfo k) {
  auto it = ctx->occ.find(k.fn);
  if (it != ctx->occ.end()) return it->second;
  cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, k.smem);
  int n = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k.fn, k.threads, k.smem) != cudaSuccess || n < 1) n = 1;
  ctx->occ[k.fn] = n;
  return n;
}

// ------------------------------------------------------------ small kernels

__global__ void k_half_edges(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                             int64_t L, int64_t m, uint32_t* __restrict__ keys,
                             uint32_t* __restrict__ vals, int* __restrict__ bad) {
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < 2 * L;
       h += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = h < L ? src[h] : dst[h - L];
    if (r < 0 || r >= m) *bad = 1;
    keys[h] = (uint32_t)max(0, min((int32_t)(m - 1), r));
    vals[h] = (uint32_t)h;
  }
}

__global__ void k_row_ptr(const uint32_t* __restrict__ keys, int64_t n, int64_t m,
                          uint32_t* __restrict__ row_ptr) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= m;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;  // first k with keys[k] >= r
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < (uint32_t)r) lo = mid + 1; else hi = mid;
    }
    row_ptr[r] = (uint32_t)lo;
  }
}

__global__ void k_binary_edges(const int32_t* __restrict__ nn, int64_t stride, int ncols,
                               const int32_t* __restrict__ rn, int nrn, int64_t m,
                               int32_t* __restrict__ src, int32_t* __restrict__ dst) {
  const int64_t n_nn = m * ncols, L = n_nn + m * nrn;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < L;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < n_nn) {
      const int64_t i = e / ncols;
      src[e] = (int32_t)i;
      dst[e] = nn[i * stride + (e - i * ncols)];
    } else {
      const int64_t q = e - n_nn, i = q / nrn;
      src[e] = (int32_t)i;
      dst[e] = rn[q];
    }
  }
}

__global__ void k_split_edges(const int32_t* __restrict__ edges, int64_t L,
                              int32_t* __restrict__ src, int32_t* __restrict__ dst) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < L;
       e += (int64_t)gridDim.x * blockDim.x) {
    src[e] = edges[2 * e];
    dst[e] = edges[2 * e + 1];
  }
}

__global__ void k_d2f(const double* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (float)in[i];
}

// host double (m, dim) in caller order -> device layout (stride ys) in the
// relabelled order: out[r] = y[perm[r]]; Nesterov look = y + beta*v
__global__ void k_pack_positions(const double* __restrict__ y, int64_t m, int dim, int ys,
                                 const int32_t* __restrict__ perm, const float* __restrict__ vel,
                                 int vel_stride, float beta, float* __restrict__ out, int f64 = 0) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    float* o = out + i * ys;
    const int64_t src = perm[i];
    if (f64) {  // fp64 layout (Adam): ys / 2 doubles per vertex
      for (int d = 0; d < dim; ++d) reinterpret_cast<double*>(o)[d] = y[src * dim + d];
      continue;
    }
    const int look_off = (ys == 4 && dim == 2) ? 2 : 4;
    for (int d = 0; d < dim; ++d) {
      const float v = (float)y[src * dim + d];
      o[d] = v;
      if (vel) o[look_off + d] = v + beta * vel[i * vel_stride + d];
    }
  }
}

// device layout (relabelled) -> double (m, dim) in caller order
__global__ void k_unpack_positions(const float* __restrict__ in, int64_t m, int dim, int ys,
                                   const int32_t* __restrict__ perm, double* __restrict__ y, int f64 = 0) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t dst = perm[i];
    if (f64) {
      const double* q = reinterpret_cast<const double*>(in + i * ys);
      for (int d = 0; d < dim; ++d) y[dst * dim + d] = q[d];
    } else {
      for (int d = 0; d < dim; ++d) y[dst * dim + d] = (double)in[i * ys + d];
    }
  }
}

__global__ void k_unpermute_f64(const double* __restrict__ in, int64_t m, int dim,
                                const int32_t* __restrict__ perm, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int d = 0; d < dim; ++d) out[(int64_t)perm[i] * dim + d] = in[i * dim + d];
}

__global__ void k_deltas(const float* __restrict__ a, const float* __restrict__ b, int64_t m,
                         int dim, int ys, int commit, const int32_t* __restrict__ perm,
                         double* __restrict__ out, int f64 = 0) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t dst = perm[i];
    for (int d = 0; d < dim; ++d) {
      double va, vb;
      if (f64) {
        va = reinterpret_cast<const double*>(a + i * ys)[d];
        vb = reinterpret_cast<const double*>(b + i * ys)[d];
      } else {
        va = a[i * ys + d];
        vb = b[i * ys + d];
      }
      out[dst * dim + d] = commit ? va - vb : 0.0;
    }
  }
}

__global__ void k_iota(int32_t* __restrict__ a, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (int32_t)i;
}

__global__ void k_degrees(const uint32_t* __restrict__ row_ptr, int64_t m, uint32_t* __restrict__ deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    deg[i] = row_ptr[i + 1] - row_ptr[i];
}

// Windowed relabelling key: windows of W consecutive ids stay in order, ids
// inside a window are sorted by descending degree (descending sort on
// (reversed window << 32 | degree)).
__global__ void k_window_keys(const uint32_t* __restrict__ row_ptr, int64_t m, int64_t W,
                              uint64_t* __restrict__ key) {
  const int64_t nwin = (m + W - 1) / W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    key[i] = ((uint64_t)(nwin - 1 - i / W) << 32) | (uint64_t)(row_ptr[i + 1] - row_ptr[i]);
}

// Locality statistic of the caller's ids: connections whose endpoints lie
// within kOrderWindow ids of each other (integer count, order independent).
__global__ void k_local_edges(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t L,
                              int64_t W, unsigned long long* __restrict__ count) {
  unsigned long long c = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < L; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = (int64_t)src[e] - (int64_t)dst[e];
    c += (d < W && d > -W) ? 1ull : 0ull;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// Sharded relabelling: deal the degree-sorted vertices (position p of
// `sorted`) over the 8 rank groups of C ids in snake order (0..7, 7..0, ...),
// so every group gets the same mix of hubs and leaves, i.e. equal edge
// counts for equal vertex ranges.  Groups g < gfull hold C ids, group gfull
// holds cap_p < C (the padded tail), later groups none: the first
// (gfull + 1) * cap_p positions are dealt over gfull + 1 groups, the rest
// over the gfull full ones.  Always 8 groups, so the order (and the fixed
// tile reduction order) is the same for 1, 2, 4 and 8 ranks.
__global__ void k_snake_deal(const int32_t* __restrict__ sorted, int64_t m, int64_t C, int gfull, int64_t cap_p,
                             int32_t* __restrict__ out) {
  const int64_t n1 = (int64_t)(gfull + 1) * cap_p;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
    int64_t g, idx;
    if (p < n1) {
      const int64_t n = gfull + 1, r = p / n, j = p % n;
      g = (r & 1) ? n - 1 - j : j;
      idx = r;
    } else {
      const int64_t q = p - n1, n = gfull, r = q / n, j = q % n;
      g = (r & 1) ? n - 1 - j : j;
      idx = cap_p + r;
    }
    out[g * C + idx] = sorted[p];
  }
}

__global__ void k_inverse(const int32_t* __restrict__ perm, int64_t m, int32_t* __restrict__ inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    inv[perm[i]] = (int32_t)i;
}

// out[r] = in[src(r)] for rows of `stride` floats; src(r) = inv_old[perm_new[r]]
__global__ void k_permute_rows(const float* __restrict__ in, int64_t m, int stride,
                               const int32_t* __restrict__ perm_new, const int32_t* __restrict__ inv_old,
                               float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t src = inv_old[perm_new[i]];
    for (int d = 0; d < stride; ++d) out[i * stride + d] = in[src * stride + d];
  }
}

// new-order degrees: deg_n[r] = deg_o[perm[r]]
__global__ void k_gather_u32(const uint32_t* __restrict__ in, const int32_t* __restrict__ perm, int64_t m,
                             uint32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[perm[i]];
}

// One warp per relabelled row: copy the old row's entries in order, mapping
// the neighbour id through inv and attaching the class bit / weights.
__global__ void k_fill_perm_cols(const uint32_t* __restrict__ rp_old, const uint32_t* __restrict__ rp_new,
                                 const uint32_t* __restrict__ vals, int64_t m, int64_t L,
                                 const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                 const uint8_t* __restrict__ rand, int64_t n_nn,
                                 const float* __restrict__ tgt, const float* __restrict__ scl,
                                 const int32_t* __restrict__ perm, const int32_t* __restrict__ inv,
                                 uint32_t* __restrict__ col, float2* __restrict__ ew) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < m; r += nwarps) {
    const int64_t o = perm[r];
    const uint32_t b0 = rp_old[o], b1 = rp_old[o + 1], nb = rp_new[r];
    for (uint32_t k = b0 + lane; k < b1; k += 32) {
      const int64_t h = vals[k];
      const int64_t e = h < L ? h : h - L;
      const uint32_t other = (uint32_t)inv[h < L ? dst[e] : src[e]];
      const bool rn = rand ? (rand[e] != 0) : (e >= n_nn);
      const uint32_t kn = nb + (k - b0);
      col[kn] = other | (rn ? kRandBit : 0u);
      if (ew) ew[kn] = make_float2(tgt ? tgt[e] : (rn ? 1.f : 0.f), scl ? scl[e] : 1.f);
    }
  }
}

// Lanes per vertex of each tile: smallest power of two G with
// G * kUnroll >= the tile's max degree (capped at a warp); pad tiles get 1.
__global__ void k_tile_g(const uint32_t* __restrict__ rp, int64_t m, int n_tiles_cap,
                         uint8_t* __restrict__ tile_g, uint32_t* __restrict__ tile_dm) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < n_tiles_cap; t += nwarps) {
    uint32_t mx = 0;
    for (int64_t r = t * kBlock + lane; r < min(m, (t + 1) * (int64_t)kBlock); r += 32)
      mx = max(mx, rp[r + 1] - rp[r]);
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int G = 1;
    while (G < 32 && (uint32_t)(G * kUnroll) < mx) G <<= 1;
    if (lane == 0) {
      tile_g[t] = (uint8_t)G;
      tile_dm[t] = mx;  // unclamped: the slots-per-lane bound must cover hub rows
    }
  }
}

// Sharded mode: fold this rank's work-unit partials into one partial per tile
// (units of a tile in unit order), so the exchanged array is indexed by tile
// and every rank owns the contiguous chunk of its tile range.
// (unit_base == nullptr: the fp64 kernel wrote tile partials already).  The
// rank's first tile also carries 2^32 if this rank met degenerate pairs
// without a direction (decide pauses every rank then).
__global__ void k_fold_tiles(const double4* __restrict__ unit_part, const int* __restrict__ unit_base, int t0,
                             int t1, double4* __restrict__ tpart, Ctrl* ctrl) {
  for (int t = t0 + blockIdx.x * blockDim.x + threadIdx.x; t < t1; t += gridDim.x * blockDim.x) {
    double4 s = make_double4(0, 0, 0, 0);
    if (unit_base) {
      for (int u = unit_base[t]; u < unit_base[t + 1]; ++u) {
        const double4 q = unit_part[u];
        s.x += q.x; s.y += q.y; s.z += q.z; s.w += q.w;
      }
    } else {
      s = tpart[t];
    }
    if (t == t0 && ctrl->need) {
      s.w += kMissUnit;
      ctrl->need = 0;
    }
    tpart[t] = s;
  }
}

// Halo masks of this rank's vertices: bit r of mask[v] is set when a row
// owned by rank r (r != own) lists v, i.e. rank r gathers v's position.  The
// symmetrised CSR makes that the set of ranks of v's own row entries.
__global__ void k_halo_mask(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ col, int64_t v0,
                            int64_t v1, int64_t range_v, int own, uint8_t* __restrict__ mask) {
  for (int64_t v = v0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < v1; v += (int64_t)gridDim.x * blockDim.x) {
    unsigned mk = mask[v];
    for (uint32_t k = rp[v]; k < rp[v + 1]; ++k) mk |= 1u << (int)((col[k] & kIdMask) / range_v);
    mask[v] = (uint8_t)(mk & ~(1u << own));
  }
}

// After a peer-mode run: complete this rank's replica (both buffers) with
// every peer's own range read over NVLink — the halo exchange only kept the
// entries this rank gathers current.
__global__ void k_peer_pull(float4* __restrict__ dst0, float4* __restrict__ dst1, const float4* __restrict__ src0,
                            const float4* __restrict__ src1, int64_t f4_begin, int64_t f4_end) {
  for (int64_t i = f4_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < f4_end;
       i += (int64_t)gridDim.x * blockDim.x) {
    dst0[i] = src0[i];
    dst1[i] = src1[i];
  }
}

// All-rank barrier at the end of a peer-mode segment: raise flag [8 + rank]
// on every rank, wait until all ranks raised theirs (same timeout and status
// 3 as the finalizer).
__global__ void k_peer_barrier(PeerArgs pe, Ctrl* ctrl) {
  const unsigned long long s = pe.stamp[1] + 1;
  __syncwarp();
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(pe.fl_local + 8 + pe.rank, s);
    for (int q = 0; q < pe.n_peers; ++q) st_release_sys(pe.fl[q] + 8 + pe.rank, s);
  }
  if (threadIdx.x < pe.world) {
    long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (ld_acquire_sys(pe.fl_local + 8 + threadIdx.x) < s) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > pe.timeout_ns) {
        ctrl->status = 3;
        break;
      }
      __nanosleep(100);
    }
  }
  __syncwarp();
  if (threadIdx.x == 0) pe.stamp[1] = s;
}

// Positions a paused iteration evaluated its forces at, in the operator
// layout (ys_out floats per vertex): y itself, or Nesterov's y + beta v (at
// float offset `off` of the record).
__global__ void k_eval_positions(const float* __restrict__ y, int64_t m, int ys_in, int off, int dim, int ys_out,
                                 float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    for (int d = 0; d < ys_out; ++d) out[i * ys_out + d] = d < dim ? y[i * ys_in + off + d] : 0.f;
}

// Undo the in-place fp32 state update of a paused iteration from the forces
// it used (optim.py:95-236 solved for the old state; recovered to rounding).
template <int DIM, int OPT>
__global__ void k_unstep(float* __restrict__ state, const double* __restrict__ force, int64_t m, float step, Hyper h) {
  using L = Layout<DIM, OPT>;
  constexpr int V = DIM == 2 ? 2 : 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    float* sv = state + i * L::SS;
    for (int d = 0; d < DIM; ++d) {
      const double f = force[i * DIM + d], g = -2.0 * f;
      if constexpr (OPT == OPT_FD) {  // dn = a d + b f
        sv[d] = (float)(((double)sv[d] - (double)(step * (float)f)) / (double)h.a);
      } else if constexpr (OPT == OPT_MOM || OPT == OPT_NEST) {  // v' = beta v - alpha g
        sv[d] = (float)(((double)sv[d] + (double)step * g) / (double)h.beta);
      } else if constexpr (OPT == OPT_ADADELTA) {
        const double rho = h.rho, eps = h.eps, sg_new = sv[d], sd_new = sv[V + d];
        const double k = (double)step * step * g * g / (sg_new + eps);
        sv[d] = (float)((sg_new - (1.0 - rho) * g * g) / rho);
        sv[V + d] = (float)((sd_new - (1.0 - rho) * k * eps) / (rho + (1.0 - rho) * k));
      }
    }
  }
}

// {target, scale} per entry of a binary connection set (rn -> 1, nn -> 0;
// scale 1): lets the weighted kernel instantiation re-run a paused iteration.
__global__ void k_binary_ew(const uint32_t* __restrict__ col, int64_t n, float2* __restrict__ ew) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    ew[k] = make_float2((col[k] & kRandBit) ? 1.f : 0.f, 1.f);
}

// fixed-order reduction of partial tiles into one double4 (operator calls)
__global__ void __launch_bounds__(kBlock) k_reduce_partials(const double4* __restrict__ p, int n,
                                                            double4* __restrict__ out) {
  __shared__ double4 sm[kBlock / 32];
  double4 s = make_double4(0, 0, 0, 0);
  for (int t = threadIdx.x; t < n; t += kBlock) {
    const double4 q = p[t];
    s.x += q.x; s.y += q.y; s.z += q.z; s.w += q.w;
  }
  s = block_sum4(s, sm);
  if (threadIdx.x == 0) *out = s;
}

inline int grid_for(int64_t n, int sms) {
  const int64_t g = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sms * 16));
}

// ------------------------------------------------------------- CSR builder

int ensure_slot(ivhd_ctx* ctx, CsrSlot& s, int64_t n, bool weighted) {
  // +16 entries: TMA copies round sizes up to 16 bytes
  if (s.row_ptr == nullptr) CU(ctx, dalloc(ctx, &s.row_ptr, sizeof(uint32_t) * (ctx->m + 1 + 16)));
  if (s.tile_g == nullptr) CU(ctx, dalloc(ctx, &s.tile_g, (size_t)ctx->n_tiles_cap));
  if (s.tile_dm == nullptr) CU(ctx, dalloc(ctx, &s.tile_dm, sizeof(uint32_t) * ctx->n_tiles_cap));
  if (n > s.cap) {
    if (s.col) dfree(ctx, s.col);
    if (s.ew) dfree(ctx, s.ew);
    s.col = nullptr;
    s.ew = nullptr;
    CU(ctx, dalloc(ctx, &s.col, sizeof(uint32_t) * (std::max<int64_t>(n, 1) + 16)));
    s.cap = n;
  }
  if (weighted && s.ew == nullptr) CU(ctx, dalloc(ctx, &s.ew, sizeof(float2) * std::max<int64_t>(s.cap, 1)));
  if (!weighted && s.ew != nullptr) {
    dfree(ctx, s.ew);
    s.ew = nullptr;
  }
  return IVHD_OK;
}

void drop_graphs(ivhd_ctx* ctx) {
  for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
  ctx->graphs.clear();
  ++ctx->graph_epoch;  // callers' own captures (sharded loop) must be redone too
}

int ys_now(ivhd_ctx* ctx);
int ss_now(ivhd_ctx* ctx);
int64_t state_stride(ivhd_ctx* ctx);
float* state_buf(ivhd_ctx* ctx, int b);
int pull_ctrl(ivhd_ctx* ctx);

// Fix the vertex order from the degrees of the first CSR built: stable sort
// by descending degree (hubs first, so the dynamic tile scheduler starts the
// longest tiles early).  Positions/state already uploaded are re-ordered.
//
// Locality-ordered inputs (at least half of the connections join ids less
// than kOrderWindow apart, e.g. the planted graphs of C4/C5) instead sort by
// degree inside windows of kOrderWindow ids and run the tiles in order, so a
// tile's nn partners stay in the same few L2 lines: 10^8 planted 6217 ->
// 5481 us per iteration, 10^7 271 -> 265 (profiles/r01_kernel_experiments.md).
// Inputs without id locality (real kNN graphs) keep the global degree sort:
// windows cost them 2.6x in load imbalance.
constexpr int64_t kOrderWindow = 2048;

int fix_permutation(ivhd_ctx* ctx, const uint32_t* rp_old, const int32_t* src, const int32_t* dst, int64_t L) {
  const int64_t m = ctx->m;
  cudaStream_t st = ctx->stream;
  int64_t window = 0;
  if (L > 0 && m > 2 * kOrderWindow) {
    unsigned long long* dcount = nullptr;
    unsigned long long hcount = 0;
    cudaError_t e0 = dalloc(ctx, &dcount, sizeof(unsigned long long));
    if (e0 == cudaSuccess) e0 = cudaMemsetAsync(dcount, 0, sizeof(unsigned long long), st);
    if (e0 == cudaSuccess) {
      k_local_edges<<<grid_for(L, ctx->sm_count), 256, 0, st>>>(src, dst, L, kOrderWindow, dcount);
      e0 = cudaMemcpyAsync(&hcount, dcount, sizeof(hcount), cudaMemcpyDeviceToHost, st);
    }
    if (e0 == cudaSuccess) e0 = cudaStreamSynchronize(st);
    dfree(ctx, dcount);
    if (e0 != cudaSuccess) return fail(ctx, IVHD_ERR_CUDA, "locality statistic: %s", cudaGetErrorString(e0));
    if (2 * (int64_t)hcount >= L) window = kOrderWindow;
  }
  ctx->window_order = window > 0 && window < m;
  uint32_t *deg = nullptr, *deg2 = nullptr;
  int32_t *ids = nullptr, *perm = nullptr;
  float* big_scratch = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  TRY(pull_ctrl(ctx));
  cudaError_t e = cudaSuccess;
  do {
    if ((e = dalloc(ctx, &deg, 4 * m)) != cudaSuccess) break;
    if ((e = dalloc(ctx, &deg2, 4 * m)) != cudaSuccess) break;
    if ((e = dalloc(ctx, &ids, 4 * m)) != cudaSuccess) break;
    if ((e = dalloc(ctx, &perm, 4 * m)) != cudaSuccess) break;
    k_iota<<<grid_for(m, ctx->sm_count), 256, 0, st>>>(ids, m);
    if (ctx->window_order) {
      uint64_t *k1 = nullptr, *k2 = nullptr;
      int eb = 33;
      while (eb < 64 && ((int64_t)1 << (eb - 32)) < (m + window - 1) / window) ++eb;
      do {
        if ((e = dalloc(ctx, &k1, 8 * m)) != cudaSuccess) break;
        if ((e = dalloc(ctx, &k2, 8 * m)) != cudaSuccess) break;
        k_window_keys<<<grid_for(m, ctx->sm_count), 256, 0, st>>>(rp_old, m, window, k1);
        if ((e = cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, k1, k2, ids, perm, (int)m, 0, eb, st)) !=
            cudaSuccess) break;
        if ((e = dalloc(ctx, &tmp, std::max<size_t>(tb, 16))) != cudaSuccess) break;
        e = cub::DeviceRadixSort::SortPairsDescending(tmp, tb, k1, k2, ids, perm, (int)m, 0, eb, st);
      } while (0);
      dfree(ctx, k1);
      dfree(ctx, k2);
      if (e != cudaSuccess) break;
    } else {
      k_degrees<<<grid_for(m, ctx->sm_count), 256, 0, st>>>(rp_old, m, deg);
      if ((e = cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, deg, deg2, ids, perm, (int)m, 0, 32, st)) !=
          cudaSuccess) break;
      if ((e = dalloc(ctx, &tmp, std::max<size_t>(tb, 16))) != cudaSuccess) break;
      if ((e = cub::DeviceRadixSort::SortPairsDescending(tmp, tb, deg, deg2, ids, perm, (int)m, 0, 32, st)) !=
          cudaSuccess) break;
      if (ctx->sharded) {  // equal-edge rank groups (k_snake_deal); ids stays the scratch
        const int64_t C = (int64_t)(ctx->n_tiles_cap / 8) * ctx->tile_v;
        const int gfull = (int)(m / C);
        const int64_t cap_p = m - (int64_t)gfull * C;
        k_snake_deal<<<grid_for(m, ctx->sm_count), 256, 0, st>>>(perm, m, C, gfull, cap_p, ids);
        if ((e = cudaGetLastError()) != cudaSuccess) break;
        std::swap(ids, perm);
      }
    }
    if (ctx->pos_set) {
      // data is currently in the old order (ctx->perm / ctx->inv): re-order
      const int ys = ys_now(ctx), ss = ss_now(ctx);
      float* scratch = reinterpret_cast<float*>(ctx->stage);  // 32 bytes/vertex
      if (ss > 8) {  // fp64 Adam state in 3-D: 64 bytes/vertex
        if ((e = dalloc(ctx, &big_scratch, sizeof(float) * ss * m)) != cudaSuccess) break;
        scratch = big_scratch;
      }
      float* y = ctx->ybuf[ctx->ctrl_h->cur];
      k_permute_rows<<<grid_for(m, ctx->sm_count), 256, 0, st>>>(y, m, ys, perm, ctx->inv, scratch);
      if ((e = cudaMemcpyAsync(y, scratch, sizeof(float) * ys * m, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
        break;
      if (ss > 0) {
        float* sc = state_buf(ctx, ctx->ctrl_h->scur);
        k_permute_rows<<<grid_for(m, ctx->sm_count), 256, 0, st>>>(sc, m, ss, perm, ctx->inv, scratch);
        if ((e = cudaMemcpyAsync(sc, scratch, sizeof(float) * ss * m, cudaMemcpyDeviceToDevice, st)) !=
            cudaSuccess) break;
      }
    }
    if ((e = cudaMemcpyAsync(ctx->perm, perm, 4 * m, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) break;
    k_inverse<<<grid_for(m, ctx->sm_count), 256, 0, st>>>(ctx->perm, m, ctx->inv);
    e = cudaStreamSynchronize(st);
  } while (0);
  dfree(ctx, deg); dfree(ctx, deg2); dfree(ctx, ids); dfree(ctx, perm); dfree(ctx, tmp); dfree(ctx, big_scratch);
  if (e != cudaSuccess) return fail(ctx, IVHD_ERR_CUDA, "vertex relabelling: %s", cudaGetErrorString(e));
  ctx->perm_fixed = true;
  return IVHD_OK;
}

// src/dst: device int32 [L]; rand: device u8 [L] or null (then e >= n_nn is random);
// tgt/scl: device float [L] or null.  Builds the symmetrised CSR in the
// relabelled vertex order: row r lists every connection incident to vertex
// perm[r] — first those where it is the source, then those where it is the
// destination, each in connection order (the reference's edge order,
// engine.py:245-262) — so per-row summation order is independent of the
// relabelling.
int build_csr(ivhd_ctx* ctx, int slot, const int32_t* src, const int32_t* dst, const uint8_t* rand,
              int64_t n_nn, const float* tgt, const float* scl, int64_t L) {
  CsrSlot& S = ctx->slots[slot];
  const int64_t n = 2 * L, m = ctx->m;
  if (n >= (int64_t)0x7fffffffLL) return fail(ctx, IVHD_ERR_INVALID_ARG, "too many connections (%lld)", (long long)L);
  const bool weighted = (tgt != nullptr) || (scl != nullptr);
  TRY(ensure_slot(ctx, S, n, weighted));
  drop_graphs(ctx);
  S.valid = false;
  S.n = n;
  cudaStream_t st = ctx->stream;
  uint32_t *keys = nullptr, *keys2 = nullptr, *vals = nullptr, *vals2 = nullptr, *rp_old = nullptr, *deg = nullptr;
  int* bad = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int end_bit = 1;
  while (end_bit < 32 && ((int64_t)1 << end_bit) < m) ++end_bit;
  cudaError_t e = cudaSuccess;
  int hbad = 0, rc = IVHD_OK;
  const int64_t nc = std::max<int64_t>(n, 1);
  do {
    if ((e = dalloc(ctx, &keys, 4 * nc)) != cudaSuccess) break;
    if ((e = dalloc(ctx, &keys2, 4 * nc)) != cudaSuccess) break;
    if ((e = dalloc(ctx, &vals, 4 * nc)) != cudaSuccess) break;
    if ((e = dalloc(ctx, &vals2, 4 * nc)) != cudaSuccess) break;
    if ((e = dalloc(ctx, &rp_old, 4 * (m + 1))) != cudaSuccess) break;
    if ((e = dalloc(ctx, &deg, 4 * (m + 1))) != cudaSuccess) break;
    if ((e = dalloc(ctx, &bad, sizeof(int))) != cudaSuccess) break;
    if ((e = cudaMemsetAsync(bad, 0, sizeof(int), st)) != cudaSuccess) break;
    if (n > 0) {
      k_half_edges<<<grid_for(n, ctx->sm_count), 256, 0, st>>>(src, dst, L, m, keys, vals, bad);
      if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, vals, vals2, (int)n, 0, end_bit,
                                               st)) != cudaSuccess) break;
      if ((e = dalloc(ctx, &tmp, std::max<size_t>(tmp_bytes, 16))) != cudaSuccess) break;
      // LSD radix sort is stable: rows list out-halves (connection order) then in-halves.
      if ((e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, vals, vals2, (int)n, 0, end_bit,
                                               st)) != cudaSuccess) break;
      k_row_ptr<<<grid_for(m + 1, ctx->sm_count), 256, 0, st>>>(keys2, n, m, rp_old);
    } else {
      if ((e = cudaMemsetAsync(rp_old, 0, 4 * (m + 1), st)) != cudaSuccess) break;
    }
    if ((e = cudaGetLastError()) != cudaSuccess) break;
    if ((e = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
    if (hbad) break;
    if (!ctx->perm_fixed && (rc = fix_permutation(ctx, rp_old, src, dst, L)) != IVHD_OK) break;
    // relabelled row pointers: exclusive scan of the permuted degrees
    k_degrees<<<grid_for(m, ctx->sm_count), 256, 0, st>>>(rp_old, m, keys);
    k_gather_u32<<<grid_for(m, ctx->sm_count), 256, 0, st>>>(keys, ctx->perm, m, deg);
    if ((e = cudaMemsetAsync(deg + m, 0, 4, st)) != cudaSuccess) break;
    size_t sb = 0;
    if ((e = cub::DeviceScan::ExclusiveSum(nullptr, sb, deg, S.row_ptr, (int)(m + 1), st)) != cudaSuccess) break;
    void* stmp = nullptr;
    if ((e = dalloc(ctx, &stmp, std::max<size_t>(sb, 16))) != cudaSuccess) break;
    e = cub::DeviceScan::ExclusiveSum(stmp, sb, deg, S.row_ptr, (int)(m + 1), st);
    cudaStreamSynchronize(st);
    dfree(ctx, stmp);
    if (e != cudaSuccess) break;
    if (n > 0)
      k_fill_perm_cols<<<grid_for(m * 32, ctx->sm_count), 256, 0, st>>>(
          rp_old, S.row_ptr, vals2, m, L, src, dst, rand, n_nn, tgt, scl, ctx->perm, ctx->inv, S.col, S.ew);
    k_tile_g<<<grid_for((int64_t)ctx->n_tiles_cap * 32, ctx->sm_count), 256, 0, st>>>(S.row_ptr, m,
                                                                                     ctx->n_tiles_cap, S.tile_g, S.tile_dm);
    if ((e = cudaGetLastError()) != cudaSuccess) break;
    // work units: one per (tile, pass), in tile order
    std::vector<uint8_t> g(ctx->n_tiles_cap);
    std::vector<uint32_t> dm(ctx->n_tiles_cap);
    if ((e = cudaMemcpyAsync(g.data(), S.tile_g, g.size(), cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
    if ((e = cudaMemcpyAsync(dm.data(), S.tile_dm, sizeof(uint32_t) * dm.size(), cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess) break;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
    S.unit_base.assign(ctx->n_tiles_cap + 1, 0);
    std::vector<int> units;
    for (int t = 0; t < ctx->n_tiles_cap; ++t) {
      S.unit_base[t + 1] = S.unit_base[t] + g[t];
      const int lg = __builtin_ctz((unsigned)g[t]);
      const int d15 = std::min<int>((dm[t] + g[t] - 1) / g[t], 15);  // slots per lane
      for (int p = 0; p < g[t]; ++p) units.push_back(t << 12 | p << 7 | d15 << 3 | lg);
    }
    S.unit_words = units;
    S.unit_cost.resize(units.size());
    for (size_t u = 0; u < units.size(); ++u) {
      const int t = units[u] >> 12, G = 1 << (units[u] & 7);
      S.unit_cost[u] = (dm[t] + G - 1) / G;  // slots per lane
    }
    S.sched_grid = 0;
    S.sched_u1 = -1;
    S.n_units = (int)units.size();
    if (S.units) dfree(ctx, S.units);
    S.units = nullptr;
    if ((e = dalloc(ctx, &S.units, sizeof(int) * units.size())) != cudaSuccess) break;
    if ((e = cudaMemcpyAsync(S.units, units.data(), sizeof(int) * units.size(), cudaMemcpyHostToDevice, st)) !=
        cudaSuccess) break;
    if (S.d_unit_base == nullptr &&
        (e = dalloc(ctx, &S.d_unit_base, sizeof(int) * (ctx->n_tiles_cap + 1))) != cudaSuccess) break;
    if ((e = cudaMemcpyAsync(S.d_unit_base, S.unit_base.data(), sizeof(int) * (ctx->n_tiles_cap + 1),
                             cudaMemcpyHostToDevice, st)) != cudaSuccess) break;
    e = cudaStreamSynchronize(st);
  } while (0);
  dfree(ctx, keys); dfree(ctx, keys2); dfree(ctx, vals); dfree(ctx, vals2); dfree(ctx, rp_old); dfree(ctx, deg);
  dfree(ctx, bad); dfree(ctx, tmp);
  if (rc != IVHD_OK) return rc;
  if (e != cudaSuccess) return fail(ctx, IVHD_ERR_CUDA, "CSR build: %s", cudaGetErrorString(e));
  if (hbad) return fail(ctx, IVHD_ERR_INVALID_ARG, "connection endpoint outside [0, %lld)", (long long)m);
  S.valid = true;
  ctx->masks_stale = true;  // peer mode: halo masks follow the connection sets
  return IVHD_OK;
}

// ---------------------------------------------------------- launch helpers

// Cost-balanced static schedule for the fused loop: longest-processing-time
// greedy over the modelled unit costs (slot rounds per lane + a fixed
// per-unit overhead), ties to the lowest block; each block then runs its
// units heavy first.  Deterministic for a given graph and grid, so the
// per-thread partial sums keep a fixed order.
// Units [u0, u1) (a sharded rank's range; the whole graph by default).
int build_schedule(ivhd_ctx* ctx, CsrSlot& S, int grid, int u0 = 0, int u1 = -1) {
  if (u1 < 0) u1 = S.n_units;
  if (S.sched_grid == grid && S.sched_u0 == u0 && S.sched_u1 == u1) return IVHD_OK;
  constexpr int c0 = 3;  // modelled fixed cost of a unit, in slot rounds (profiles/r01_c0_sweep.txt)
  const int n = u1 - u0;
  std::vector<std::vector<int>> per(grid);
  if (ctx->window_order) {
    // id-local input: contiguous unit ranges of equal modelled cost, so one
    // block sweeps a window's tiles back to back and its nn partners are
    // still in L2 (and L1) when the neighbouring tiles gather them
    int64_t total = 0, acc = 0;
    for (int u = u0; u < u1; ++u) total += S.unit_cost[u] + c0;
    int b = 0;
    for (int u = u0; u < u1; ++u) {
      per[b].push_back(u);
      acc += S.unit_cost[u] + c0;
      while (b < grid - 1 && acc * grid >= (int64_t)(b + 1) * total) ++b;
    }
  } else {
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = u0 + i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return S.unit_cost[a] > S.unit_cost[b]; });
    std::vector<std::pair<int64_t, int>> heap;  // (load, block), min-heap
    for (int b = 0; b < grid; ++b) heap.push_back({0, b});
    auto cmp = [](const std::pair<int64_t, int>& x, const std::pair<int64_t, int>& y) { return x > y; };
    std::make_heap(heap.begin(), heap.end(), cmp);
    for (int u : order) {
      std::pop_heap(heap.begin(), heap.end(), cmp);
      auto& top = heap.back();
      per[top.second].push_back(u);
      top.first += S.unit_cost[u] + c0;
      std::push_heap(heap.begin(), heap.end(), cmp);
    }
  }
  std::vector<int> words, off(grid + 1, 0);
  words.reserve(n);
  for (int b = 0; b < grid; ++b) {
    for (int u : per[b]) words.push_back(S.unit_words[u]);
    off[b + 1] = (int)words.size();
  }
  drop_graphs(ctx);  // captured launches hold the old schedule pointers
  dfree(ctx, S.sched_units);
  dfree(ctx, S.sched_off);
  S.sched_units = nullptr;
  S.sched_off = nullptr;
  S.sched_grid = 0;
  CU(ctx, dalloc(ctx, &S.sched_units, sizeof(int) * std::max(n, 1)));
  CU(ctx, dalloc(ctx, &S.sched_off, sizeof(int) * (grid + 1)));
  CU(ctx, cudaMemcpyAsync(S.sched_units, words.data(), sizeof(int) * n, cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, cudaMemcpyAsync(S.sched_off, off.data(), sizeof(int) * (grid + 1), cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));  // host vectors go out of scope
  S.sched_grid = grid;
  S.sched_u0 = u0;
  S.sched_u1 = u1;
  return IVHD_OK;
}

StepArgs make_args(ivhd_ctx* ctx, int slot, int norm, int fuse) {
  const CsrSlot& S = ctx->slots[slot];
  StepArgs A{};
  A.row_ptr = S.row_ptr;
  A.col = S.col;
  A.ew = S.ew;
  A.ybuf0 = ctx->ybuf[0];
  A.ybuf1 = ctx->ybuf[1];
  A.state = ctx->state;
  A.sstride = state_stride(ctx);
  {  // streamed graph bytes + positions + state per iteration vs the L2 size
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device);
    const int64_t ws = 4 * S.n + 4 * ctx->m + (int64_t)4 * ctx->m * (2 * ys_now(ctx) + ss_now(ctx));
    A.stream_hint = ws > (int64_t)l2 ? 1 : 0;
  }
  A.dg_key = ctx->dg_key;
  A.dg_vec = ctx->dg_vec;
  A.miss_n = ctx->miss_n;
  A.miss = ctx->miss;
  A.miss_cap = ctx->miss_cap;
  A.partial = ctx->partial;
  A.tpart = ctx->tpart;
  A.unit_base = S.d_unit_base;
  A.bpart = ctx->bpart;
  A.trace = ctx->trace;
  A.ctrl = ctx->ctrl;
  A.force_out = nullptr;
  A.tile_g = S.tile_g;
  A.units = S.units;
  A.tile_v = ctx->tile_v;
  A.norm = norm;
  A.fuse_finalize = fuse;
  A.h = ctx->hyper;
  A.v_begin = 0;
  A.v_end = ctx->m;
  if (ctx->sharded) {
    // every unit up to the padded tile count is written by some rank (pad
    // tiles hold zeros), so all ranks reduce the same array in the same order
    const int t0 = (int)(ctx->shard_begin / ctx->tile_v), t1 = (int)(ctx->shard_end / ctx->tile_v);
    A.tile0 = S.unit_base[t0];
    A.n_tiles = S.unit_base[t1] - S.unit_base[t0];
    A.n_tiles_global = ctx->n_tiles_cap;  // the finalizer reduces the exchanged tile partials
    A.v_begin = ctx->shard_begin;
    A.v_end = std::min<int64_t>(ctx->shard_end, ctx->m);
    if (ctx->peer_on) A.pe = ctx->pe;
  } else {
    A.tile0 = 0;
    A.n_tiles = S.unit_base[ctx->n_tiles];
    A.n_tiles_global = A.n_tiles;
  }
  return A;
}

// The peer finalizer, also programmatically dependent: it becomes resident
// while the step drains and waits (griddepcontrol.wait) for it.
int launch_finalize_peer(ivhd_ctx* ctx, const StepArgs& A) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CU(ctx, cudaLaunchKernelEx(&cfg, pick_finalize_peer(ctx->opt.kind), A));
  return IVHD_OK;
}

// Deferred decisions: decide the last launch's iteration at the end of a run
// segment (the launches of the segment each decided their predecessor's).
template <int OPT>
__global__ void k_defer_finalize(StepArgs A) {
  Ctrl* c = A.ctrl;
  if (!c->pend || threadIdx.x != 0) return;
  DState d = dstate_load(c);
  const long long it = d.iter;
  double2 tr;
  if (d.status == 0 && decide_core<OPT>(A, fix_read(c, c->pslot), c->needw[c->pslot], d, tr) && A.trace)
    A.trace[it] = tr;
  dstate_store(c, d);
  c->needw[c->pslot] = 0;
  c->fnf[c->pslot] = 0;
  for (int q = 0; q < 4; ++q) c->facc[c->pslot][q] = 0ull;
  c->pend = 0;
  c->readers = 0;
  c->next_tile = 0;
  c->arrive = 0;
}

int launch_step(ivhd_ctx* ctx, KernelInfo k, const StepArgs& A) {
  const int grid = std::max(1, std::min(A.n_tiles, occupancy(ctx, k) * ctx->sm_count));
  // Programmatic dependent launch: this grid may become resident while the
  // previous iteration drains; it prefetches graph constants and then waits
  // (griddepcontrol.wait) before reading positions, state or ctrl.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(k.threads);
  cfg.dynamicSmemBytes = k.smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CU(ctx, cudaLaunchKernelEx(&cfg, k.fn, A));
  return IVHD_OK;
}

int check_ready(ivhd_ctx* ctx, int slot) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  if (slot < 0 || slot > 1) return fail(ctx, IVHD_ERR_INVALID_ARG, "slot must be 0 or 1");
  if (!ctx->slots[slot].valid) return fail(ctx, IVHD_ERR_STATE, "connection slot %d not set", slot);
  CU(ctx, cudaSetDevice(ctx->device));
  return IVHD_OK;
}

int push_ctrl(ivhd_ctx* ctx) {
  CU(ctx, cudaMemcpyAsync(ctx->ctrl, ctx->ctrl_h, sizeof(Ctrl), cudaMemcpyHostToDevice, ctx->stream));
  return IVHD_OK;
}

int pull_ctrl(ivhd_ctx* ctx) {
  CU(ctx, cudaMemcpyAsync(ctx->ctrl_h, ctx->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  return IVHD_OK;
}

int upload_stage(ivhd_ctx* ctx, const double* host, int64_t count) {
  CU(ctx, cudaMemcpyAsync(ctx->stage, host, sizeof(double) * count, cudaMemcpyHostToDevice, ctx->stream));
  return IVHD_OK;
}

int vel_stride(int dim) { return dim == 2 ? 2 : 4; }

// Optimizer-state buffer b (0/1); ctrl.scur names the current one.  Only the
// fp64 Adam kernel double-buffers (stride > 0); the fp32 kernels update in
// place (stride 0: both indices name buffer 0) — a paused iteration's state is
// recovered by inverting the update instead (resume_degenerate).
int64_t state_stride(ivhd_ctx* ctx) { return f64_of(ctx->opt.kind) ? (int64_t)ctx->state_fpv * ctx->v_cap : 0; }
float* state_buf(ivhd_ctx* ctx, int b) { return ctx->state + (size_t)b * state_stride(ctx); }

int ys_now(ivhd_ctx* ctx) { return ys_of(ctx->dim, ctx->opt.kind); }

int ss_now(ivhd_ctx* ctx) {
  const int k = ctx->opt.kind;
  if (k == OPT_ADAM) return ctx->dim == 2 ? 8 : 16;  // fp64 {v, s}
  const int nv = (k == OPT_FD || k == OPT_MOM || k == OPT_NEST) ? 1 : (k == OPT_ADADELTA) ? 2 : 0;
  return nv == 0 ? 0 : (ctx->dim == 2 ? 2 * nv : 4 * nv);
}


}  // namespace


// ======================================================================= C ABI

extern "C" {

int ivhd_abi_version(void) { return IVHD_ABI_VERSION; }

const char* ivhd_global_error(void) { return g_error.c_str(); }

const char* ivhd_last_error(const ivhd_ctx* ctx) { return ctx ? ctx->err.c_str() : g_error.c_str(); }

int ivhd_host_alloc(int device, uint64_t bytes, void** out) {
  if (!out || !bytes) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null output or zero size");
  *out = nullptr;
  CU(nullptr, cudaSetDevice(device));
  CU(nullptr, cudaHostAlloc(out, bytes, cudaHostAllocPortable));
  return IVHD_OK;
}

int ivhd_host_free(void* p) {
  if (p) CU(nullptr, cudaFreeHost(p));
  return IVHD_OK;
}

int ivhd_create(ivhd_ctx** out, int device, int64_t m, int dim, uint64_t stream) {
  if (!out) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null output pointer");
  *out = nullptr;
  if (m < 1) return fail(nullptr, IVHD_ERR_INVALID_ARG, "need at least one point");
  if (m >= (int64_t)0x7fffffff) return fail(nullptr, IVHD_ERR_INVALID_ARG, "M too large for 31-bit ids");
  if (dim != 2 && dim != 3) return fail(nullptr, IVHD_ERR_INVALID_ARG, "target_dim must be 2 or 3");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(nullptr, IVHD_ERR_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(nullptr, IVHD_ERR_INVALID_ARG, "bad device %d", device);
  ivhd_ctx* ctx = new ivhd_ctx();
  ctx->device = device;
  ctx->m = m;
  ctx->dim = dim;
  auto bail = [&](int code) {
    g_error = ctx->err;
    ivhd_destroy(ctx);
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) return bail(fail(ctx, IVHD_ERR_CUDA, "cudaSetDevice failed"));
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  {  // keep freed stream-ordered memory pooled across contexts (repeated embeds)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  if (stream) {
    ctx->stream = reinterpret_cast<cudaStream_t>(stream);
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess)
      return bail(fail(ctx, IVHD_ERR_CUDA, "stream create failed"));
    ctx->own_stream = true;
  }
  // Fixed tile size: the reduction order is the same for any grid size and
  // any number of ranks.
  const int64_t tv = kBlock;
  ctx->tile_v = (int)tv;
  ctx->n_tiles = (int)((m + tv - 1) / tv);
  ctx->n_tiles_cap = (ctx->n_tiles + 7) / 8 * 8;
  ctx->v_cap = (int64_t)ctx->n_tiles_cap * tv;
  const int64_t vc = ctx->v_cap;
  int rc = IVHD_OK;
  auto alloc = [&](void** p, size_t bytes) {
    if (rc != IVHD_OK) return;
    cudaError_t ee = cudaMallocAsync(p, bytes, ctx->stream);
    if (ee != cudaSuccess) rc = fail(ctx, IVHD_ERR_CUDA, "cudaMallocAsync(%zu): %s", bytes, cudaGetErrorString(ee));
    else cudaMemsetAsync(*p, 0, bytes, ctx->stream);
  };
  alloc((void**)&ctx->ybuf[0], sizeof(float) * 8 * vc);
  alloc((void**)&ctx->ybuf[1], sizeof(float) * 8 * vc);
  alloc((void**)&ctx->state, sizeof(float) * 2 * 8 * vc);
  alloc((void**)&ctx->miss_n, sizeof(int));
  alloc((void**)&ctx->miss, sizeof(int2) * ctx->miss_cap);
  alloc((void**)&ctx->partial, sizeof(double4) * 32 * ctx->n_tiles_cap);  // <= 32 units per tile
  alloc((void**)&ctx->tpart, sizeof(double4) * ctx->n_tiles_cap);
  alloc((void**)&ctx->bpart, sizeof(double4) * 8 * ctx->sm_count);  // <= 2048/288 blocks per SM
  alloc((void**)&ctx->ctrl, sizeof(Ctrl));
  alloc((void**)&ctx->opctrl, sizeof(Ctrl));
  alloc((void**)&ctx->red_out, sizeof(double4));
  alloc((void**)&ctx->stage, sizeof(double) * 4 * vc);
  alloc((void**)&ctx->perm, sizeof(int32_t) * vc);
  alloc((void**)&ctx->inv, sizeof(int32_t) * vc);
  if (rc != IVHD_OK) return bail(rc);
  k_iota<<<grid_for(vc, ctx->sm_count), 256, 0, ctx->stream>>>(ctx->perm, vc);  // identity until the first CSR
  k_iota<<<grid_for(vc, ctx->sm_count), 256, 0, ctx->stream>>>(ctx->inv, vc);
  cudaStreamSynchronize(ctx->stream);
  if ((ctx->ctrl_h = pinned_ctrl_get()) == nullptr)
    return bail(fail(ctx, IVHD_ERR_CUDA, "pinned alloc failed"));
  memset(ctx->ctrl_h, 0, sizeof(Ctrl));
  ctx->ctrl_h->c = 0.1;
  ctx->ctrl_h->step = 0.002;
  cudaMemcpy(ctx->ctrl, ctx->ctrl_h, sizeof(Ctrl), cudaMemcpyHostToDevice);
  // default optimizer: force-directed with the reference defaults (optim.py:24-29)
  ivhd_optimizer_params p{};
  p.kind = IVHD_OPT_FORCE_DIRECTED;
  p.auto_adapt = 1;
  p.step = 0.002;
  p.a = 0.99;
  p.tau = 1e-3 * (double)m;
  p.gamma1 = 1.1;
  p.gamma2 = 0.9;
  p.beta = 0.9;
  p.gamma_v = 0.9;
  p.gamma_s = 0.999;
  p.rho = 0.95;
  p.eps = 1e-8;
  if ((rc = ivhd_set_optimizer(ctx, &p)) != IVHD_OK) return bail(rc);
  *out = ctx;
  return IVHD_OK;
}

int ivhd_destroy(ivhd_ctx* ctx) {
  if (!ctx) return IVHD_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  drop_graphs(ctx);
  for (auto& s : ctx->slots) {
    dfree(ctx, s.row_ptr); dfree(ctx, s.col); dfree(ctx, s.ew); dfree(ctx, s.tile_g); dfree(ctx, s.tile_dm); dfree(ctx, s.units);
    dfree(ctx, s.sched_units); dfree(ctx, s.sched_off); dfree(ctx, s.d_unit_base);
  }
  dfree(ctx, ctx->perm); dfree(ctx, ctx->inv);
  for (void* p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
  if (ctx->ybuf_malloc) {
    cudaFree(ctx->ybuf[0]);
    cudaFree(ctx->ybuf[1]);
    ctx->ybuf[0] = ctx->ybuf[1] = nullptr;
  }
  if (ctx->tp2) cudaFree(ctx->tp2);
  dfree(ctx, ctx->hmask);
  if (ctx->flags) cudaFree(ctx->flags);
  if (ctx->stamp) cudaFree(ctx->stamp);
  dfree(ctx, ctx->ybuf[0]); dfree(ctx, ctx->ybuf[1]); dfree(ctx, ctx->state); dfree(ctx, ctx->partial); dfree(ctx, ctx->tpart); dfree(ctx, ctx->bpart);
  dfree(ctx, ctx->trace); dfree(ctx, ctx->ctrl); dfree(ctx, ctx->opctrl); dfree(ctx, ctx->red_out);
  dfree(ctx, ctx->stage); dfree(ctx, ctx->op_y); dfree(ctx, ctx->op_force);
  dfree(ctx, ctx->snap_y); dfree(ctx, ctx->snap_state);
  dfree(ctx, ctx->dg_key); dfree(ctx, ctx->dg_vec); dfree(ctx, ctx->miss_n); dfree(ctx, ctx->miss);
  if (ctx->ctrl_h) pinned_ctrl_put(ctx->ctrl_h);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return IVHD_OK;
}

// binary connection set from device-resident nn ids [m, nn_stride] and random
// partners [m, rn] (engine.py:165-221 with distance_mode == "binary")
static int graph_from_device(ivhd_ctx* ctx, int slot, const int32_t* d_nn, int64_t nn_stride, int ncols,
                             const int32_t* d_rn, int rn) {
  const int64_t m = ctx->m, n_nn = m * ncols, L = n_nn + m * rn;
  int32_t *d_src = nullptr, *d_dst = nullptr;
  cudaError_t e = cudaSuccess;
  do {
    if ((e = dalloc(ctx, &d_src, sizeof(int32_t) * std::max<int64_t>(L, 1))) != cudaSuccess) break;
    if ((e = dalloc(ctx, &d_dst, sizeof(int32_t) * std::max<int64_t>(L, 1))) != cudaSuccess) break;
    if (L > 0)
      k_binary_edges<<<grid_for(L, ctx->sm_count), 256, 0, ctx->stream>>>(d_nn, nn_stride, ncols, d_rn, rn,
                                                                          m, d_src, d_dst);
    e = cudaGetLastError();
  } while (0);
  int rc = IVHD_OK;
  if (e != cudaSuccess) rc = fail(ctx, IVHD_ERR_CUDA, "set_graph: %s", cudaGetErrorString(e));
  else rc = build_csr(ctx, slot, d_src, d_dst, nullptr, n_nn, nullptr, nullptr, L);
  dfree(ctx, d_src); dfree(ctx, d_dst);
  return rc;
}

int ivhd_set_graph(ivhd_ctx* ctx, int slot, const int32_t* nn_ids, int64_t nn_stride, int ncols,
                   const int32_t* rn_ids, int rn) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  if (slot < 0 || slot > 1) return fail(ctx, IVHD_ERR_INVALID_ARG, "slot must be 0 or 1");
  if (ncols < 0 || rn < 0 || nn_stride < ncols || (ncols > 0 && !nn_ids) || (rn > 0 && !rn_ids))
    return fail(ctx, IVHD_ERR_INVALID_ARG, "bad graph arguments");
  CU(ctx, cudaSetDevice(ctx->device));
  const int64_t m = ctx->m;
  int32_t *d_nn = nullptr, *d_rn = nullptr;
  cudaError_t e = cudaSuccess;
  do {
    if (ncols > 0) {
      if ((e = dalloc(ctx, &d_nn, sizeof(int32_t) * m * nn_stride)) != cudaSuccess) break;
      if ((e = cudaMemcpyAsync(d_nn, nn_ids, sizeof(int32_t) * m * nn_stride, cudaMemcpyHostToDevice,
                               ctx->stream)) != cudaSuccess) break;
    }
    if (rn > 0) {
      if ((e = dalloc(ctx, &d_rn, sizeof(int32_t) * m * rn)) != cudaSuccess) break;
      if ((e = cudaMemcpyAsync(d_rn, rn_ids, sizeof(int32_t) * m * rn, cudaMemcpyHostToDevice,
                               ctx->stream)) != cudaSuccess) break;
    }
  } while (0);
  int rc = IVHD_OK;
  if (e != cudaSuccess) rc = fail(ctx, IVHD_ERR_CUDA, "set_graph upload: %s", cudaGetErrorString(e));
  else rc = graph_from_device(ctx, slot, d_nn, nn_stride, ncols, d_rn, rn);
  dfree(ctx, d_nn); dfree(ctx, d_rn);
  return rc;
}

// ------------------------------------------------------ device RNG (PCG64)

__global__ void k_accept_scatter(const int32_t* __restrict__ val, const int32_t* __restrict__ ok,
                                 const int32_t* __restrict__ pos, int64_t n_cand, int64_t N, int32_t* __restrict__ picks,
                                 int64_t* __restrict__ last_q) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_cand; q += (int64_t)gridDim.x * blockDim.x) {
    if (!ok[q]) continue;
    const int64_t r = pos[q];  // inclusive rank among accepted draws
    if (r <= N) picks[r - 1] = val[q];
    if (r == N) *last_q = q;
  }
}

__global__ void k_flag_to_index(const int32_t* __restrict__ flag, const int32_t* __restrict__ pos, int64_t n,
                                int64_t* __restrict__ idx) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    if (flag[k]) idx[pos[k] - 1] = k;
}

__global__ void k_u8_to_i32(const uint8_t* __restrict__ a, int64_t n, int32_t* __restrict__ b) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    b[k] = a[k];
}

__global__ void k_scatter_i32(const int64_t* __restrict__ idx, const int32_t* __restrict__ v, int64_t n,
                              int32_t* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    out[idx[k]] = v[k];
}

// inclusive prefix sum of int32 flags (n < 2^31)
static cudaError_t scan_flags(ivhd_ctx* ctx, const int32_t* in, int32_t* out, int64_t n) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::InclusiveSum(nullptr, tb, in, out, (int)n, ctx->stream);
  if (e != cudaSuccess) return e;
  void* tmp = nullptr;
  if ((e = dalloc(ctx, &tmp, std::max<size_t>(tb, 16))) != cudaSuccess) return e;
  e = cub::DeviceScan::InclusiveSum(tmp, tb, in, out, (int)n, ctx->stream);
  dfree(ctx, tmp);
  return e;
}

int ivhd_init_positions(ivhd_ctx* ctx, uint64_t* rng, double lo, double hi) {
  if (!ctx || !rng) return fail(ctx, IVHD_ERR_INVALID_ARG, "null argument");
  CU(ctx, cudaSetDevice(ctx->device));
  TRY(pull_ctrl(ctx));
  pcg::State st = pcg::load(rng);
  const int64_t n = ctx->m * ctx->dim;
  const int64_t chunks = (n + pcg::kChunk - 1) / pcg::kChunk;
  pcg::k_uniform<<<grid_for(chunks, ctx->sm_count), 256, 0, ctx->stream>>>(
      rng[0], rng[1], rng[2], rng[3], n, lo, hi - lo, ctx->stage);
  CU(ctx, cudaGetLastError());
  const int ys = ys_of(ctx->dim, ctx->opt.kind);
  const bool nest = ctx->opt.kind == IVHD_OPT_NESTEROV;
  k_pack_positions<<<grid_for(ctx->m, ctx->sm_count), 256, 0, ctx->stream>>>(
      ctx->stage, ctx->m, ctx->dim, ys, ctx->perm, nest ? state_buf(ctx, ctx->ctrl_h->scur) : nullptr,
      vel_stride(ctx->dim), (float)ctx->hyper.beta, ctx->ybuf[ctx->ctrl_h->cur], f64_of(ctx->opt.kind));
  CU(ctx, cudaGetLastError());
  ctx->ctrl_h->status = 0;
  ctx->ctrl_h->last_commit = 0;
  TRY(push_ctrl(ctx));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->pos_set = true;
  st.s = pcg::advance(st.s, st.inc, (uint64_t)n);  // uniform() leaves the buffered half alone
  pcg::store(st, rng);
  return IVHD_OK;
}

int ivhd_set_graph_sampled(ivhd_ctx* ctx, int slot, const int32_t* nn_ids, int64_t nn_stride, int ncols, int rn,
                           uint64_t* rng, int32_t* picks_out) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  if (slot < 0 || slot > 1) return fail(ctx, IVHD_ERR_INVALID_ARG, "slot must be 0 or 1");
  if (!rng || ncols < 0 || rn < 0 || nn_stride < ncols || (ncols > 0 && !nn_ids))
    return fail(ctx, IVHD_ERR_INVALID_ARG, "bad graph arguments");
  const int64_t m = ctx->m, N = m * rn;
  if (m <= (int64_t)ncols + rn)
    return fail(ctx, IVHD_ERR_INVALID_ARG, "M=%lld too small for nn=%d plus rn=%d", (long long)m, ncols, rn);
  CU(ctx, cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  pcg::State gs = pcg::load(rng);
  const uint32_t mu = (uint32_t)m;
  const uint32_t thr = (uint32_t)(((1ull << 32) - (uint64_t)m) % (uint64_t)m);
  int32_t *d_nn = nullptr, *d_rn = nullptr, *val = nullptr, *ok = nullptr, *pos = nullptr;
  uint8_t* ok8 = nullptr;
  int64_t *d_last = nullptr, *d_idx = nullptr;
  cudaError_t e = cudaSuccess;
  int rc = IVHD_OK;
  do {
    if (ncols > 0) {
      if ((e = dalloc(ctx, &d_nn, sizeof(int32_t) * m * nn_stride)) != cudaSuccess) break;
      if ((e = cudaMemcpyAsync(d_nn, nn_ids, sizeof(int32_t) * m * nn_stride, cudaMemcpyHostToDevice, st)) !=
          cudaSuccess) break;
    }
    if (N == 0) break;
    if ((e = dalloc(ctx, &d_rn, sizeof(int32_t) * N)) != cudaSuccess) break;
    if ((e = dalloc(ctx, &d_last, sizeof(int64_t))) != cudaSuccess) break;
    // first batch: the first N accepted Lemire draws of the stream
    int64_t n_cand = N + N / 32 + 1024, consumed = 0;
    for (;;) {
      if (n_cand >= (1ll << 31)) { e = cudaErrorInvalidValue; break; }
      dfree(ctx, val); dfree(ctx, ok8); dfree(ctx, ok); dfree(ctx, pos);
      val = nullptr; ok8 = nullptr; ok = nullptr; pos = nullptr;
      if ((e = dalloc(ctx, &val, sizeof(int32_t) * n_cand)) != cudaSuccess) break;
      if ((e = dalloc(ctx, &ok8, n_cand)) != cudaSuccess) break;
      if ((e = dalloc(ctx, &ok, sizeof(int32_t) * n_cand)) != cudaSuccess) break;
      if ((e = dalloc(ctx, &pos, sizeof(int32_t) * n_cand)) != cudaSuccess) break;
      const int64_t outs = (n_cand + 1) / 2 + 1;
      pcg::k_lemire_candidates<<<grid_for((outs + pcg::kChunk - 1) / pcg::kChunk, ctx->sm_count), 256, 0, st>>>(
          rng[0], rng[1], rng[2], rng[3], gs.has, gs.ub, n_cand, mu, thr, val, ok8);
      k_u8_to_i32<<<grid_for(n_cand, ctx->sm_count), 256, 0, st>>>(ok8, n_cand, ok);
      if ((e = scan_flags(ctx, ok, pos, n_cand)) != cudaSuccess) break;
      int32_t got = 0;
      if ((e = cudaMemcpyAsync(&got, pos + n_cand - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        break;
      if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
      if (got >= N) {
        k_accept_scatter<<<grid_for(n_cand, ctx->sm_count), 256, 0, st>>>(val, ok, pos, n_cand, N, d_rn, d_last);
        int64_t last = 0;
        if ((e = cudaMemcpyAsync(&last, d_last, sizeof(int64_t), cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
        consumed = last + 1;
        break;
      }
      n_cand *= 2;
    }
    if (e != cudaSuccess) break;
    // generator state after `consumed` 32-bit draws
    {
      const int64_t c64 = consumed - (gs.has ? 1 : 0);  // draws taken from fresh 64-bit outputs
      const int64_t outs = (c64 + 1) / 2;
      gs.s = pcg::advance(gs.s, gs.inc, (uint64_t)outs);
      gs.has = (int)(c64 & 1);
      if (outs > 0) gs.ub = (uint32_t)(pcg::output(gs.s) >> 32);  // last high half drawn
    }
    // picks that hit their own row or an nn id are re-drawn in row-major order
    // from the continued stream until none is left (engine.py:141-146)
    {
      uint8_t* bad8 = ok8;  // reuse (n_cand >= N)
      pcg::k_pick_collisions<<<grid_for(N, ctx->sm_count), 256, 0, st>>>(d_rn, m, rn, d_nn, nn_stride, ncols, bad8);
      k_u8_to_i32<<<grid_for(N, ctx->sm_count), 256, 0, st>>>(bad8, N, ok);
      if ((e = scan_flags(ctx, ok, pos, N)) != cudaSuccess) break;
      int32_t n_bad = 0;
      if ((e = cudaMemcpyAsync(&n_bad, pos + N - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        break;
      if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
      if (n_bad > 0) {
        if ((e = dalloc(ctx, &d_idx, sizeof(int64_t) * n_bad)) != cudaSuccess) break;
        k_flag_to_index<<<grid_for(N, ctx->sm_count), 256, 0, st>>>(ok, pos, N, d_idx);
        std::vector<int64_t> idx(n_bad);
        if ((e = cudaMemcpyAsync(idx.data(), d_idx, sizeof(int64_t) * n_bad, cudaMemcpyDeviceToHost, st)) !=
            cudaSuccess) break;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
        std::vector<int64_t> fix_idx;
        std::vector<int32_t> fix_val;
        std::vector<int64_t> cur = idx;
        while (!cur.empty()) {
          std::vector<int64_t> next;
          for (int64_t k : cur) {
            const int32_t v = (int32_t)pcg::bounded(gs, mu, thr);
            const int64_t row = k / rn;
            bool b = v == (int32_t)row;
            for (int c = 0; c < ncols; ++c) b |= v == nn_ids[row * nn_stride + c];
            fix_idx.push_back(k);
            fix_val.push_back(v);
            if (b) next.push_back(k);
          }
          cur.swap(next);
        }
        // later writes win: apply in order
        int64_t* d_fi = nullptr;
        int32_t* d_fv = nullptr;
        const int64_t nf = (int64_t)fix_idx.size();
        if ((e = dalloc(ctx, &d_fi, sizeof(int64_t) * nf)) != cudaSuccess) break;
        if ((e = dalloc(ctx, &d_fv, sizeof(int32_t) * nf)) != cudaSuccess) { dfree(ctx, d_fi); break; }
        e = cudaMemcpyAsync(d_fi, fix_idx.data(), sizeof(int64_t) * nf, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(d_fv, fix_val.data(), sizeof(int32_t) * nf, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) {
          k_scatter_i32<<<1, 1, 0, st>>>(d_fi, d_fv, nf, d_rn);  // one thread: sequential, last write wins
          e = cudaStreamSynchronize(st);  // host vectors die at scope end
        }
        dfree(ctx, d_fi); dfree(ctx, d_fv);
        if (e != cudaSuccess) break;
      }
    }
    if (picks_out) {
      if ((e = cudaMemcpyAsync(picks_out, d_rn, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        break;
    }
    e = cudaGetLastError();
  } while (0);
  if (e != cudaSuccess) rc = fail(ctx, IVHD_ERR_CUDA, "random-neighbor sampling: %s", cudaGetErrorString(e));
  else rc = graph_from_device(ctx, slot, d_nn, nn_stride, ncols, d_rn, rn);
  if (rc == IVHD_OK && picks_out) {
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (e2 != cudaSuccess) rc = fail(ctx, IVHD_ERR_CUDA, "random-neighbor sampling: %s", cudaGetErrorString(e2));
  }
  if (rc == IVHD_OK) pcg::store(gs, rng);
  dfree(ctx, d_nn); dfree(ctx, d_rn); dfree(ctx, val); dfree(ctx, ok8); dfree(ctx, ok); dfree(ctx, pos);
  dfree(ctx, d_last); dfree(ctx, d_idx);
  return rc;
}

int ivhd_set_connections(ivhd_ctx* ctx, int slot, const int32_t* edges, const uint8_t* is_random,
                         const double* targets, const double* scale, int64_t n_conn) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  if (slot < 0 || slot > 1) return fail(ctx, IVHD_ERR_INVALID_ARG, "slot must be 0 or 1");
  if (n_conn < 0 || (n_conn > 0 && (!edges || !is_random)))
    return fail(ctx, IVHD_ERR_INVALID_ARG, "bad connection arguments");
  CU(ctx, cudaSetDevice(ctx->device));
  const int64_t L = n_conn, Lc = std::max<int64_t>(L, 1);
  int32_t *d_e = nullptr, *d_src = nullptr, *d_dst = nullptr;
  uint8_t* d_r = nullptr;
  double* d_tmp = nullptr;
  float *d_t = nullptr, *d_s = nullptr;
  cudaError_t e = cudaSuccess;
  cudaStream_t st = ctx->stream;
  do {
    if ((e = dalloc(ctx, &d_e, sizeof(int32_t) * 2 * Lc)) != cudaSuccess) break;
    if ((e = dalloc(ctx, &d_src, sizeof(int32_t) * Lc)) != cudaSuccess) break;
    if ((e = dalloc(ctx, &d_dst, sizeof(int32_t) * Lc)) != cudaSuccess) break;
    if ((e = dalloc(ctx, &d_r, Lc)) != cudaSuccess) break;
    if (L > 0) {
      if ((e = cudaMemcpyAsync(d_e, edges, sizeof(int32_t) * 2 * L, cudaMemcpyHostToDevice, st)) != cudaSuccess) break;
      if ((e = cudaMemcpyAsync(d_r, is_random, L, cudaMemcpyHostToDevice, st)) != cudaSuccess) break;
      k_split_edges<<<grid_for(L, ctx->sm_count), 256, 0, st>>>(d_e, L, d_src, d_dst);
    }
    if (targets || scale) {
      if ((e = dalloc(ctx, &d_tmp, sizeof(double) * Lc)) != cudaSuccess) break;
    }
    if (targets) {
      if ((e = dalloc(ctx, &d_t, sizeof(float) * Lc)) != cudaSuccess) break;
      if (L > 0) {
        if ((e = cudaMemcpyAsync(d_tmp, targets, sizeof(double) * L, cudaMemcpyHostToDevice, st)) != cudaSuccess) break;
        k_d2f<<<grid_for(L, ctx->sm_count), 256, 0, st>>>(d_tmp, d_t, L);
      }
    }
    if (scale) {
      if ((e = dalloc(ctx, &d_s, sizeof(float) * Lc)) != cudaSuccess) break;
      if (L > 0) {
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;  // d_tmp reuse
        if ((e = cudaMemcpyAsync(d_tmp, scale, sizeof(double) * L, cudaMemcpyHostToDevice, st)) != cudaSuccess) break;
        k_d2f<<<grid_for(L, ctx->sm_count), 256, 0, st>>>(d_tmp, d_s, L);
      }
    }
    e = cudaGetLastError();
  } while (0);
  int rc = IVHD_OK;
  if (e != cudaSuccess) rc = fail(ctx, IVHD_ERR_CUDA, "set_connections: %s", cudaGetErrorString(e));
  else rc = build_csr(ctx, slot, d_src, d_dst, d_r, 0, d_t, d_s, L);
  dfree(ctx, d_e); dfree(ctx, d_src); dfree(ctx, d_dst); dfree(ctx, d_r); dfree(ctx, d_tmp); dfree(ctx, d_t); dfree(ctx, d_s);
  return rc;
}

int ivhd_set_positions(ivhd_ctx* ctx, const double* y) {
  if (!ctx || !y) return fail(ctx, IVHD_ERR_INVALID_ARG, "null argument");
  CU(ctx, cudaSetDevice(ctx->device));
  TRY(pull_ctrl(ctx));
  const int ys = ys_of(ctx->dim, ctx->opt.kind);
  TRY(upload_stage(ctx, y, ctx->m * ctx->dim));
  const bool nest = ctx->opt.kind == IVHD_OPT_NESTEROV;
  float* dst = ctx->ybuf[ctx->ctrl_h->cur];
  k_pack_positions<<<grid_for(ctx->m, ctx->sm_count), 256, 0, ctx->stream>>>(
      ctx->stage, ctx->m, ctx->dim, ys, ctx->perm, nest ? state_buf(ctx, ctx->ctrl_h->scur) : nullptr,
      vel_stride(ctx->dim), (float)ctx->hyper.beta, dst, f64_of(ctx->opt.kind));
  CU(ctx, cudaGetLastError());
  ctx->ctrl_h->status = 0;
  ctx->ctrl_h->last_commit = 0;
  TRY(push_ctrl(ctx));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->pos_set = true;
  return IVHD_OK;
}

int ivhd_get_positions(ivhd_ctx* ctx, double* y_out) {
  if (!ctx || !y_out) return fail(ctx, IVHD_ERR_INVALID_ARG, "null argument");
  CU(ctx, cudaSetDevice(ctx->device));
  TRY(pull_ctrl(ctx));
  const int ys = ys_of(ctx->dim, ctx->opt.kind);
  k_unpack_positions<<<grid_for(ctx->m, ctx->sm_count), 256, 0, ctx->stream>>>(
      ctx->ybuf[ctx->ctrl_h->cur], ctx->m, ctx->dim, ys, ctx->perm, ctx->stage, f64_of(ctx->opt.kind));
  CU(ctx, cudaGetLastError());
  CU(ctx, cudaMemcpyAsync(y_out, ctx->stage, sizeof(double) * ctx->m * ctx->dim, cudaMemcpyDeviceToHost,
                          ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  return IVHD_OK;
}

int ivhd_get_deltas(ivhd_ctx* ctx, double* d_out) {
  if (!ctx || !d_out) return fail(ctx, IVHD_ERR_INVALID_ARG, "null argument");
  CU(ctx, cudaSetDevice(ctx->device));
  TRY(pull_ctrl(ctx));
  const int ys = ys_of(ctx->dim, ctx->opt.kind);
  const int cur = ctx->ctrl_h->cur;
  k_deltas<<<grid_for(ctx->m, ctx->sm_count), 256, 0, ctx->stream>>>(
      ctx->ybuf[cur], ctx->ybuf[cur ^ 1], ctx->m, ctx->dim, ys, ctx->ctrl_h->last_commit, ctx->perm,
      ctx->stage, f64_of(ctx->opt.kind));
  CU(ctx, cudaGetLastError());
  CU(ctx, cudaMemcpyAsync(d_out, ctx->stage, sizeof(double) * ctx->m * ctx->dim, cudaMemcpyDeviceToHost,
                          ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  return IVHD_OK;
}

int ivhd_set_optimizer(ivhd_ctx* ctx, const ivhd_optimizer_params* p) {
  if (!ctx || !p) return fail(ctx, IVHD_ERR_INVALID_ARG, "null argument");
  if (p->kind < 0 || p->kind > 5) return fail(ctx, IVHD_ERR_INVALID_ARG, "unknown optimizer kind %d", p->kind);
  CU(ctx, cudaSetDevice(ctx->device));
  TRY(pull_ctrl(ctx));
  const int old_ys = ys_of(ctx->dim, ctx->opt.kind);
  const int new_ys = ys_of(ctx->dim, p->kind);
  const int old_f64 = f64_of(ctx->opt.kind), new_f64 = f64_of(p->kind);
  // fp64 Adam state in 3-D: 8 doubles per vertex (16 floats)
  const int need_fpv = (new_f64 && ctx->dim == 3) ? 16 : 8;
  if (need_fpv > ctx->state_fpv) {
    float* ns = nullptr;
    CU(ctx, dalloc(ctx, &ns, sizeof(float) * 2 * need_fpv * ctx->v_cap));
    dfree(ctx, ctx->state);
    dfree(ctx, ctx->snap_state);
    ctx->snap_state = nullptr;
    ctx->snap_valid = false;
    ctx->state = ns;
    ctx->state_fpv = need_fpv;
    drop_graphs(ctx);
  }
  if (ctx->pos_set && (old_ys != new_ys || old_f64 != new_f64)) {
    // re-pack the current positions for the new layout (velocity starts at 0)
    float* cur = ctx->ybuf[ctx->ctrl_h->cur];
    k_unpack_positions<<<grid_for(ctx->m, ctx->sm_count), 256, 0, ctx->stream>>>(cur, ctx->m, ctx->dim,
                                                                                old_ys, ctx->perm, ctx->stage,
                                                                                old_f64);
    CU(ctx, cudaMemsetAsync(ctx->state, 0, sizeof(float) * 2 * ctx->state_fpv * ctx->v_cap, ctx->stream));
    k_pack_positions<<<grid_for(ctx->m, ctx->sm_count), 256, 0, ctx->stream>>>(
        ctx->stage, ctx->m, ctx->dim, new_ys, ctx->perm,
        p->kind == IVHD_OPT_NESTEROV ? state_buf(ctx, ctx->ctrl_h->scur) : nullptr, vel_stride(ctx->dim),
        (float)p->beta, cur, new_f64);
    CU(ctx, cudaGetLastError());
  }
  CU(ctx, cudaMemsetAsync(ctx->state, 0, sizeof(float) * 2 * ctx->state_fpv * ctx->v_cap, ctx->stream));
  ctx->opt = *p;
  ctx->opt_set = true;
  Hyper h{};
  h.a = (float)p->a;
  h.g1 = p->gamma1;
  h.g2 = p->gamma2;
  h.tau = p->tau;
  h.adapt = p->auto_adapt;
  h.beta = (float)p->beta;
  h.gv = (float)p->gamma_v;
  h.gs = (float)p->gamma_s;
  h.rho = (float)p->rho;
  h.eps = (float)p->eps;
  h.gv_d = p->gamma_v;
  h.gs_d = p->gamma_s;
  h.eps_d = p->eps;
  ctx->hyper = h;
  ctx->ctrl_h->step = p->step;
  ctx->ctrl_h->adam_t = 0;
  ctx->ctrl_h->last_commit = 0;
  TRY(push_ctrl(ctx));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  drop_graphs(ctx);
  return IVHD_OK;
}

int ivhd_set_step_size(ivhd_ctx* ctx, double step) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  if (!(step > 0)) return fail(ctx, IVHD_ERR_INVALID_ARG, "step size must be positive, got %g", step);
  CU(ctx, cudaSetDevice(ctx->device));
  TRY(pull_ctrl(ctx));
  ctx->ctrl_h->step = step;
  TRY(push_ctrl(ctx));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  return IVHD_OK;
}

int ivhd_get_step_size(ivhd_ctx* ctx, double* step_out) {
  if (!ctx || !step_out) return fail(ctx, IVHD_ERR_INVALID_ARG, "null argument");
  CU(ctx, cudaSetDevice(ctx->device));
  TRY(pull_ctrl(ctx));
  *step_out = ctx->ctrl_h->step;
  return IVHD_OK;
}

static int ensure_trace(ivhd_ctx* ctx, int64_t n) {
  if (n <= ctx->trace_cap) return IVHD_OK;
  const int64_t cap = std::max<int64_t>(n, 4096);
  if (ctx->trace) dfree(ctx, ctx->trace);
  ctx->trace = nullptr;
  CU(ctx, dalloc(ctx, &ctx->trace, sizeof(double2) * cap));
  ctx->trace_cap = cap;
  drop_graphs(ctx);
  return IVHD_OK;
}

static int peer_masks(ivhd_ctx* ctx);
static int peer_pull(ivhd_ctx* ctx, bool barrier);

static void launch_unstep(ivhd_ctx* ctx, float* state, float step) {
  const int g = grid_for(ctx->m, ctx->sm_count);
  cudaStream_t st = ctx->stream;
  const double* f = ctx->op_force;
  const int64_t m = ctx->m;
  const Hyper h = ctx->hyper;
  const bool d2 = ctx->dim == 2;
  switch (ctx->opt.kind) {  // SGD keeps no state
    case OPT_FD:
      if (d2) k_unstep<2, OPT_FD><<<g, 256, 0, st>>>(state, f, m, step, h);
      else k_unstep<3, OPT_FD><<<g, 256, 0, st>>>(state, f, m, step, h);
      break;
    case OPT_MOM:
      if (d2) k_unstep<2, OPT_MOM><<<g, 256, 0, st>>>(state, f, m, step, h);
      else k_unstep<3, OPT_MOM><<<g, 256, 0, st>>>(state, f, m, step, h);
      break;
    case OPT_NEST:
      if (d2) k_unstep<2, OPT_NEST><<<g, 256, 0, st>>>(state, f, m, step, h);
      else k_unstep<3, OPT_NEST><<<g, 256, 0, st>>>(state, f, m, step, h);
      break;
    case OPT_ADADELTA:
      if (d2) k_unstep<2, OPT_ADADELTA><<<g, 256, 0, st>>>(state, f, m, step, h);
      else k_unstep<3, OPT_ADADELTA><<<g, 256, 0, st>>>(state, f, m, step, h);
      break;
    default: break;
  }
}

// Before re-running an iteration that paused at degenerate pairs (forces.py:
// 167-174): the fp32 kernels updated the optimizer state in place, so recover
// the old state by inverting that update with the forces the paused
// iteration used (the same kernel family at the same positions, without the
// missing directions); then choose the re-run kernel: the 2-D binary fast
// path only records degenerate pairs, so a binary set re-runs through the
// weighted instantiation (general path, applies the table) with {t, 1}
// entry weights built here.  The fp64 Adam kernel double-buffers its state
// and re-runs as is.
static int resume_degenerate(ivhd_ctx* ctx, int slot, int norm, StepArgs& R, KernelInfo& k, float2** tmp_ew) {
  const CsrSlot& S = ctx->slots[slot];
  const int opt = ctx->opt.kind, dim = ctx->dim;
  if (f64_of(opt)) return IVHD_OK;
  if (!ctx->op_y) CU(ctx, dalloc(ctx, &ctx->op_y, sizeof(float) * 4 * ctx->v_cap));
  if (!ctx->op_force) CU(ctx, dalloc(ctx, &ctx->op_force, sizeof(double) * 3 * ctx->v_cap));
  const int ys = ys_now(ctx), ys_op = dim == 2 ? 2 : 4, off = opt == OPT_NEST ? (dim == 2 ? 2 : 4) : 0;
  k_eval_positions<<<grid_for(ctx->m, ctx->sm_count), 256, 0, ctx->stream>>>(
      ctx->ybuf[ctx->ctrl_h->cur], ctx->m, ys, off, dim, ys_op, ctx->op_y);
  Ctrl oc{};
  oc.c = ctx->ctrl_h->c;
  oc.gstep = ctx->ctrl_h->gstep;
  CU(ctx, cudaMemcpyAsync(ctx->opctrl, &oc, sizeof(Ctrl), cudaMemcpyHostToDevice, ctx->stream));
  StepArgs O{};
  O.row_ptr = S.row_ptr;
  O.col = S.col;
  O.ew = S.ew;
  O.ybuf0 = O.ybuf1 = ctx->op_y;
  O.partial = ctx->partial;
  O.ctrl = ctx->opctrl;
  O.force_out = ctx->op_force;
  O.dg_key = ctx->dg_key;
  O.dg_vec = ctx->dg_vec;
  O.miss_n = ctx->miss_n;
  O.miss = ctx->miss;
  O.miss_cap = ctx->miss_cap;
  O.tile_g = S.tile_g;
  O.units = S.units;
  O.v_begin = 0;
  O.v_end = ctx->m;
  O.tile_v = ctx->tile_v;
  O.n_tiles = S.unit_base[ctx->n_tiles];
  O.n_tiles_global = O.n_tiles;
  O.norm = norm;
  TRY(launch_step(ctx, pick_kernel(dim, OPT_NONE, S.ew != nullptr, norm), O));
  float* st = state_buf(ctx, 0);
  launch_unstep(ctx, st, (float)ctx->ctrl_h->step);
  CU(ctx, cudaGetLastError());
  CU(ctx, cudaMemsetAsync(ctx->miss_n, 0, sizeof(int), ctx->stream));
  const bool fast = dim == 2 && S.ew == nullptr && norm == IVHD_NORM_L2 && opt != OPT_NEST;
  if (fast) {
    CU(ctx, dalloc(ctx, tmp_ew, sizeof(float2) * std::max<int64_t>(S.n, 1)));
    k_binary_ew<<<grid_for(S.n, ctx->sm_count), 256, 0, ctx->stream>>>(S.col, S.n, *tmp_ew);
    CU(ctx, cudaGetLastError());
    R.ew = *tmp_ew;
    k = pick_kernel(dim, opt, true, norm, ctx->peer_on);
    if (R.boff) {  // the cost-balanced schedule was built for the fast kernel's grid: plain round robin
      R.units = S.units;
      R.boff = nullptr;
    }
  }
  return IVHD_OK;
}

// After a run segment: status, trace and done count (engine.py:373-377 contract).
static int read_trace(ivhd_ctx* ctx, double* stress_out, double* step_out, int64_t* done_out) {
  TRY(pull_ctrl(ctx));
  const Ctrl& C = *ctx->ctrl_h;
  if (C.status == 3) return fail(ctx, IVHD_ERR_PEER, "peer exchange: a rank did not arrive within the time limit");
  if (C.status == 2) {  // paused before iteration C.iter: degenerate pairs need host-drawn directions
    const int64_t done = C.iter;
    if (done > 0 && (stress_out || step_out)) {
      std::vector<double2> tr(done);
      CU(ctx, cudaMemcpy(tr.data(), ctx->trace, sizeof(double2) * done, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < done; ++i) {
        if (stress_out) stress_out[i] = tr[i].x;
        if (step_out) step_out[i] = tr[i].y;
      }
    }
    if (done_out) *done_out = done;
    return IVHD_PAUSED_DEGENERATE;
  }
  const bool diverged = C.status != 0;
  const int64_t done = diverged ? C.diverged_at : C.iter;
  const int64_t ntr = diverged ? done + 1 : done;
  if (ntr > 0 && (stress_out || step_out)) {
    std::vector<double2> tr(ntr);
    CU(ctx, cudaMemcpy(tr.data(), ctx->trace, sizeof(double2) * ntr, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < ntr; ++i) {
      if (stress_out) stress_out[i] = tr[i].x;
      if (step_out) step_out[i] = tr[i].y;
    }
  }
  if (done_out) *done_out = done;
  if (diverged) return fail(ctx, IVHD_ERR_DIVERGED, "embedding diverged at local iteration %lld", (long long)done);
  return IVHD_OK;
}

int ivhd_run(ivhd_ctx* ctx, int slot, int norm, double c, int64_t n_iter, double* stress_out,
             double* step_out, int64_t* done_out) {
  TRY(check_ready(ctx, slot));
  if (done_out) *done_out = 0;
  if (norm != IVHD_NORM_L2 && norm != IVHD_NORM_L1) return fail(ctx, IVHD_ERR_INVALID_ARG, "unknown norm %d", norm);
  if (n_iter < 0) return fail(ctx, IVHD_ERR_INVALID_ARG, "n_iter must be >= 0");
  if (!ctx->pos_set) return fail(ctx, IVHD_ERR_STATE, "positions not set");
  if (ctx->sharded && !ctx->peer_on)
    return fail(ctx, IVHD_ERR_STATE, "context is sharded; use ivhd_shard_* or the peer exchange (ivhd_peer_*)");
  TRY(ensure_trace(ctx, n_iter));
  TRY(pull_ctrl(ctx));
  if (ctx->ctrl_h->status == 2)
    return fail(ctx, IVHD_ERR_STATE, "paused at a degenerate pair: call ivhd_set_degenerate first");
  if (ctx->ctrl_h->status != 0) return fail(ctx, IVHD_ERR_DIVERGED, "context already diverged");
  ctx->ctrl_h->c = c;
  ctx->ctrl_h->iter = 0;
  ctx->ctrl_h->arrive = 0;
  ctx->ctrl_h->next_tile = 0;
  ctx->ctrl_h->pend = 0;
  ctx->ctrl_h->readers = 0;
  ctx->ctrl_h->needw[0] = ctx->ctrl_h->needw[1] = 0;
  ctx->ctrl_h->fnf[0] = ctx->ctrl_h->fnf[1] = 0;
  for (int q = 0; q < 4; ++q) ctx->ctrl_h->facc[0][q] = ctx->ctrl_h->facc[1][q] = 0ull;
  TRY(push_ctrl(ctx));
  CU(ctx, cudaMemsetAsync(ctx->miss_n, 0, sizeof(int), ctx->stream));
  const CsrSlot& S = ctx->slots[slot];
  const bool peer = ctx->peer_on;
  KernelInfo fn = pick_kernel(ctx->dim, ctx->opt.kind, S.ew != nullptr, norm, peer);
  if (peer && ctx->masks_stale) TRY(peer_masks(ctx));
  StepArgs A = make_args(ctx, slot, norm, 1);  // peer mode too: running sums, one partial per block
  // one GPU, fp32 kernels: each launch decides its predecessor's iteration
  // (off the critical path of the launch boundary); k_defer_finalize decides
  // the segment's last one
  A.defer = (!peer && fn.smem > 0) ? 1 : 0;
  if (A.n_tiles > 0) {  // cost-balanced static schedule over this context's (rank's) units
    const int grid = std::max(1, std::min(A.n_tiles, occupancy(ctx, fn) * ctx->sm_count));
    TRY(build_schedule(ctx, ctx->slots[slot], grid, A.tile0, A.tile0 + A.n_tiles));
    A.units = S.sched_units;
    A.boff = S.sched_off;
  }
  // one iteration: the fused kernel (one GPU), or step + peer finalizer
  // peer mode: the step kernel's last block waits for the peers and decides
  // (one process per GPU); in-process contexts use the finalizer kernel
  auto launch_step = [&](ivhd_ctx* c, KernelInfo k, const StepArgs& a) -> int {
    TRY(::launch_step(c, k, a));
    return (peer && !c->pe.decide_here) ? launch_finalize_peer(c, a) : IVHD_OK;
  };
  int64_t left = n_iter;
  if (left > 0 && ctx->ctrl_h->dg_n > 0 && ctx->ctrl_h->dg_gstep == ctx->ctrl_h->gstep) {
    // re-run of the iteration that paused at degenerate pairs, with the
    // host-drawn directions (one launch, outside the graphs)
    StepArgs R = A;
    KernelInfo k = fn;
    float2* tmp_ew = nullptr;
    TRY(resume_degenerate(ctx, slot, norm, R, k, &tmp_ew));
    const int rc = launch_step(ctx, k, R);
    dfree(ctx, tmp_ew);  // stream-ordered after the launch
    TRY(rc);
    --left;
  }
  const int chunk = ctx->graph_chunk;
  if (left >= chunk) {
    const GraphKey key{slot, norm, ctx->opt.kind, (S.ew != nullptr ? 1 : 0) | (peer ? 2 : 0)};
    auto it = ctx->graphs.find(key);
    cudaGraphExec_t exec = nullptr;
    if (it == ctx->graphs.end()) {
      cudaGraph_t graph = nullptr;
      (void)occupancy(ctx, fn);  // not inside the capture
      CU(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
      int rc = IVHD_OK;
      for (int i = 0; i < chunk && rc == IVHD_OK; ++i) rc = launch_step(ctx, fn, A);
      cudaError_t ce = cudaStreamEndCapture(ctx->stream, &graph);
      if (rc != IVHD_OK) return rc;
      if (ce != cudaSuccess) return fail(ctx, IVHD_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ce));
      ce = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ce != cudaSuccess) return fail(ctx, IVHD_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ce));
      ctx->graphs[key] = exec;
    } else {
      exec = it->second;
    }
    while (left >= chunk) {
      CU(ctx, cudaGraphLaunch(exec, ctx->stream));
      left -= chunk;
    }
  }
  for (; left > 0; --left) TRY(launch_step(ctx, fn, A));
  if (A.defer) {
    if (ctx->opt.kind == OPT_FD) k_defer_finalize<OPT_FD><<<1, 32, 0, ctx->stream>>>(A);
    else k_defer_finalize<OPT_SGD><<<1, 32, 0, ctx->stream>>>(A);
    CU(ctx, cudaGetLastError());
  }
  if (peer && n_iter > 0) TRY(peer_pull(ctx, true));
  return read_trace(ctx, stress_out, step_out, done_out);
}

static int op_launch(ivhd_ctx* ctx, int slot, int norm, double c, const double* y, bool want_forces,
                     double* forces_out, double* stress_out) {
  TRY(check_ready(ctx, slot));
  if (norm != IVHD_NORM_L2 && norm != IVHD_NORM_L1) return fail(ctx, IVHD_ERR_INVALID_ARG, "unknown norm %d", norm);
  if (!y) return fail(ctx, IVHD_ERR_INVALID_ARG, "null positions");
  if (!ctx->op_y) CU(ctx, dalloc(ctx, &ctx->op_y, sizeof(float) * 4 * ctx->v_cap));
  if (!ctx->op_force) CU(ctx, dalloc(ctx, &ctx->op_force, sizeof(double) * 3 * ctx->v_cap));
  const int ys = ctx->dim == 2 ? 2 : 4;
  TRY(upload_stage(ctx, y, ctx->m * ctx->dim));
  k_pack_positions<<<grid_for(ctx->m, ctx->sm_count), 256, 0, ctx->stream>>>(ctx->stage, ctx->m, ctx->dim, ys,
                                                                           ctx->perm, nullptr, 0, 0.f, ctx->op_y);
  TRY(pull_ctrl(ctx));
  Ctrl oc{};
  oc.c = c;
  oc.gstep = ctx->ctrl_h->gstep;
  oc.dg_gstep = ctx->ctrl_h->dg_gstep;  // directions the host drew for this evaluation (forces.py:167-174)
  oc.dg_n = ctx->ctrl_h->dg_n;
  CU(ctx, cudaMemcpyAsync(ctx->opctrl, &oc, sizeof(Ctrl), cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, cudaMemsetAsync(ctx->miss_n, 0, sizeof(int), ctx->stream));
  const CsrSlot& S = ctx->slots[slot];
  StepArgs A{};
  A.row_ptr = S.row_ptr;
  A.col = S.col;
  A.ew = S.ew;
  A.ybuf0 = ctx->op_y;
  A.ybuf1 = ctx->op_y;
  A.partial = ctx->partial;
  A.ctrl = ctx->opctrl;
  A.force_out = ctx->op_force;
  A.dg_key = ctx->dg_key;
  A.dg_vec = ctx->dg_vec;
  A.miss_n = ctx->miss_n;
  A.miss = ctx->miss;
  A.miss_cap = ctx->miss_cap;
  A.tile_g = S.tile_g;
  A.units = S.units;
  A.v_begin = 0;
  A.v_end = ctx->m;
  A.tile_v = ctx->tile_v;
  A.n_tiles = S.unit_base[ctx->n_tiles];
  A.n_tiles_global = A.n_tiles;
  A.norm = norm;
  A.fuse_finalize = 0;
  // with host-drawn directions for this evaluation, a binary 2-D L2 set runs
  // through the weighted instantiation (the fast path only records pairs)
  float2* tmp_ew = nullptr;
  bool weighted = S.ew != nullptr;
  if (oc.dg_n > 0 && oc.dg_gstep == oc.gstep && !weighted && ctx->dim == 2 && norm == IVHD_NORM_L2) {
    CU(ctx, dalloc(ctx, &tmp_ew, sizeof(float2) * std::max<int64_t>(S.n, 1)));
    k_binary_ew<<<grid_for(S.n, ctx->sm_count), 256, 0, ctx->stream>>>(S.col, S.n, tmp_ew);
    A.ew = tmp_ew;
    weighted = true;
  }
  const int lrc = launch_step(ctx, pick_kernel(ctx->dim, OPT_NONE, weighted, norm), A);
  dfree(ctx, tmp_ew);
  TRY(lrc);
  k_reduce_partials<<<1, kBlock, 0, ctx->stream>>>(ctx->partial, A.n_tiles, ctx->red_out);
  CU(ctx, cudaGetLastError());
  double4 red;
  CU(ctx, cudaMemcpyAsync(&red, ctx->red_out, sizeof(double4), cudaMemcpyDeviceToHost, ctx->stream));
  if (want_forces) {
    k_unpermute_f64<<<grid_for(ctx->m, ctx->sm_count), 256, 0, ctx->stream>>>(ctx->op_force, ctx->m, ctx->dim,
                                                                             ctx->perm, ctx->stage);
    CU(ctx, cudaMemcpyAsync(forces_out, ctx->stage, sizeof(double) * ctx->m * ctx->dim,
                            cudaMemcpyDeviceToHost, ctx->stream));
  }
  int nmiss = 0;
  CU(ctx, cudaMemcpyAsync(&nmiss, ctx->miss_n, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  if (stress_out) *stress_out = 0.5 * red.x;
  if (want_forces && nmiss > 0) {  // directions needed: ivhd_degenerate_pending, then call again
    ctx->op_paused = true;
    return IVHD_PAUSED_DEGENERATE;
  }
  if (ctx->ctrl_h->dg_n > 0) {  // the table served this evaluation only
    ctx->ctrl_h->dg_n = 0;
    TRY(push_ctrl(ctx));
  }
  return IVHD_OK;
}

// Degenerate pairs met by the paused iteration (or operator call): row in
// the caller's ids and entry index in that row of the symmetrised CSR (out-
// halves in connection order, then in-halves in connection order).
int ivhd_degenerate_pending(ivhd_ctx* ctx, int64_t cap, int64_t* n_out, int32_t* rows_out, int32_t* entries_out) {
  if (!ctx || !n_out) return fail(ctx, IVHD_ERR_INVALID_ARG, "null argument");
  CU(ctx, cudaSetDevice(ctx->device));
  int n = 0;
  CU(ctx, cudaMemcpy(&n, ctx->miss_n, sizeof(int), cudaMemcpyDeviceToHost));
  if (n > ctx->miss_cap)
    return fail(ctx, IVHD_ERR_STATE, "%d degenerate pairs in one iteration (capacity %d)", n, ctx->miss_cap);
  *n_out = n;
  if (n == 0 || cap <= 0) return IVHD_OK;
  const int k = (int)std::min<int64_t>(n, cap);
  std::vector<int2> ms(k);
  std::vector<int32_t> perm(1);
  CU(ctx, cudaMemcpy(ms.data(), ctx->miss, sizeof(int2) * k, cudaMemcpyDeviceToHost));
  for (int i = 0; i < k; ++i) {
    int32_t orig = 0;
    CU(ctx, cudaMemcpy(&orig, ctx->perm + ms[i].x, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (rows_out) rows_out[i] = orig;
    if (entries_out) entries_out[i] = ms[i].y;
  }
  return IVHD_OK;
}

// Directions for the paused iteration: (row, entry) as reported by
// ivhd_degenerate_pending, vecs (n, dim) = w * t * unit direction with the
// sign of the row's side (+ for the connection's source row, - for its
// destination row).  Resumes the context; the table is valid for that one
// iteration (or the next operator call).
int ivhd_set_degenerate(ivhd_ctx* ctx, int64_t n, const int32_t* rows, const int32_t* entries, const double* vecs) {
  if (!ctx || n < 0 || (n > 0 && (!rows || !entries || !vecs))) return fail(ctx, IVHD_ERR_INVALID_ARG, "bad arguments");
  CU(ctx, cudaSetDevice(ctx->device));
  TRY(pull_ctrl(ctx));
  if (n > ctx->dg_cap) {
    dfree(ctx, ctx->dg_key);
    dfree(ctx, ctx->dg_vec);
    ctx->dg_key = nullptr;
    ctx->dg_vec = nullptr;
    CU(ctx, dalloc(ctx, &ctx->dg_key, sizeof(int2) * n));
    CU(ctx, dalloc(ctx, &ctx->dg_vec, sizeof(float4) * n));
    ctx->dg_cap = n;
    drop_graphs(ctx);  // captured launches hold the table pointers
  }
  std::vector<int32_t> inv(ctx->m);
  if (n > 0) CU(ctx, cudaMemcpy(inv.data(), ctx->inv, sizeof(int32_t) * ctx->m, cudaMemcpyDeviceToHost));
  std::vector<int2> key(n);
  std::vector<float4> vec(n);
  for (int64_t i = 0; i < n; ++i) {
    if (rows[i] < 0 || rows[i] >= ctx->m) return fail(ctx, IVHD_ERR_INVALID_ARG, "row %d out of range", rows[i]);
    key[i] = make_int2(inv[rows[i]], entries[i]);
    const double* v = vecs + i * ctx->dim;
    vec[i] = make_float4((float)v[0], (float)v[1], ctx->dim == 3 ? (float)v[2] : 0.f, 0.f);
  }
  if (n > 0) {
    CU(ctx, cudaMemcpy(ctx->dg_key, key.data(), sizeof(int2) * n, cudaMemcpyHostToDevice));
    CU(ctx, cudaMemcpy(ctx->dg_vec, vec.data(), sizeof(float4) * n, cudaMemcpyHostToDevice));
  }
  ctx->ctrl_h->dg_n = (int)n;
  ctx->ctrl_h->dg_gstep = ctx->ctrl_h->gstep;
  if (ctx->ctrl_h->status == 2) ctx->ctrl_h->status = 0;
  ctx->ctrl_h->need = 0;
  ctx->op_paused = false;
  TRY(push_ctrl(ctx));
  CU(ctx, cudaMemsetAsync(ctx->miss_n, 0, sizeof(int), ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  return IVHD_OK;
}

int ivhd_compute_forces(ivhd_ctx* ctx, int slot, int norm, double c, const double* y, double* forces_out,
                        double* stress_out) {
  if (!forces_out) return fail(ctx, IVHD_ERR_INVALID_ARG, "null forces_out");
  return op_launch(ctx, slot, norm, c, y, true, forces_out, stress_out);
}

int ivhd_stress(ivhd_ctx* ctx, int slot, int norm, double c, const double* y, double* stress_out) {
  return op_launch(ctx, slot, norm, c, y, false, nullptr, stress_out);
}

int ivhd_snapshot(ivhd_ctx* ctx) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  CU(ctx, cudaSetDevice(ctx->device));
  const size_t bytes = sizeof(float) * 8 * ctx->v_cap;
  if (!ctx->snap_y) CU(ctx, dalloc(ctx, &ctx->snap_y, bytes));
  if (!ctx->snap_state) CU(ctx, dalloc(ctx, &ctx->snap_state, sizeof(float) * ctx->state_fpv * ctx->v_cap));
  TRY(pull_ctrl(ctx));
  const size_t used = sizeof(float) * 8 * ctx->m;
  CU(ctx, cudaMemcpyAsync(ctx->snap_y, ctx->ybuf[ctx->ctrl_h->cur], used, cudaMemcpyDeviceToDevice, ctx->stream));
  CU(ctx, cudaMemcpyAsync(ctx->snap_state, state_buf(ctx, ctx->ctrl_h->scur), sizeof(float) * ctx->state_fpv * ctx->m,
                          cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->snap_ctrl = *ctx->ctrl_h;
  ctx->snap_valid = true;
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  return IVHD_OK;
}

int ivhd_restore(ivhd_ctx* ctx) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  if (!ctx->snap_valid) return fail(ctx, IVHD_ERR_STATE, "no snapshot taken");
  CU(ctx, cudaSetDevice(ctx->device));
  const size_t used = sizeof(float) * 8 * ctx->m;
  *ctx->ctrl_h = ctx->snap_ctrl;
  CU(ctx, cudaMemcpyAsync(ctx->ybuf[ctx->snap_ctrl.cur], ctx->snap_y, used, cudaMemcpyDeviceToDevice, ctx->stream));
  CU(ctx, cudaMemcpyAsync(state_buf(ctx, ctx->snap_ctrl.scur), ctx->snap_state, sizeof(float) * ctx->state_fpv * ctx->m,
                          cudaMemcpyDeviceToDevice, ctx->stream));
  TRY(push_ctrl(ctx));
  return IVHD_OK;  // asynchronous: ordered before the next launch on the stream
}


}  // extern "C"

// gather-only pass over a CSR (ivhd_gather_floor), in one of two orders:
// BLOCKED (8 or, like the step kernel, 3 blocks per SM) — every block sweeps
// one contiguous slice of the column ids, as the
// step kernel's blocks sweep contiguous unit ranges (id-local neighbourhoods
// are reused in L1); STRIDED — the whole grid sweeps the ids front to back
// (no per-SM locality, all SMs on one region of L2).  8 column ids and 8
// position gathers in flight per thread, the step kernel's load instructions
// (streamed ids, evict-first in L2 when the working set exceeds it;
// L1-allocating position loads).
__device__ __forceinline__ uint32_t ld_col_first(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
template <int YS, bool BLOCKED>
__global__ void k_gather_floor(const uint32_t* __restrict__ col, int64_t n, const float* __restrict__ Y,
                               int stream_hint, float* __restrict__ sink) {
  using V = typename std::conditional<YS == 2, float2, float4>::type;
  constexpr int kStride = YS / (int)(sizeof(V) / 4);
  const V* Yv = reinterpret_cast<const V*>(Y);
  int64_t b0 = 0, b1 = n, i, stride;
  if (BLOCKED) {
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    b0 = blockIdx.x * per;
    b1 = min(n, b0 + per);
    i = b0 + threadIdx.x;
    stride = blockDim.x;
  } else {
    i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    stride = (int64_t)gridDim.x * blockDim.x;
  }
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  float acc = 0.f;
  for (; i + 7 * stride < b1; i += 8 * stride) {
    uint32_t j[8];
    V p[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      j[q] = (stream_hint ? ld_col_first(col + i + q * stride, pol) : ld_col(col + i + q * stride)) & kIdMask;
#pragma unroll
    for (int q = 0; q < 8; ++q) p[q] = __ldg(Yv + (size_t)j[q] * kStride);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += p[q].x * p[q].y;
  }
  for (; i < b1; i += stride) {
    const V p = __ldg(Yv + (size_t)(ld_col(col + i) & kIdMask) * kStride);
    acc += p.x * p.y;
  }
  if (acc == 1.2345e-30f) *sink = acc;  // keeps the loads
}

extern "C" {

int ivhd_gather_floor(ivhd_ctx* ctx, int slot, int reps, double* us_out) {
  TRY(check_ready(ctx, slot));
  if (!us_out || reps < 1) return fail(ctx, IVHD_ERR_INVALID_ARG, "us_out and reps >= 1 required");
  CU(ctx, cudaSetDevice(ctx->device));
  const CsrSlot& S = ctx->slots[slot];
  const int ys = ys_now(ctx);
  const float* y = ctx->ybuf[ctx->ctrl_h->cur];
  float* sink = reinterpret_cast<float*>(ctx->stage);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device);
  const int hint = 4 * S.n + (int64_t)4 * ctx->m * ys > (int64_t)l2 ? 1 : 0;
  int which = 0;  // launch order: blocked (8 and 3 blocks per SM), strided; the best is the floor
  auto launch = [&] {
    const int grid = ctx->sm_count * (which == 1 ? 3 : 8);
#define IVHD_GF(Y)                                                                                   \
  if (which < 2) k_gather_floor<Y, true><<<grid, 256, 0, ctx->stream>>>(S.col, S.n, y, hint, sink); \
  else k_gather_floor<Y, false><<<grid, 256, 0, ctx->stream>>>(S.col, S.n, y, hint, sink);
    if (ys == 2) { IVHD_GF(2) } else if (ys == 4) { IVHD_GF(4) } else { IVHD_GF(8) }
#undef IVHD_GF
  };
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  CU(ctx, cudaEventCreate(&e0));
  CU(ctx, cudaEventCreate(&e1));
  double best = 1e30;
  cudaError_t e = cudaSuccess;
  for (int r = 0; r < 3 * (reps + 2) && e == cudaSuccess; ++r) {
    which = r % 3;
    cudaEventRecord(e0, ctx->stream);
    launch();
    cudaEventRecord(e1, ctx->stream);
    if ((e = cudaEventSynchronize(e1)) != cudaSuccess) break;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 6) best = std::min(best, (double)ms * 1e3);  // two warm-up passes each (L2 warm like the loop's)
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (e != cudaSuccess) return fail(ctx, IVHD_ERR_CUDA, "gather floor: %s", cudaGetErrorString(e));
  CU(ctx, cudaGetLastError());
  *us_out = best;
  return IVHD_OK;
}

int ivhd_synchronize(ivhd_ctx* ctx) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  CU(ctx, cudaSetDevice(ctx->device));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  return IVHD_OK;
}

// ------------------------------------------------------------ sharded mode

// unit partials of this rank's tiles -> tile partials (the fp64 kernel writes tiles directly)
static int fold_tiles(ivhd_ctx* ctx, const CsrSlot& S) {
  const int t0 = (int)(ctx->shard_begin / ctx->tile_v), t1 = (int)(ctx->shard_end / ctx->tile_v);
  if (t1 > t0)
    k_fold_tiles<<<(t1 - t0 + 255) / 256, 256, 0, ctx->stream>>>(
        ctx->partial, f64_of(ctx->opt.kind) ? nullptr : S.d_unit_base, t0, t1, ctx->tpart, ctx->ctrl);
  CU(ctx, cudaGetLastError());
  return IVHD_OK;
}

int ivhd_tile_vertices(ivhd_ctx* ctx, int64_t* tile_v_out, int64_t* n_tiles_out) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  if (tile_v_out) *tile_v_out = ctx->tile_v;
  if (n_tiles_out) *n_tiles_out = ctx->n_tiles_cap;
  return IVHD_OK;
}

int ivhd_shard_set_range(ivhd_ctx* ctx, int64_t v_begin, int64_t v_end) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  if (v_begin < 0 || v_end < v_begin || v_end > ctx->v_cap || v_begin % ctx->tile_v || v_end % ctx->tile_v)
    return fail(ctx, IVHD_ERR_INVALID_ARG, "shard range [%lld, %lld) not tile aligned (tile %d, cap %lld)",
                (long long)v_begin, (long long)v_end, ctx->tile_v, (long long)ctx->v_cap);
  ctx->shard_begin = v_begin;
  ctx->shard_end = v_end;
  ctx->sharded = true;
  CU(ctx, cudaSetDevice(ctx->device));
  CU(ctx, cudaMemsetAsync(ctx->partial, 0, sizeof(double4) * 32 * ctx->n_tiles_cap, ctx->stream));
  CU(ctx, cudaMemsetAsync(ctx->tpart, 0, sizeof(double4) * ctx->n_tiles_cap, ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  return IVHD_OK;
}

int ivhd_shard_buffers(ivhd_ctx* ctx, uint64_t* ybuf0, uint64_t* ybuf1, int64_t* floats_per_vertex,
                       uint64_t* partials, int* cur_out) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  TRY(pull_ctrl(ctx));
  if (ybuf0) *ybuf0 = reinterpret_cast<uint64_t>(ctx->ybuf[0]);
  if (ybuf1) *ybuf1 = reinterpret_cast<uint64_t>(ctx->ybuf[1]);
  if (floats_per_vertex) *floats_per_vertex = ys_of(ctx->dim, ctx->opt.kind);
  if (partials) *partials = reinterpret_cast<uint64_t>(ctx->tpart);
  if (cur_out) *cur_out = ctx->ctrl_h->cur;
  return IVHD_OK;
}

int ivhd_step_local(ivhd_ctx* ctx, int slot, int norm, double c) {
  TRY(check_ready(ctx, slot));
  if (!ctx->sharded) return fail(ctx, IVHD_ERR_STATE, "call ivhd_shard_set_range first");
  if (!ctx->pos_set) return fail(ctx, IVHD_ERR_STATE, "positions not set");
  TRY(ensure_trace(ctx, 1));
  TRY(pull_ctrl(ctx));
  if (ctx->ctrl_h->status != 0) return fail(ctx, IVHD_ERR_DIVERGED, "context already diverged");
  ctx->ctrl_h->c = c;
  ctx->ctrl_h->iter = 0;
  ctx->ctrl_h->arrive = 0;
  ctx->ctrl_h->next_tile = 0;
  TRY(push_ctrl(ctx));
  StepArgs A = make_args(ctx, slot, norm, 0);
  const CsrSlot& S = ctx->slots[slot];
  if (A.n_tiles > 0) TRY(launch_step(ctx, pick_kernel(ctx->dim, ctx->opt.kind, S.ew != nullptr, norm), A));
  TRY(fold_tiles(ctx, S));
  ctx->shard_slot = slot;
  return IVHD_OK;
}

int ivhd_step_finalize(ivhd_ctx* ctx, double* stress_out, double* step_out, int* committed_out) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  CU(ctx, cudaSetDevice(ctx->device));
  StepArgs A = make_args(ctx, ctx->shard_slot, 0, 0);
  pick_finalize(ctx->opt.kind)<<<1, kBlock, 0, ctx->stream>>>(A);
  CU(ctx, cudaGetLastError());
  TRY(pull_ctrl(ctx));
  double2 tr;
  CU(ctx, cudaMemcpy(&tr, ctx->trace, sizeof(double2), cudaMemcpyDeviceToHost));
  if (stress_out) *stress_out = tr.x;
  if (step_out) *step_out = tr.y;
  if (committed_out) *committed_out = ctx->ctrl_h->last_commit;
  if (ctx->ctrl_h->status != 0) return fail(ctx, IVHD_ERR_DIVERGED, "embedding diverged");
  return IVHD_OK;
}

// ---- asynchronous sharded loop: no host round trip per iteration.  The
// host picks the buffers by parity (read ybuf[cur], write ybuf[cur^1]); the
// finalizer makes the written buffer current (refilling it on a rollback),
// so the exchange buffer of every iteration is known without reading ctrl.

int ivhd_shard_begin(ivhd_ctx* ctx, int slot, double c, int64_t n_iter, int* cur_out, int64_t* epoch_out) {
  TRY(check_ready(ctx, slot));
  if (!ctx->sharded) return fail(ctx, IVHD_ERR_STATE, "call ivhd_shard_set_range first");
  if (!ctx->pos_set) return fail(ctx, IVHD_ERR_STATE, "positions not set");
  if (n_iter < 0) return fail(ctx, IVHD_ERR_INVALID_ARG, "n_iter must be >= 0");
  TRY(ensure_trace(ctx, std::max<int64_t>(n_iter, 1)));
  TRY(pull_ctrl(ctx));
  if (ctx->ctrl_h->status != 0) return fail(ctx, IVHD_ERR_DIVERGED, "context already diverged");
  ctx->ctrl_h->c = c;
  ctx->ctrl_h->iter = 0;
  ctx->ctrl_h->arrive = 0;
  ctx->ctrl_h->next_tile = 0;
  TRY(push_ctrl(ctx));
  ctx->shard_cur = ctx->ctrl_h->cur;
  ctx->shard_slot = slot;
  if (cur_out) *cur_out = ctx->shard_cur;
  if (epoch_out) *epoch_out = ctx->graph_epoch;
  return IVHD_OK;
}

static void shard_io(ivhd_ctx* ctx, StepArgs& A) {
  A.fixed_io = 1;
  A.ybuf0 = ctx->ybuf[ctx->shard_cur];
  A.ybuf1 = ctx->ybuf[ctx->shard_cur ^ 1];
  A.out_index = ctx->shard_cur ^ 1;
  A.v_cap_floats = ctx->v_cap * ys_of(ctx->dim, ctx->opt.kind);
}

int ivhd_shard_step(ivhd_ctx* ctx, int slot, int norm, uint64_t* exchange_out) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  if (slot < 0 || slot > 1 || !ctx->slots[slot].valid) return fail(ctx, IVHD_ERR_STATE, "connection slot %d not set", slot);
  if (norm != IVHD_NORM_L2 && norm != IVHD_NORM_L1) return fail(ctx, IVHD_ERR_INVALID_ARG, "unknown norm %d", norm);
  if (!ctx->sharded) return fail(ctx, IVHD_ERR_STATE, "call ivhd_shard_set_range first");
  CU(ctx, cudaSetDevice(ctx->device));
  StepArgs A = make_args(ctx, slot, norm, 0);
  const CsrSlot& S = ctx->slots[slot];
  ctx->shard_slot = slot;
  if (ctx->peer_on) {  // fused peer exchange: the kernel publishes to every rank itself
    if (ctx->masks_stale) {
      TRY(peer_masks(ctx));
      A.pe = ctx->pe;
    }
    A.fuse_finalize = 1;  // running sums, one partial per block (round-robin units here)
    if (A.n_tiles > 0) TRY(launch_step(ctx, pick_kernel(ctx->dim, ctx->opt.kind, S.ew != nullptr, norm, true), A));
    if (exchange_out) *exchange_out = 0;
    return IVHD_OK;
  }
  shard_io(ctx, A);
  if (A.n_tiles > 0) TRY(launch_step(ctx, pick_kernel(ctx->dim, ctx->opt.kind, S.ew != nullptr, norm), A));
  TRY(fold_tiles(ctx, S));
  if (exchange_out) *exchange_out = reinterpret_cast<uint64_t>(ctx->ybuf[ctx->shard_cur ^ 1]);
  return IVHD_OK;
}

int ivhd_shard_finalize(ivhd_ctx* ctx) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  CU(ctx, cudaSetDevice(ctx->device));
  StepArgs A = make_args(ctx, ctx->shard_slot, 0, 0);
  if (ctx->peer_on) return launch_finalize_peer(ctx, A);
  shard_io(ctx, A);
  pick_finalize(ctx->opt.kind)<<<1, kBlock, 0, ctx->stream>>>(A);
  CU(ctx, cudaGetLastError());
  ctx->shard_cur ^= 1;
  return IVHD_OK;
}

int ivhd_shard_end(ivhd_ctx* ctx, double* stress_out, double* step_out, int64_t* done_out) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  CU(ctx, cudaSetDevice(ctx->device));
  const int rc = read_trace(ctx, stress_out, step_out, done_out);
  ctx->shard_cur = ctx->ctrl_h->cur;
  return rc;
}

// ------------------------------------------------------ fused peer exchange

// Move the buffers peers write into to cudaMalloc memory (CUDA IPC needs it)
// and allocate the tile partials [2][n_tiles_cap], arrival flags and stamp.
static int peer_alloc(ivhd_ctx* ctx, int world, int rank) {
  if (!ctx->sharded) return fail(ctx, IVHD_ERR_STATE, "call ivhd_shard_set_range first");
  if (world < 1 || world > kMaxPeers + 1 || rank < 0 || rank >= world)
    return fail(ctx, IVHD_ERR_INVALID_ARG, "peer exchange: world %d rank %d (1..8 ranks)", world, rank);
  CU(ctx, cudaSetDevice(ctx->device));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  if (!ctx->ybuf_malloc) {
    const size_t bytes = sizeof(float) * 8 * ctx->v_cap;
    for (int b = 0; b < 2; ++b) {
      float* nb = nullptr;
      CU(ctx, cudaMalloc(&nb, bytes));
      CU(ctx, cudaMemcpy(nb, ctx->ybuf[b], bytes, cudaMemcpyDeviceToDevice));
      dfree(ctx, ctx->ybuf[b]);
      ctx->ybuf[b] = nb;
    }
    ctx->ybuf_malloc = true;
  }
  // rank-partial slots: [2 parities][world ranks]
  const int64_t n_slots = world;
  if (ctx->tp2 && ctx->tp2_slots < n_slots) {
    cudaFree(ctx->tp2);
    ctx->tp2 = nullptr;
  }
  if (!ctx->tp2) {
    CU(ctx, cudaMalloc(&ctx->tp2, sizeof(double4) * 2 * n_slots));
    ctx->tp2_slots = n_slots;
  }
  // flags: [0, 8) iteration arrivals, [8, 16) end-of-run barrier; stamp: [0] iterations, [1] barriers
  if (!ctx->flags) CU(ctx, cudaMalloc(&ctx->flags, sizeof(unsigned long long) * 16));
  if (!ctx->stamp) CU(ctx, cudaMalloc(&ctx->stamp, sizeof(unsigned long long) * 2));
  CU(ctx, cudaMemset(ctx->tp2, 0, sizeof(double4) * 2 * ctx->tp2_slots));
  CU(ctx, cudaMemset(ctx->flags, 0, sizeof(unsigned long long) * 16));
  CU(ctx, cudaMemset(ctx->stamp, 0, sizeof(unsigned long long) * 2));
  CU(ctx, cudaDeviceSynchronize());
  ctx->world = world;
  ctx->rank = rank;
  PeerArgs& pe = ctx->pe;
  pe = PeerArgs{};
  pe.n_peers = 0;
  pe.rank = rank;
  pe.world = world;
  pe.t0 = (int)(ctx->shard_begin / ctx->tile_v);
  pe.t1 = (int)(ctx->shard_end / ctx->tile_v);
  pe.tp_local = ctx->tp2;
  pe.fl_local = ctx->flags;
  pe.stamp = ctx->stamp;
  pe.n_tiles_cap = ctx->n_tiles_cap;
  pe.decide_here = 1;
  pe.timeout_ns = 60LL * 1000 * 1000 * 1000;  // peer failure detection (ranks start segments with skew)
  drop_graphs(ctx);
  return IVHD_OK;
}

int ivhd_peer_export(ivhd_ctx* ctx, int world, int rank, uint8_t* handle_out) {
  if (!ctx || !handle_out) return fail(ctx, IVHD_ERR_INVALID_ARG, "null argument");
  TRY(peer_alloc(ctx, world, rank));
  cudaIpcMemHandle_t h[4];
  CU(ctx, cudaIpcGetMemHandle(&h[0], ctx->ybuf[0]));
  CU(ctx, cudaIpcGetMemHandle(&h[1], ctx->ybuf[1]));
  CU(ctx, cudaIpcGetMemHandle(&h[2], ctx->tp2));
  CU(ctx, cudaIpcGetMemHandle(&h[3], ctx->flags));
  static_assert(sizeof(h) <= IVHD_PEER_HANDLE_BYTES, "handle size");
  memset(handle_out, 0, IVHD_PEER_HANDLE_BYTES);
  memcpy(handle_out, h, sizeof(h));
  return IVHD_OK;
}

// Halo masks of the own range from every valid connection set (called when
// the peer exchange is set up and after every CSR build in peer mode).
static int peer_masks(ivhd_ctx* ctx) {
  if (!ctx->peer_on) return IVHD_OK;
  if (!ctx->hmask) CU(ctx, dalloc(ctx, &ctx->hmask, (size_t)ctx->v_cap));
  CU(ctx, cudaMemsetAsync(ctx->hmask, 0, (size_t)ctx->v_cap, ctx->stream));
  const int64_t range_v = (int64_t)(ctx->n_tiles_cap / ctx->world) * ctx->tile_v;
  const int64_t v1 = std::min<int64_t>(ctx->shard_end, ctx->m);
  for (const CsrSlot& S : ctx->slots)
    if (S.valid && v1 > ctx->shard_begin)
      k_halo_mask<<<grid_for(v1 - ctx->shard_begin, ctx->sm_count), 256, 0, ctx->stream>>>(
          S.row_ptr, S.col, ctx->shard_begin, v1, range_v, ctx->rank, ctx->hmask);
  CU(ctx, cudaGetLastError());
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->pe.mask = ctx->hmask;
  ctx->masks_stale = false;
  return IVHD_OK;
}

static int peer_finish(ivhd_ctx* ctx) {
  ctx->pe.on = 1;
  ctx->peer_on = true;
  drop_graphs(ctx);
  return peer_masks(ctx);
}

// End of a peer-mode run segment: complete the local replica (both buffers)
// with every peer's own range, then an all-rank barrier (flags [8, 16)) so no
// rank starts its next segment — which overwrites its buffers — while another
// is still reading them.
static int peer_pull(ivhd_ctx* ctx, bool barrier) {
  const int64_t range_v = (int64_t)(ctx->n_tiles_cap / ctx->world) * ctx->tile_v;
  const int ys = ys_of(ctx->dim, ctx->opt.kind);
  const PeerArgs& pe = ctx->pe;
  for (int k = 0; k < pe.n_peers; ++k) {
    const int q = pe.prank[k];
    const int64_t a = (int64_t)q * range_v * ys / 4, b = std::min<int64_t>(ctx->m, (int64_t)(q + 1) * range_v) * ys / 4 + 1;
    if (b <= a) continue;
    k_peer_pull<<<grid_for(b - a, ctx->sm_count), 256, 0, ctx->stream>>>(
        reinterpret_cast<float4*>(ctx->ybuf[0]), reinterpret_cast<float4*>(ctx->ybuf[1]),
        reinterpret_cast<const float4*>(pe.y0[k]), reinterpret_cast<const float4*>(pe.y1[k]), a, b);
  }
  if (barrier) k_peer_barrier<<<1, 32, 0, ctx->stream>>>(pe, ctx->ctrl);
  CU(ctx, cudaGetLastError());
  return IVHD_OK;
}

int ivhd_peer_halo(ivhd_ctx* ctx, int64_t* records_out, int64_t* bytes_out) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  if (!ctx->peer_on) return fail(ctx, IVHD_ERR_STATE, "peer exchange not set up");
  CU(ctx, cudaSetDevice(ctx->device));
  if (ctx->masks_stale) TRY(peer_masks(ctx));
  const int64_t v0 = ctx->shard_begin, v1 = std::min<int64_t>(ctx->shard_end, ctx->m);
  std::vector<uint8_t> mk(std::max<int64_t>(v1 - v0, 0));
  if (!mk.empty()) CU(ctx, cudaMemcpy(mk.data(), ctx->hmask + v0, mk.size(), cudaMemcpyDeviceToHost));
  int64_t n = 0;
  for (uint8_t b : mk) n += __builtin_popcount(b);
  if (records_out) *records_out = n;
  if (bytes_out) *bytes_out = n * (int64_t)sizeof(float) * ys_of(ctx->dim, ctx->opt.kind);
  return IVHD_OK;
}

int ivhd_peer_set_timeout(ivhd_ctx* ctx, double seconds) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  if (!ctx->peer_on) return fail(ctx, IVHD_ERR_STATE, "peer exchange not set up");
  if (!(seconds > 0.0) || seconds > 3600.0) return fail(ctx, IVHD_ERR_INVALID_ARG, "timeout must be in (0, 3600] s");
  ctx->pe.timeout_ns = (long long)(seconds * 1e9);
  drop_graphs(ctx);  // captured launches hold the old arguments
  return IVHD_OK;
}

int ivhd_peer_pull(ivhd_ctx* ctx, int barrier) {
  if (!ctx) return fail(nullptr, IVHD_ERR_INVALID_ARG, "null context");
  if (!ctx->peer_on) return fail(ctx, IVHD_ERR_STATE, "peer exchange not set up");
  CU(ctx, cudaSetDevice(ctx->device));
  TRY(peer_pull(ctx, barrier != 0));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  return IVHD_OK;
}

int ivhd_peer_import(ivhd_ctx* ctx, const uint8_t* all_handles) {
  if (!ctx || !all_handles) return fail(ctx, IVHD_ERR_INVALID_ARG, "null argument");
  if (!ctx->tp2) return fail(ctx, IVHD_ERR_STATE, "call ivhd_peer_export first");
  CU(ctx, cudaSetDevice(ctx->device));
  PeerArgs& pe = ctx->pe;
  pe.n_peers = 0;
  for (int q = 0; q < ctx->world; ++q) {
    if (q == ctx->rank) continue;
    cudaIpcMemHandle_t h[4];
    memcpy(h, all_handles + (size_t)q * IVHD_PEER_HANDLE_BYTES, sizeof(h));
    void* p[4];
    for (int i = 0; i < 4; ++i) {
      CU(ctx, cudaIpcOpenMemHandle(&p[i], h[i], cudaIpcMemLazyEnablePeerAccess));
      ctx->ipc_opened.push_back(p[i]);
    }
    const int k = pe.n_peers++;
    pe.prank[k] = q;
    pe.y0[k] = static_cast<float*>(p[0]);
    pe.y1[k] = static_cast<float*>(p[1]);
    pe.tp[k] = static_cast<double4*>(p[2]);
    pe.fl[k] = static_cast<unsigned long long*>(p[3]);
  }
  return peer_finish(ctx);
}

int ivhd_peer_import_local(ivhd_ctx* ctx, ivhd_ctx* const* ctxs) {
  if (!ctx || !ctxs) return fail(ctx, IVHD_ERR_INVALID_ARG, "null argument");
  if (!ctx->tp2) return fail(ctx, IVHD_ERR_STATE, "call ivhd_peer_export first");
  PeerArgs& pe = ctx->pe;
  pe.n_peers = 0;
  pe.decide_here = 0;  // ranks share this process (and GPU): a separate finalizer decides
  for (int q = 0; q < ctx->world; ++q) {
    if (q == ctx->rank) continue;
    const ivhd_ctx* o = ctxs[q];
    if (!o || !o->tp2 || o->world != ctx->world || o->rank != q)
      return fail(ctx, IVHD_ERR_STATE, "peer context %d not exported for world %d", q, ctx->world);
    const int k = pe.n_peers++;
    pe.prank[k] = q;
    pe.y0[k] = o->ybuf[0];
    pe.y1[k] = o->ybuf[1];
    pe.tp[k] = o->tp2;
    pe.fl[k] = o->flags;
  }
  return peer_finish(ctx);
}

}  // extern "C"
