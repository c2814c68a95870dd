// ivhd_rng.cuh — numpy's default generator stream (PCG64, XSL-RR 128/64) on the
// device, so the run's initial layout and random partners are drawn on the GPU
// bit-identically to engine.py:124-146 (init_layout, sample_random_neighbors).
//
// The reference draws, from ONE numpy Generator:
//   * gen.uniform(-1, 1, size=(M, dim))  -> M*dim 64-bit outputs,
//     lo + (hi-lo) * ((x >> 11) * 2^-53)                       (row-major)
//   * gen.integers(0, M, size=(M, rn))   -> Lemire's bounded 32-bit sampler
//     over the 32-bit halves of the 64-bit outputs (low half first, the high
//     half is buffered in the generator: has_uint32 / uinteger), rejecting a
//     draw iff (u32 * M) mod 2^32 < (2^32 - M) mod M
//   * then, while any pick equals its row or one of the row's nn ids, the
//     rejected slots (row-major order) are re-drawn with further integers().
//
// Every output is a pure function of (start state, index): a thread jumps the
// LCG ahead to its chunk (O(log n) 128-bit multiplies) and steps from there.
// Lemire acceptance does not depend on the position, so the first batch is
// a stream compaction of candidates; the few collision re-draws continue the
// stream on the host (same arithmetic, host side of the boundary).
#pragma once
#include <cstdint>

namespace ivhd {
namespace pcg {

typedef unsigned __int128 u128;

__host__ __device__ __forceinline__ u128 multiplier() {
  return ((u128)2549297995355413924ULL << 64) | (u128)4865540595714422341ULL;
}

__host__ __device__ __forceinline__ uint64_t output(u128 s) {
  const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__host__ __device__ __forceinline__ u128 step(u128 s, u128 inc) { return s * multiplier() + inc; }

// state after `delta` LCG steps (Brown's jump-ahead)
__host__ __device__ inline u128 advance(u128 s, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = multiplier(), cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * s + acc_plus;
}

// numpy's bit-generator state as passed through the C ABI:
// {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger}
struct State {
  u128 s, inc;
  int has;
  uint32_t ub;
};

inline State load(const uint64_t* a) {
  State st;
  st.s = ((u128)a[0] << 64) | a[1];
  st.inc = ((u128)a[2] << 64) | a[3];
  st.has = a[4] != 0;
  st.ub = (uint32_t)a[5];
  return st;
}

inline void store(const State& st, uint64_t* a) {
  a[0] = (uint64_t)(st.s >> 64);
  a[1] = (uint64_t)st.s;
  a[4] = st.has ? 1u : 0u;
  a[5] = st.ub;  // numpy keeps the last high half even once consumed
}

// host: one buffered 32-bit draw (pcg64_next32)
inline uint32_t next32(State& st) {
  if (st.has) {
    st.has = 0;
    return st.ub;
  }
  st.s = step(st.s, st.inc);
  const uint64_t x = output(st.s);
  st.has = 1;
  st.ub = (uint32_t)(x >> 32);
  return (uint32_t)x;
}

// host: numpy's buffered_bounded_lemire_uint32 for range [0, m)
inline uint32_t bounded(State& st, uint32_t m, uint32_t threshold) {
  uint64_t mm = (uint64_t)next32(st) * m;
  while ((uint32_t)mm < threshold) mm = (uint64_t)next32(st) * m;
  return (uint32_t)(mm >> 32);
}

constexpr int kChunk = 32;  // 64-bit outputs per thread

// out[j] = lo + range * ((x_j >> 11) * 2^-53), x_j = output after j+1 steps
__global__ void k_uniform(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, int64_t n, double lo,
                          double range, double* __restrict__ out) {
  const u128 s0 = ((u128)s_hi << 64) | s_lo, inc = ((u128)i_hi << 64) | i_lo;
  const int64_t n_chunks = (n + kChunk - 1) / kChunk;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_chunks; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j0 = c * kChunk;
    u128 s = advance(s0, inc, (uint64_t)j0);
    for (int i = 0; i < kChunk && j0 + i < n; ++i) {
      s = step(s, inc);
      const double u = __dmul_rn((double)(output(s) >> 11), 1.0 / 9007199254740992.0);
      out[j0 + i] = __dadd_rn(lo, __dmul_rn(range, u));
    }
  }
}

// Lemire candidates over the buffered 32-bit stream.  Candidate q is the q-th
// 32-bit draw: with a buffered half (has) q = 0 is `ub` and q >= 1 maps to
// half (q-1)&1 of output (q-1)>>1; otherwise half q&1 of output q>>1.
__global__ void k_lemire_candidates(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, int has, uint32_t ub,
                                    int64_t n_cand, uint32_t m, uint32_t threshold, int32_t* __restrict__ val,
                                    uint8_t* __restrict__ ok) {
  const u128 s0 = ((u128)s_hi << 64) | s_lo, inc = ((u128)i_hi << 64) | i_lo;
  const int64_t base = has ? 1 : 0;
  const int64_t n_out = (n_cand - base + 1) / 2;
  const int64_t n_chunks = (n_out + kChunk - 1) / kChunk;
  auto emit = [&](int64_t q, uint32_t u) {
    if (q >= n_cand) return;
    const uint64_t mm = (uint64_t)u * m;
    val[q] = (int32_t)(mm >> 32);
    ok[q] = (uint32_t)mm >= threshold;
  };
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid == 0 && has) emit(0, ub);
  for (int64_t c = tid; c < n_chunks; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o0 = c * kChunk;
    u128 s = advance(s0, inc, (uint64_t)o0);
    for (int i = 0; i < kChunk && o0 + i < n_out; ++i) {
      s = step(s, inc);
      const uint64_t x = output(s);
      const int64_t q = base + 2 * (o0 + i);
      emit(q, (uint32_t)x);
      emit(q + 1, (uint32_t)(x >> 32));
    }
  }
}

// 1 where a pick equals its row or one of the row's nn ids (engine.py:141-145)
__global__ void k_pick_collisions(const int32_t* __restrict__ picks, int64_t m, int rn, const int32_t* __restrict__ nn,
                                  int64_t nn_stride, int ncols, uint8_t* __restrict__ bad) {
  const int64_t n = m * rn;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = k / rn;
    const int32_t p = picks[k];
    bool b = p == (int32_t)row;
    for (int c = 0; c < ncols; ++c) b |= p == nn[row * nn_stride + c];
    bad[k] = b;
  }
}

}  // namespace pcg
}  // namespace ivhd
