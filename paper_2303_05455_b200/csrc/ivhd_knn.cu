// ivhd_knn.cu — exact kNN graph construction on B200.
//
// Replaces knng.build_exact_knn (/root/reference/pkg/src/ivhd/knng.py:158-194)
// for the "euclidean" and "cosine" metrics: every row's k nearest other rows,
// ordered by (distance, index) — on exact distance ties the smaller index wins
// (knng.py:1-6, _row_topk knng.py:122-155).
//
// Three kernels:
//   1. k_pack      fp64 rows -> tf32-rounded fp32 tiles in the tcgen05
//                  canonical K-major no-swizzle layout (one contiguous image
//                  per 128-row tile and 32-float K chunk, so every shared-memory
//                  fill is ONE cp.async.bulk), plus fp32 squared norms.
//   2. k_knn_tc    candidate pass on the 5th-generation tensor cores: a CTA
//                  owns 128 queries and streams every 128-row candidate tile;
//                  tcgen05.mma (kind::tf32, M=128 N=128, fp32 accumulators in
//                  TMEM, double buffered) computes the 128x128 dot products,
//                  four epilogue warps read them back with tcgen05.ld and keep
//                  each query's KMAX smallest approximate squared distances.
//                  Warp roles: 0 = TMA producer, 1 = MMA issuer (one lane),
//                  2..5 = epilogue (TMEM lane quarter = warp % 4).
//   3. k_rerank    exact fp64 distances to the KMAX candidates, (distance,
//                  index) order, and a certificate: the candidate pass cannot
//                  have dropped a closer row if the error-bounded lower bound
//                  of every rejected row's distance exceeds the k-th exact
//                  distance.  Uncertified rows (rare) go to
//   4. k_exact_seg fp64 brute force over all rows for that query, split
//                  into candidate segments (warp per candidate, coalesced
//                  rows), merged in segment order by k_exact_merge.
//
// No CPU fallback: every distance is computed on the GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ivhd_b200.h"

namespace knn {

constexpr int TQ = 128;       // queries per CTA (UMMA M)
#ifndef KNN_TCN
#define KNN_TCN 256
#endif
constexpr int TCN = KNN_TCN;  // candidates per tile (UMMA N): TCN/TQ consecutive 128-row images
constexpr int KC = 32;        // floats per K chunk (128 bytes per row)
constexpr int KMAX = 32;      // list slots per (epilogue group, query)
constexpr int UMAX = 128;     // union of the group lists handed to the re-rank
constexpr int NACC = 512 / TCN;  // TMEM accumulator buffers (TCN columns each; 512 columns in all)
constexpr int HALVES = TCN / TQ;
constexpr int STAGES = 4;     // smem ring depth (A chunk + B chunk per stage)
#ifndef KNN_EPI_GROUPS
#define KNN_EPI_GROUPS 4
#endif
constexpr int EG = KNN_EPI_GROUPS;       // epilogue groups: group g owns columns [g*TCN/EG, (g+1)*TCN/EG)
constexpr int THREADS = 64 + 128 * EG;   // producer warp, MMA warp, 4*EG epilogue warps
constexpr int CHUNK_BYTES = TQ * KC * 4;                // 16 KB: one 128-row image chunk
constexpr int BCHUNK_BYTES = HALVES * CHUNK_BYTES;      // candidate chunk (TCN rows)
constexpr int STAGE_BYTES = CHUNK_BYTES + BCHUNK_BYTES; // A + B chunk (query tile not resident)

// byte offset of element (r, k) inside a chunk image with kc floats per row:
// core matrices of 8 rows x 16 bytes; K-chunk stride (LBO) 128 bytes, 8-row
// group stride (SBO) kc * 32 bytes.
__host__ __device__ __forceinline__ uint32_t img_off(int r, int k, int kc) {
  return (uint32_t)((r >> 3) * (kc * 32) + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ float tf32_round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// tcgen05 helpers (PTX ISA 8.7, sm_100a)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // SWIZZLE_NONE K-major: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
  // version 1 at bit 46, base offset 0, legacy LBO mode, layout type 0.
  return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, K-major both, N, M
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ------------------------------------------------------------------ pack
// One warp per row: tf32-rounded values into the tile images of the query
// operand PA and the candidate operand PB, fp32 norm s of the rounded row.
// Two augmented columns fold the candidate norm into the MMA:
//     PA[.., n:n+2] = (1, 1),   PB[.., n:n+2] = -(h_hi, h_lo),  h = s / 2
// so each accumulator holds q.c - |c|^2 / 2 = -(d^2 - |q|^2) / 2 and the
// epilogue filter is one compare per candidate.  Padding candidate rows get
// h = +inf (never a candidate) and norm +inf.
__global__ void k_pack(const double* __restrict__ X, int64_t m, int n, int kp, int64_t m_pad,
                       float* __restrict__ PA, float* __restrict__ PB, float* __restrict__ nrm) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < m_pad; r += nw) {
    const int64_t t = r / TQ;
    const int rr = (int)(r % TQ);
    auto off = [&](int k) {
      const int c = k / KC, kk = k % KC, kc = min(KC, kp - c * KC);
      return (t * (int64_t)TQ * kp * 4 + (int64_t)c * CHUNK_BYTES + img_off(rr, kk, kc)) >> 2;
    };
    float s = 0.f;
    for (int k = lane; k < kp; k += 32) {
      const float v = (r < m && k < n) ? tf32_round((float)X[r * n + k]) : 0.f;
      s = fmaf(v, v, s);
      if (k < n || k >= n + 2) {
        PA[off(k)] = v;
        PB[off(k)] = v;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      nrm[r] = r < m ? s : INFINITY;
      const float h = r < m ? 0.5f * s : INFINITY;
      const float hi = tf32_round(h), lo = r < m ? tf32_round(h - hi) : 0.f;
      PA[off(n)] = 1.f;
      PA[off(n + 1)] = 1.f;
      PB[off(n)] = -hi;
      PB[off(n + 1)] = -lo;
    }
  }
}

// Rows scaled to unit norm (cosine metric, knng.py:105-115); a zero row sets *bad.
__global__ void k_normalize(double* __restrict__ X, int64_t m, int n, long long* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < m; r += nw) {
    double s = 0.0;
    for (int k = lane; k < n; k += 32) s = fma(X[r * n + k], X[r * n + k], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double nr = sqrt(s);
    if (nr == 0.0) {
      if (lane == 0) atomicMin(bad, (long long)r);
      continue;
    }
    for (int k = lane; k < n; k += 32) X[r * n + k] /= nr;
  }
}

// ---------------------------------------------------------- candidate pass
// RES: the query tile (all K chunks) is loaded once and stays in shared
// memory when the deepest ring still fits beside it (decided at launch from the
// shared-memory plan); otherwise each ring stage carries the query chunk next to
// the candidate chunk.
constexpr int STAGES_RES = 4;
// dynamic shared memory: [query tile (RES)] [ring] [EG x 2 x keep x TQ lists]
inline int tc_smem_bytes(bool res, int kp, int keep, int nst) {
  const int a = res ? (TQ * kp * 4 + 1023) / 1024 * 1024 : 0;
  return a + nst * (res ? BCHUNK_BYTES : STAGE_BYTES) + EG * 2 * keep * TQ * 4 + 1024;
}

__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  // producer-side wait: back off so the spin does not take issue slots from
  // the epilogue warps sharing the SM sub-partition
  uint32_t ok;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(64);
  }
}

// Rare path of the epilogue, kept out of line so the unrolled filter stays
// small enough for the instruction cache: overwrite the list maximum with
// (d2, cid), rescan for the new maximum; returns the new threshold - nq.
__device__ __noinline__ float knn_insert(float* ld, int* li, int* pm_s, int r, int keep, float d2, int cid, float nq) {
  const int pm = pm_s[r];
  ld[pm * TQ + r] = d2;
  li[pm * TQ + r] = cid;
  float mx = -INFINITY;
  int p = 0;
  for (int i = 0; i < keep; ++i) {
    const float x = ld[i * TQ + r];
    if (x > mx) {
      mx = x;
      p = i;
    }
  }
  pm_s[r] = p;
  return mx - nq;
}

template <bool RES>
__global__ void __launch_bounds__(THREADS, 1)
    k_knn_tc(const float* __restrict__ PA, const float* __restrict__ P, const float* __restrict__ nrm, int64_t m,
             int kp, int n_tiles, int keep,
             int nst, int32_t* __restrict__ cand_id, float* __restrict__ cand_d2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int NSTMAX = RES ? STAGES_RES : STAGES;
  const int NST = nst;                                  // ring depth (<= NSTMAX, sized by the host)
  constexpr int SB = RES ? BCHUNK_BYTES : STAGE_BYTES;  // bytes per ring stage
  uint8_t* aq = smem;                                   // RES: resident query tile
  uint8_t* ring = smem + (RES ? (TQ * kp * 4 + 1023) / 1024 * 1024 : 0);
  float* lst_base = reinterpret_cast<float*>(ring + NST * SB);  // [EG][2][keep][TQ]
  __shared__ __align__(8) uint64_t full[NSTMAX], empty[NSTMAX], accf[NACC], acce[NACC], abar;
  __shared__ uint32_t tmem_sh;
  __shared__ int pm_sh[EG][TQ];  // slot of each list's current maximum

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x;
  const int nchunks = (kp + KC - 1) / KC;
  const int64_t tile_floats = (int64_t)TQ * kp;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < NACC; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], 4 * EG);
    }
    mbar_init(&abar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // NACC x TCN fp32 accumulator columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_sh)),
                 "r"(NACC * TCN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    tc_fence_before();
  }
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_sh;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      const float* Aq = PA + (int64_t)qt * tile_floats;
      if constexpr (RES) {  // the whole query tile: one contiguous copy
        mbar_expect_tx(&abar, (uint32_t)(tile_floats * 4));
        bulk_g2s(aq, Aq, (uint32_t)(tile_floats * 4), &abar);
      }
      int it = 0;
      // candidate tile j = 128-row images HALVES*j .. HALVES*j+HALVES-1; their
      // chunk-c images land back to back, which is exactly the canonical
      // layout of a TCN-row operand (row group 16 starts one image later)
      for (int j = 0; j < n_tiles; ++j) {
        for (int c = 0; c < nchunks; ++c, ++it) {
          const int s = it % NST;
          if (it >= NST) mbar_wait_sleep(&empty[s], ((it / NST) - 1) & 1);
          const uint32_t bytes = (uint32_t)TQ * min(KC, kp - c * KC) * 4;
          uint8_t* st = ring + s * SB;
          uint8_t* sbp = st + (RES ? 0 : CHUNK_BYTES);
          mbar_expect_tx(&full[s], (RES ? 0u : bytes) + HALVES * bytes);
          if constexpr (!RES) bulk_g2s(st, Aq + (int64_t)c * TQ * KC, bytes, &full[s]);
          for (int h = 0; h < HALVES; ++h)
            bulk_g2s(sbp + h * bytes, P + (int64_t)(HALVES * j + h) * tile_floats + (int64_t)c * TQ * KC, bytes,
                     &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_tf32(TQ, TCN);
      if constexpr (RES) mbar_wait(&abar, 0);
      int it = 0;
      for (int j = 0; j < n_tiles; ++j) {
        const int b = j % NACC;
        if (j >= NACC) mbar_wait(&acce[b], ((j / NACC) - 1) & 1);  // epilogue drained buffer b
        tc_fence_after();
        const uint32_t dt = tbase + (uint32_t)(b * TCN);
        for (int c = 0; c < nchunks; ++c, ++it) {
          const int s = it % NST;
          mbar_wait(&full[s], (it / NST) & 1);
          tc_fence_after();
          const int kc = min(KC, kp - c * KC);
          const uint32_t sr = smem_u32(ring + s * SB);
          const uint32_t sa = RES ? smem_u32(aq) + (uint32_t)(c * CHUNK_BYTES) : sr;
          const uint32_t sb = RES ? sr : sr + CHUNK_BYTES;
#ifndef KNN_SKIP_MMA
          for (int ks = 0; ks < kc / 8; ++ks) {
#else
          for (int ks = 0; ks < 0; ++ks) {
#endif
            const uint64_t ad = umma_desc(sa + ks * 256, 128, (uint32_t)kc * 32);
            const uint64_t bd = umma_desc(sb + ks * 256, 128, (uint32_t)kc * 32);
            umma_tf32(dt, ad, bd, idesc, (c | ks) != 0);
          }
          umma_commit(&empty[s]);  // stage free once these MMAs have read it
        }
        umma_commit(&accf[b]);  // accumulator b complete
      }
    }
  } else {
    // --------------------------------------------------------- epilogue
    // 4*EG warps: warp w reads TMEM lane quarter w % 4 (queries 32q..32q+31)
    // and, in group g, columns [g*CG, (g+1)*CG) of every tile; each (group,
    // query) keeps an unsorted list of its `keep` smallest approximate squared
    // distances with the current maximum tracked (insert = overwrite the max,
    // rescan).  Several warps per SM sub-partition hide the TMEM/branch latency.
    constexpr int CG = TCN / EG;
    const int ew = warp - 2, g = ew >> 2, q = warp & 3;
    const int r = q * 32 + lane;
    const int64_t qid = (int64_t)qt * TQ + r;
    const float nq = qid < m ? nrm[qid] : 0.f;
    float* ld = lst_base + (size_t)g * 2 * keep * TQ;
    int* li = reinterpret_cast<int*>(ld + keep * TQ);
    for (int i = 0; i < keep; ++i) {
      ld[i * TQ + r] = INFINITY;
      li[i * TQ + r] = 0x7fffffff;
    }
    int* pm_s = pm_sh[g];
    pm_s[r] = 0;
    float thq = INFINITY;  // list maximum - nq: a candidate passes if nc - 2 dot < thq
    for (int j = 0; j < n_tiles; ++j) {
      const int b = j % NACC;
      mbar_wait(&accf[b], (j / NACC) & 1);
      tc_fence_after();
      const bool diag = j == qt / HALVES;  // the only tile holding the query itself
#pragma unroll 1
      for (int h = 0; h < CG / 32; ++h) {
        uint32_t v[32];
        tmem_ld32(tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * TCN + g * CG + h * 32), v);
        if (h == CG / 32 - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acce[b]);
        }
        const int c0 = j * TCN + g * CG + h * 32;
#ifdef KNN_SKIP_EPI
        if (v[0] == 0x7fffffffu && v[31] == 0x7fffffffu) ld[r] = 0.f;
        continue;
#endif
        // fast pass, one compare per candidate: acc = q.c - |c|^2/2 and
        // d^2 - nq = -2 acc < thq  <=>  acc > -thq/2
        const float thh = -0.5f * thq;
        // any candidate above the threshold?  a max tree first (3-input FMNMX:
        // ~16 instructions for 32 values, against a compare + select each)
        float mx = __uint_as_float(v[0]);
#pragma unroll
        for (int i = 1; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(v[i]));
        unsigned msk = 0;
        if (mx > thh) {
#pragma unroll
          for (int i = 0; i < 32; ++i) msk |= __uint_as_float(v[i]) > thh ? (1u << i) : 0u;
        }
        if (msk) {  // rare: re-test in order against the moving threshold, insert
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            if ((msk >> i) & 1u) {
              const float t = -2.f * __uint_as_float(v[i]);  // d2 - nq
              if (t < thq && !(diag && c0 + i == (int)qid))
                thq = knn_insert(ld, li, pm_s, r, keep, t + nq, c0 + i, nq);
            }
          }
        }
      }
    }
    // hand-off: group 0 writes the union of the EG lists (EG * keep <= UMAX
    // entries) and the certificate threshold T = min over groups of the
    // group's final maximum: every rejected row had d2 >= its group's maximum.
    asm volatile("barrier.sync 1, %0;" ::"r"(128 * EG) : "memory");
    if (g == 0 && qid < m) {
      float T = INFINITY;
      int o = 0;
      for (int gg = 0; gg < EG; ++gg) {
        const float* gd = lst_base + (size_t)gg * 2 * keep * TQ;
        const int* gi = reinterpret_cast<const int*>(gd + keep * TQ);
        float mx = -INFINITY;
        for (int i = 0; i < keep; ++i, ++o) {
          const float x = gd[i * TQ + r];
          const int xi = gi[i * TQ + r];
          mx = fmaxf(mx, x);
          cand_id[qid * UMAX + o] = xi == 0x7fffffff ? -1 : xi;
        }
        T = fminf(T, mx);
      }
      for (; o < UMAX; ++o) cand_id[qid * UMAX + o] = -1;
      cand_d2[qid] = T;
    }
  }
  // non-aligned barrier: the producer and MMA warps arrive diverged (lane 0 ran the loop)
  asm volatile("barrier.sync 0;" ::: "memory");
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(NACC * TCN) : "memory");
  }
}

// --------------------------------------------------------------- re-rank
// Exact fp64 distance between rows a and b (euclidean: sqrt of the summed
// squared differences; cosine on unit rows: max(1 - dot, 0), knng.py:185-189).
__device__ __forceinline__ double exact_dist(const double* __restrict__ X, int n, int64_t a, int64_t b, int metric) {
  const double* xa = X + a * n;
  const double* xb = X + b * n;
  double s = 0.0;
  if (metric == 0) {
    for (int k = 0; k < n; ++k) {
      const double d = xa[k] - xb[k];
      s = fma(d, d, s);
    }
    return sqrt(s);
  }
  for (int k = 0; k < n; ++k) s = fma(xa[k], xb[k], s);
  return fmax(1.0 - s, 0.0);
}

__device__ __forceinline__ bool before(double da, int ia, double db, int ib) {
  return da < db || (da == db && ia < ib);
}

// One warp per query: lane i re-scores candidate i in fp64, ranks by
// (distance, index), writes the first k, and certifies the result.
__global__ void k_rerank(const double* __restrict__ X, int64_t m, int n, int metric, int k, int n_union,
                         const int32_t* __restrict__ cand_id, const float* __restrict__ cand_d2,
                         const float* __restrict__ nrm, float rmax, float gamma, float eps_in,
                         int32_t* __restrict__ out_id, double* __restrict__ out_d, int* __restrict__ flag) {
  constexpr int CPL = UMAX / 32;  // candidates per lane
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t qy = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; qy < m; qy += nw) {
    int id[CPL];
    double d[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      id[c] = cand_id[qy * UMAX + c * 32 + lane];
      d[c] = INFINITY;
      if (id[c] >= 0) d[c] = exact_dist(X, n, qy, id[c], metric);
      else id[c] = 0x7fffffff;
    }
    int rank[CPL] = {};
    for (int c2 = 0; c2 < CPL; ++c2) {
      if (c2 * 32 >= n_union) break;
      for (int o = 0; o < 32; ++o) {
        const double od = __shfl_sync(0xffffffffu, d[c2], o);
        const int oi = __shfl_sync(0xffffffffu, id[c2], o);
#pragma unroll
        for (int c = 0; c < CPL; ++c) rank[c] += before(od, oi, d[c], id[c]) ? 1 : 0;
      }
    }
    double dk = 0.0;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      if (rank[c] < k) {
        out_id[qy * k + rank[c]] = id[c];
        out_d[qy * k + rank[c]] = d[c];
      }
      if (rank[c] == k - 1) dk = d[c];
    }
    // certificate: every row outside the union had approximate squared
    // distance >= T; its true distance is at least
    //   sqrt(max(T - gamma (|q~| + R)^2, 0)) - eps_in (|q| + R)
    // (gamma: fp32 Gram-expansion error, eps_in: tf32 input rounding).
    bool have = false;
#pragma unroll
    for (int c = 0; c < CPL; ++c) have |= rank[c] == k - 1;
    const unsigned who = __ballot_sync(0xffffffffu, have);
    dk = __shfl_sync(0xffffffffu, dk, __ffs(who) - 1);
    if (lane == 0) {
      bool ok = true;
      if (m - 1 > (int64_t)n_union) {
        const double T = (double)cand_d2[qy];
        const double qn = sqrt((double)nrm[qy]) * (1.0 + 1e-6);
        const double s = qn + (double)rmax;
        const double lb = sqrt(fmax(T - (double)gamma * s * s, 0.0)) - (double)eps_in * s;
        double dke = dk;
        if (metric == 1) dke = sqrt(2.0 * dk);  // cosine distance -> unit-row euclidean
        ok = isfinite(T) && lb > dke;
      }
      if (!ok) flag[qy] = 1;
    }
  }
}

// ------------------------------------------------------------ exact scan
// Rows the certificate does not cover (and every row when the tensor-core
// pass does not apply): exact fp64 scan split into segments of candidates.
// Block (query i, segment s): each warp takes candidates c = seg0 + warp,
// +8, ...; the lanes read the row coalesced and reduce the distance with a
// fixed butterfly; lane 0 keeps the warp's sorted (distance, index) list;
// the 8 warp lists are merged into the segment's top k (scratch), and
// k_exact_merge merges the segments of a query in segment order.
constexpr int EX_THREADS = 256;
constexpr int EX_WARPS = EX_THREADS / 32;
constexpr int EX_K = 64;

__global__ void __launch_bounds__(EX_THREADS) k_exact_seg(const double* __restrict__ X, int64_t m, int n, int metric,
                                                         int k, const int* __restrict__ list, int n_list, int n_seg,
                                                         double* __restrict__ sd_out, int* __restrict__ si_out) {
  extern __shared__ __align__(16) unsigned char exs[];
  double* wd = reinterpret_cast<double*>(exs);           // [EX_WARPS][k]
  int* wi = reinterpret_cast<int*>(wd + EX_WARPS * k);   // [EX_WARPS][k]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qi = blockIdx.x / n_seg, seg = blockIdx.x % n_seg;
  if (qi >= n_list) return;
  const int64_t qy = list[qi];
  const int64_t per = (m + n_seg - 1) / n_seg, c_lo = seg * per, c_hi = min(m, c_lo + per);
  double* md = wd + warp * k;
  int* mi = wi + warp * k;
  if (lane == 0)
    for (int i = 0; i < k; ++i) {
      md[i] = INFINITY;
      mi[i] = 0x7fffffff;
    }
  __syncwarp();
  const double* xq = X + qy * n;
  for (int64_t c = c_lo + warp; c < c_hi; c += EX_WARPS) {
    const double* xc = X + c * n;
    double s = 0.0;
    if (metric == 0) {
      for (int t = lane; t < n; t += 32) {
        const double d = xq[t] - xc[t];
        s = fma(d, d, s);
      }
    } else {
      for (int t = lane; t < n; t += 32) s = fma(xq[t], xc[t], s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double d = metric == 0 ? sqrt(s) : fmax(1.0 - s, 0.0);
    if (lane == 0 && c != qy && before(d, (int)c, md[k - 1], mi[k - 1])) {
      int p = k - 1;
      while (p > 0 && before(d, (int)c, md[p - 1], mi[p - 1])) {
        md[p] = md[p - 1];
        mi[p] = mi[p - 1];
        --p;
      }
      md[p] = d;
      mi[p] = (int)c;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // merge the warp lists (k-way, fixed order)
    int pos[EX_WARPS] = {};
    double* od = sd_out + ((int64_t)qi * n_seg + seg) * k;
    int* oi = si_out + ((int64_t)qi * n_seg + seg) * k;
    for (int o = 0; o < k; ++o) {
      int bw = 0;
      for (int w = 1; w < EX_WARPS; ++w)
        if (before(wd[w * k + pos[w]], wi[w * k + pos[w]], wd[bw * k + pos[bw]], wi[bw * k + pos[bw]])) bw = w;
      od[o] = wd[bw * k + pos[bw]];
      oi[o] = wi[bw * k + pos[bw]];
      if (pos[bw] < k - 1) ++pos[bw];
      else wd[bw * k + pos[bw]] = INFINITY, wi[bw * k + pos[bw]] = 0x7fffffff;
    }
  }
}

// One thread per flagged query: merge its n_seg sorted segment lists.
__global__ void k_exact_merge(const int* __restrict__ list, int n_list, int n_seg, int k,
                              double* __restrict__ sd, int* __restrict__ si, int32_t* __restrict__ out_id,
                              double* __restrict__ out_d) {
  const int qi = blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= n_list) return;
  const int64_t qy = list[qi];
  double* d = sd + (int64_t)qi * n_seg * k;
  int* id = si + (int64_t)qi * n_seg * k;
  // repeated selection of the smallest segment head; heads advance in place
  for (int o = 0; o < k; ++o) {
    int bs = 0;
    for (int sg = 1; sg < n_seg; ++sg)
      if (before(d[sg * k], id[sg * k], d[bs * k], id[bs * k])) bs = sg;
    out_id[qy * k + o] = id[bs * k];
    out_d[qy * k + o] = d[bs * k];
    for (int i = 0; i < k - 1; ++i) {  // pop the head of segment bs
      d[bs * k + i] = d[bs * k + i + 1];
      id[bs * k + i] = id[bs * k + i + 1];
    }
    d[bs * k + k - 1] = INFINITY;
    id[bs * k + k - 1] = 0x7fffffff;
  }
}

// metric "precomputed" (knng.py:175-181, _row_topk knng.py:122-155): the k
// smallest entries of every row of a dense (m, m) distance matrix, self
// excluded, by (value, index).  One warp per row streams it coalesced; the
// row's current k best live in registers across the lanes (slot s = lane +
// 32 j, sorted), candidates that beat the k-th enter one at a time (warp
// ballot), so each row costs one pass over its m values.
constexpr int PK_MAX = 128;
__global__ void __launch_bounds__(256) k_topk_rows(const double* __restrict__ D, int64_t m, int k,
                                                  int32_t* __restrict__ out_id, double* __restrict__ out_d) {
  constexpr int SPL = PK_MAX / 32;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < m; r += nw) {
    double ld[SPL];
    int li[SPL];
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
      ld[j] = INFINITY;
      li[j] = 0x7fffffff;
    }
    double thr = INFINITY;
    int thr_i = 0x7fffffff;
    int cnt = 0;
    const double* row = D + r * m;
    for (int64_t c0 = 0; c0 < m; c0 += 32) {
      const int64_t c = c0 + lane;
      double d = INFINITY;
      int id = 0x7fffffff;
      if (c < m && c != r) {
        d = row[c];
        id = (int)c;
      }
      unsigned pass = __ballot_sync(0xffffffffu, id != 0x7fffffff && (cnt < k || before(d, id, thr, thr_i)));
      while (pass) {
        const int src = __ffs(pass) - 1;
        pass &= pass - 1;
        const double nd = __shfl_sync(0xffffffffu, d, src);
        const int ni = __shfl_sync(0xffffffffu, id, src);
        if (!(cnt < k || before(nd, ni, thr, thr_i))) continue;
        int bef = 0;
#pragma unroll
        for (int j = 0; j < SPL; ++j) bef += before(ld[j], li[j], nd, ni) ? 1 : 0;
        const int pos = __reduce_add_sync(0xffffffffu, bef);
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
          const int sl = lane + 32 * j;
          if (sl > pos) {
            ld[j] = pd;
            li[j] = pi;
          } else if (sl == pos) {
            ld[j] = nd;
            li[j] = ni;
          }
        }
        cnt = min(cnt + 1, k);
        const int ts = k - 1;
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
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
      const int sl = lane + 32 * j;
      if (sl < k) {
        out_id[r * k + sl] = li[j];
        out_d[r * k + sl] = ld[j];
      }
    }
  }
}

__global__ void k_flag_list(const int* __restrict__ flag, int64_t m, int* __restrict__ list, int* __restrict__ cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m && flag[i]) list[atomicAdd(cnt, 1)] = (int)i;
}

__global__ void k_max_norm(const float* __restrict__ nrm, int64_t m, unsigned int* __restrict__ out) {
  float mx = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    mx = fmaxf(mx, nrm[i]);
  atomicMax(out, __float_as_uint(mx));  // non-negative floats order like their bits
}

thread_local std::string g_knn_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_knn_error = buf;
  return code;
}

}  // namespace knn

using namespace knn;

extern "C" {

const char* ivhd_knn_last_error(void) { return g_knn_error.c_str(); }

int ivhd_knn_build(int device, const double* x, int64_t m, int32_t n, int32_t k, int32_t metric,
                   int32_t* nbr_out, double* dist_out, double* stats_out) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  if (!x || !nbr_out || !dist_out) return fail(IVHD_ERR_INVALID_ARG, "null pointer");
  if (!(1 <= k && k < m)) return fail(IVHD_ERR_INVALID_ARG, "k must satisfy 1 <= k < M, got k=%d, M=%lld", k, (long long)m);
  if (n < 1) return fail(IVHD_ERR_INVALID_ARG, "need at least one feature column");
  if (metric < 0 || metric > 2)
    return fail(IVHD_ERR_INVALID_ARG, "metric must be euclidean (0), cosine (1) or precomputed (2)");
  if (metric == 2) {  // x is an (m, m) distance matrix (n must equal m)
    if (n != m) return fail(IVHD_ERR_INVALID_ARG, "precomputed metric needs a square matrix");
    if (k > PK_MAX) return fail(IVHD_ERR_INVALID_ARG, "k=%d above the supported %d", k, PK_MAX);
    if (cudaSetDevice(device) != cudaSuccess) return fail(IVHD_ERR_CUDA, "cudaSetDevice(%d) failed", device);
    cudaStream_t st;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return fail(IVHD_ERR_CUDA, "stream");
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double *dD = nullptr, *dd = nullptr;
    int32_t* di = nullptr;
    cudaError_t e = cudaSuccess;
    do {
      if ((e = cudaMallocAsync(&dD, sizeof(double) * m * m, st)) != cudaSuccess) break;
      if ((e = cudaMallocAsync(&dd, sizeof(double) * m * k, st)) != cudaSuccess) break;
      if ((e = cudaMallocAsync(&di, sizeof(int32_t) * m * k, st)) != cudaSuccess) break;
      if ((e = cudaMemcpyAsync(dD, x, sizeof(double) * m * m, cudaMemcpyHostToDevice, st)) != cudaSuccess) break;
      k_topk_rows<<<(unsigned)std::min<int64_t>((m + 7) / 8, (int64_t)sms * 16), 256, 0, st>>>(dD, m, k, di, dd);
      if ((e = cudaGetLastError()) != cudaSuccess) break;
      if ((e = cudaMemcpyAsync(nbr_out, di, sizeof(int32_t) * m * k, cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
      if ((e = cudaMemcpyAsync(dist_out, dd, sizeof(double) * m * k, cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
      e = cudaStreamSynchronize(st);
    } while (0);
    if (dD) cudaFreeAsync(dD, st);
    if (dd) cudaFreeAsync(dd, st);
    if (di) cudaFreeAsync(di, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    if (e != cudaSuccess) return fail(IVHD_ERR_CUDA, "kNN (precomputed): %s", cudaGetErrorString(e));
    if (stats_out)
      for (int i = 0; i < 8; ++i) stats_out[i] = 0.0;
    return IVHD_OK;
  }
  if (m >= 0x7fffffffLL) return fail(IVHD_ERR_INVALID_ARG, "M too large for 31-bit ids");
  if (k > EX_K) return fail(IVHD_ERR_INVALID_ARG, "k=%d above the supported %d", k, EX_K);
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

  const int kp = (n + 2 + 7) / 8 * 8;  // features + 2 augmented norm columns, K steps of 8
  // query tiles of TQ rows; candidate tiles of TCN rows (padding rows have
  // norm +inf and are never candidates)
  const int64_t n_tiles = (m + TQ - 1) / TQ, m_pad = (m + TCN - 1) / TCN * TCN, n_ctiles = m_pad / TCN;
  // candidates kept per query by the tensor-core pass; beyond KMAX-8 (or for
  // tiny inputs) every query goes to the exact scan
  const bool tc = k + 4 <= std::min(KMAX, UMAX / EG) && m > 2 * (int64_t)UMAX;
  // candidates kept per query and epilogue group (each group sees 1/EG of the
  // rows): the union of the EG lists is re-ranked, so a group needs only a
  // share of k plus slack; the insert cost grows ~keep^2
  const int keep = tc ? std::min(std::min(KMAX, UMAX / EG), k + 4) : 0;

  double *dX = nullptr, *dD = nullptr;
  float *dP = nullptr, *dPA = nullptr, *dN = nullptr, *cd2 = nullptr;
  int32_t *dI = nullptr, *cid = nullptr;
  int *flag = nullptr, *list = nullptr, *cnt = nullptr;
  long long* bad = nullptr;
  unsigned int* rmax_bits = nullptr;
  double* xsd = nullptr;
  int* xsi = nullptr;
  int rc = IVHD_OK;
  int n_fallback = 0;
  double t_tc = 0, t_rr = 0, t_setup = 0, t_ex = 0, t_d2h = 0;
  cudaError_t e = cudaSuccess;
  do {
#define KTRY(call) \
  if ((e = (call)) != cudaSuccess) break
    KTRY(cudaMallocAsync(&dX, sizeof(double) * m * n, st));
    KTRY(cudaMallocAsync(&dI, sizeof(int32_t) * m * k, st));
    KTRY(cudaMallocAsync(&dD, sizeof(double) * m * k, st));
    KTRY(cudaMallocAsync(&flag, sizeof(int) * m, st));
    KTRY(cudaMallocAsync(&list, sizeof(int) * m, st));
    KTRY(cudaMallocAsync(&cnt, sizeof(int), st));
    KTRY(cudaMallocAsync(&bad, sizeof(long long), st));
    KTRY(cudaMemcpyAsync(dX, x, sizeof(double) * m * n, cudaMemcpyHostToDevice, st));
    KTRY(cudaMemsetAsync(flag, 0, sizeof(int) * m, st));
    KTRY(cudaMemsetAsync(cnt, 0, sizeof(int), st));
    const long long big = 0x7fffffffffffffffLL;
    KTRY(cudaMemcpyAsync(bad, &big, sizeof big, cudaMemcpyHostToDevice, st));
    if (metric == 1) {
      k_normalize<<<sms * 8, 256, 0, st>>>(dX, m, n, bad);
      long long hb = big;
      KTRY(cudaMemcpyAsync(&hb, bad, sizeof hb, cudaMemcpyDeviceToHost, st));
      KTRY(cudaStreamSynchronize(st));
      if (hb != big) {
        rc = fail(IVHD_ERR_INVALID_ARG, "zero-norm vector under cosine metric (row %lld)", hb);
        break;
      }
    }
    if (tc) {
      KTRY(cudaMallocAsync(&dP, sizeof(float) * m_pad * kp, st));
      KTRY(cudaMallocAsync(&dPA, sizeof(float) * m_pad * kp, st));
      KTRY(cudaMallocAsync(&dN, sizeof(float) * m_pad, st));
      KTRY(cudaMallocAsync(&cid, sizeof(int32_t) * m * UMAX, st));
      KTRY(cudaMallocAsync(&cd2, sizeof(float) * m, st));
      KTRY(cudaMallocAsync(&rmax_bits, sizeof(unsigned int), st));
      KTRY(cudaMemsetAsync(rmax_bits, 0, sizeof(unsigned int), st));
      k_pack<<<sms * 16, 256, 0, st>>>(dX, m, n, kp, m_pad, dPA, dP, dN);
      k_max_norm<<<sms, 256, 0, st>>>(dN, m, rmax_bits);
      unsigned int hr = 0;
      KTRY(cudaMemcpyAsync(&hr, rmax_bits, sizeof hr, cudaMemcpyDeviceToHost, st));
      int smem_max = 0;
      cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
      cudaFuncAttributes fa{};
      KTRY(cudaFuncGetAttributes(&fa, k_knn_tc<true>));
      smem_max -= (int)fa.sharedSizeBytes;  // static shared memory of the kernel
      // query tile resident if the deepest ring still fits; otherwise streamed
      int nst = STAGES_RES;
      bool res = true;
      while (nst > 2 && tc_smem_bytes(true, kp, keep, nst) > smem_max) --nst;
      if (tc_smem_bytes(true, kp, keep, nst) > smem_max) {
        res = false;
        nst = STAGES;
        while (nst > 2 && tc_smem_bytes(false, kp, keep, nst) > smem_max) --nst;
      }
      const int shb = tc_smem_bytes(res, kp, keep, nst);
      if (shb > smem_max) {
        rc = fail(IVHD_ERR_INVALID_ARG, "kNN: shared memory plan %d > %d bytes", shb, smem_max);
        break;
      }
      KTRY(cudaFuncSetAttribute(k_knn_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
      KTRY(cudaFuncSetAttribute(k_knn_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
      KTRY(cudaStreamSynchronize(st));
      const auto a = clk::now();
      t_setup = std::chrono::duration<double>(a - t0).count();
      if (res)
        k_knn_tc<true><<<(unsigned)n_tiles, THREADS, shb, st>>>(dPA, dP, dN, m, kp, (int)n_ctiles, keep, nst, cid,
                                                                cd2);
      else
        k_knn_tc<false><<<(unsigned)n_tiles, THREADS, shb, st>>>(dPA, dP, dN, m, kp, (int)n_ctiles, keep, nst, cid,
                                                                 cd2);
      KTRY(cudaGetLastError());
      KTRY(cudaStreamSynchronize(st));
      const auto b = clk::now();
      t_tc = std::chrono::duration<double>(b - a).count();
      float hrf;
      memcpy(&hrf, &hr, sizeof hrf);
      float rmax = sqrtf(hrf) * (1.f + 1e-6f);
      if (metric == 1) rmax = 1.f + 1e-6f;
      // error model (see k_rerank): fp32 sums of kp terms, generous factor 8
      const float gamma = 8.f * (float)(kp + 8) * 5.96e-8f;
      const float eps_in = 4.9e-4f;  // 2^-11 relative tf32 rounding, per coordinate
      k_rerank<<<sms * 8, 256, 0, st>>>(dX, m, n, metric, k, keep * EG, cid, cd2, dN, rmax, gamma, eps_in, dI, dD, flag);
      KTRY(cudaGetLastError());
      KTRY(cudaStreamSynchronize(st));
      t_rr = std::chrono::duration<double>(clk::now() - b).count();
    } else {
      KTRY(cudaMemsetAsync(flag, 1, sizeof(int) * m, st));  // nonzero bytes: every row flagged
    }
    k_flag_list<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(flag, m, list, cnt);
    KTRY(cudaMemcpyAsync(&n_fallback, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
    KTRY(cudaStreamSynchronize(st));
    const auto tx0 = clk::now();
    if (n_fallback > 0) {
      // segments per query: fill the GPU (>= 4 blocks per SM), segments of
      // at least 256 rows; processed in batches bounding the scratch size
      int n_seg = (int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, (4LL * sms + n_fallback - 1) / n_fallback));
      const int batch = std::max(1, std::min(n_fallback, (int)((256LL << 20) / ((int64_t)n_seg * k * 12))));
      KTRY(cudaMallocAsync(&xsd, sizeof(double) * (size_t)batch * n_seg * k, st));
      KTRY(cudaMallocAsync(&xsi, sizeof(int) * (size_t)batch * n_seg * k, st));
      const size_t shb = (size_t)EX_WARPS * k * 12;
      for (int b0 = 0; b0 < n_fallback; b0 += batch) {
        const int nb = std::min(batch, n_fallback - b0);
        k_exact_seg<<<(unsigned)(nb * n_seg), EX_THREADS, shb, st>>>(dX, m, n, metric, k, list + b0, nb, n_seg, xsd, xsi);
        k_exact_merge<<<(nb + 127) / 128, 128, 0, st>>>(list + b0, nb, n_seg, k, xsd, xsi, dI, dD);
        KTRY(cudaGetLastError());
      }
      KTRY(cudaStreamSynchronize(st));
    }
    t_ex = std::chrono::duration<double>(clk::now() - tx0).count();
    const auto td0 = clk::now();
    KTRY(cudaMemcpyAsync(nbr_out, dI, sizeof(int32_t) * m * k, cudaMemcpyDeviceToHost, st));
    KTRY(cudaMemcpyAsync(dist_out, dD, sizeof(double) * m * k, cudaMemcpyDeviceToHost, st));
    KTRY(cudaStreamSynchronize(st));
    t_d2h = std::chrono::duration<double>(clk::now() - td0).count();
#undef KTRY
  } while (0);
  cudaFreeAsync(dX, st); cudaFreeAsync(dI, st); cudaFreeAsync(dD, st); cudaFreeAsync(flag, st);
  cudaFreeAsync(list, st); cudaFreeAsync(cnt, st); cudaFreeAsync(bad, st);
  if (dP) cudaFreeAsync(dP, st);
  if (dPA) cudaFreeAsync(dPA, st);
  if (dN) cudaFreeAsync(dN, st);
  if (cid) cudaFreeAsync(cid, st);
  if (cd2) cudaFreeAsync(cd2, st);
  if (rmax_bits) cudaFreeAsync(rmax_bits, st);
  if (xsd) cudaFreeAsync(xsd, st);
  if (xsi) cudaFreeAsync(xsi, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (rc != IVHD_OK) return rc;
  if (e != cudaSuccess) return fail(IVHD_ERR_CUDA, "kNN build: %s", cudaGetErrorString(e));
  if (stats_out) {
    stats_out[0] = t_tc;
    stats_out[1] = t_rr;
    stats_out[2] = (double)n_fallback;
    stats_out[3] = std::chrono::duration<double>(clk::now() - t0).count();
    stats_out[4] = t_setup;
    stats_out[5] = t_ex;
    stats_out[6] = t_d2h;
    stats_out[7] = 0.0;
  }
  return IVHD_OK;
}

}  // extern "C"
