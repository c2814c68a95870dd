// ivhd_step_f64.cuh — the IVHD iteration in float64, used for Adam.
//
// Adam (optim.py:178-205) divides the bias-corrected first moment by the
// root of the second one, so a gradient component that nearly cancels keeps
// an O(alpha) step whose value depends on the component's relative error:
// with fp32 positions and forces that error reaches ~1e-7 absolute and the
// step after it 3e-5 (round 1).  This variant keeps positions, optimizer
// state, the per-entry force terms and their sums in float64 like the
// reference, which brings Adam to the same 1e-5 per-iteration parity as the
// other optimizers.  Adam is not a throughput configuration (BASELINE.json
// configs use force-directed, Adadelta and Nesterov), so the kernel is the
// plain form: one thread per vertex walks its symmetrised-CSR row, blocks
// take 256-vertex tiles round robin (fixed grid => fixed summation order).
//
// Layout: positions double[DIM == 2 ? 2 : 4] per vertex (the fp32 buffers'
// 16/32-byte strides), state double {v[DP], s[DP]} with DP = 2 or 4.
#pragma once
#include "ivhd_step.cuh"

namespace ivhd {

template <int DIM>
struct F64Layout {
  static constexpr int DP = DIM == 2 ? 2 : 4;  // doubles per position (padded)
  static constexpr int YS = 2 * DP;             // in floats (ys_of for Adam)
  static constexpr int SD = 2 * DP;             // state doubles: v then s
};

__device__ __forceinline__ uint32_t ld_col_nc(const uint32_t* p) { return __ldg(p); }

// contribution of one entry in float64 (forces.py:97-124, same branches)
template <int DIM, int NORM>
__device__ __forceinline__ bool entry_f64(const double (&yi)[DIM], const double (&yo)[DIM], double t, double w,
                                          double (&f)[DIM], double& e) {
  double df[DIM], d2 = 0.0, d1 = 0.0;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    df[d] = yi[d] - yo[d];
    d2 += df[d] * df[d];
    d1 += fabs(df[d]);
  }
  if constexpr (NORM == 0) {
    const double dist = sqrt(d2);
    const double r = t - dist;
    e += w * r * r;
    if (t == 0.0) {
#pragma unroll
      for (int d = 0; d < DIM; ++d) f[d] -= w * df[d];
      return false;
    }
    if (dist == 0.0) return true;  // degenerate random pair: caller adds the unit direction
    const double phi = w * (t - dist) / dist;
#pragma unroll
    for (int d = 0; d < DIM; ++d) f[d] += phi * df[d];
    return false;
  } else {
    const double s = w * (t - d1);
    e += w * (t - d1) * (t - d1);
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const double sg = df[d] > 0.0 ? 1.0 : (df[d] < 0.0 ? -1.0 : 0.0);
      f[d] += sg * s;
    }
    return false;
  }
}

template <int DIM, bool WEIGHTED, int NORM>
__global__ void __launch_bounds__(kBlock) step_kernel_f64(StepArgs A) {
  using FL = F64Layout<DIM>;
  __shared__ double4 sm_red[kBlock / 32];
  Ctrl* ctrl = A.ctrl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) griddep_launch_dependents();
  griddep_wait();
  if (ctrl->status != 0) return;
  const int ycur = A.fixed_io ? 0 : ctrl->cur;
  const double* __restrict__ Yin = reinterpret_cast<const double*>(ycur ? A.ybuf1 : A.ybuf0);
  double* __restrict__ Yout = reinterpret_cast<double*>(ycur ? A.ybuf0 : A.ybuf1);
  const double* __restrict__ Sin = reinterpret_cast<const double*>(A.state + (ctrl->scur ? A.sstride : 0));
  double* __restrict__ Sout = reinterpret_cast<double*>(A.state + (ctrl->scur ? 0 : A.sstride));
  const double c = ctrl->c, alpha = ctrl->step;
  const long long gstep = ctrl->gstep;
  const double tt = (double)(ctrl->adam_t + 1);
  const double bc1 = 1.0 - pow(A.h.gv_d, tt), bc2 = 1.0 - pow(A.h.gs_d, tt);  // optim.py:201-202

  // tiles [t_lo, t_hi): the whole graph (fused) or this rank's range (sharded)
  const int t_lo = (int)(A.v_begin / kBlock), t_hi = (int)((A.v_end + kBlock - 1) / kBlock);
  double te = 0.0, tb = 0.0;  // fused: this thread's running partials (fixed tile order)
  for (int t = t_lo + blockIdx.x; t < t_hi; t += gridDim.x) {
    const long long v = (long long)t * kBlock + tid;
    double pe = 0.0, pb = 0.0;
    if (v < A.v_end) {
      double yi[DIM];
#pragma unroll
      for (int d = 0; d < DIM; ++d) yi[d] = Yin[v * FL::DP + d];
      double f[DIM] = {};
      double e = 0.0;
      const uint32_t beg = A.row_ptr[v], end = A.row_ptr[v + 1];
      for (uint32_t k = beg; k < end; ++k) {
        const uint32_t cw = ld_col_nc(A.col + k);
        const uint32_t o = cw & kIdMask;
        const bool rn = cw & kRandBit;
        double t_ = rn ? 1.0 : 0.0, w = rn ? c : 1.0;
        if constexpr (WEIGHTED) {
          const float2 tw = __ldg(A.ew + k);
          t_ = (double)tw.x;
          w *= (double)tw.y;
        }
        double yo[DIM];
#pragma unroll
        for (int d = 0; d < DIM; ++d) yo[d] = Yin[(size_t)o * FL::DP + d];
        if (entry_f64<DIM, NORM>(yi, yo, t_, w, f, e)) {  // forces.py:167-174 (host-drawn direction)
          float u[DIM];
          degenerate_vec<DIM>(A, &ctrl->need, (uint32_t)v, (int)(k - beg), gstep, u);
#pragma unroll
          for (int d = 0; d < DIM; ++d) f[d] += (double)u[d];
        }
      }
      // Adam (optim.py:195-205) with grad = -2 f (optim.py:259-263)
      const double* sv = Sin + (size_t)v * FL::SD;
      double* so = Sout + (size_t)v * FL::SD;
      double yn[DIM];
      bool ok = true;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        const double g = -2.0 * f[d];
        const double vv = A.h.gv_d * sv[d] + (1.0 - A.h.gv_d) * g;
        const double ss = A.h.gs_d * sv[FL::DP + d] + (1.0 - A.h.gs_d) * g * g;
        so[d] = vv;
        so[FL::DP + d] = ss;
        yn[d] = yi[d] - alpha * (vv / bc1) / (A.h.eps_d + sqrt(ss / bc2));
        Yout[v * FL::DP + d] = yn[d];
        ok &= isfinite(yn[d]);
      }
      if (A.pe.on) {  // fused exchange: into every peer's replica (NVLink P2P stores)
        const bool out1 = reinterpret_cast<float*>(Yout) == A.ybuf1;
        const unsigned mk = A.pe.mask[v];
        for (int q = 0; q < A.pe.n_peers; ++q) {
          if (!((mk >> A.pe.prank[q]) & 1u)) continue;
          double* py = reinterpret_cast<double*>(out1 ? A.pe.y1[q] : A.pe.y0[q]);
#pragma unroll
          for (int d = 0; d < DIM; ++d) py[v * FL::DP + d] = yn[d];
        }
      }
      pe = e;
      pb = ok ? 0.0 : 1.0;
    }
    if (A.fuse_finalize) {
      te += pe;
      tb += pb;
    } else {  // per-tile partial (sharded): block sum in fixed order
      const double4 r = block_sum4(make_double4(pe, 0.0, 0.0, pb), sm_red);
      if (tid == 0) A.tpart[t] = r;
    }
  }
  if (!A.fuse_finalize) return;
  // block partial in fixed order, then the last block to arrive decides
  // (peer mode: into every rank's partial array, then the arrival flags)
  const double4 r = block_sum4(make_double4(te, 0.0, 0.0, tb), sm_red);
  if (warp != 0) return;
  int last = 0;
  if (lane == 0) {
    A.bpart[blockIdx.x] = r;
    if (A.pe.on && A.pe.n_peers > 0) fence_release_sys();  // this block's P2P position stores first
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(&ctrl->arrive) : "memory");
    last = old == gridDim.x - 1;
  }
  if (!__shfl_sync(0xffffffffu, last, 0)) return;
  __syncwarp();
  if (A.pe.on) {  // peer mode (see ivhd_step.cuh peer_rank_publish / peer_decide)
    peer_rank_publish(A, (int)gridDim.x);
    if (A.pe.decide_here) peer_decide<OPT_ADAM>(A);
    else if (lane == 0) ctrl->arrive = 0;
    return;
  }
  finalize_warp<OPT_ADAM>(A, A.bpart, (int)gridDim.x);
}

}  // namespace ivhd
