// ivhd_kernels.h — the step-kernel table shared by the C-ABI translation unit
// and the per-dimension kernel translation units (ivhd_kern_d2.cu,
// ivhd_kern_d3.cu), which instantiate every (optimizer, weighted, norm, peer)
// variant; split so the instantiations compile in parallel.
#pragma once
#include "ivhd_step.cuh"

namespace ivhd {

using KernelFn = void (*)(StepArgs);

struct KernelInfo {
  KernelFn fn;
  int smem;
  int threads = kThreads;
};

// dim 2 / dim 3 tables (opt: Opt; norm 0 = L2, 1 = L1; peer = fused NVLink exchange)
KernelInfo kernel_d2(int opt, bool weighted, int norm, bool peer);
KernelInfo kernel_d3(int opt, bool weighted, int norm, bool peer);

inline KernelInfo pick_kernel(int dim, int opt, bool weighted, int norm, bool peer = false) {
  return dim == 2 ? kernel_d2(opt, weighted, norm, peer) : kernel_d3(opt, weighted, norm, peer);
}

}  // namespace ivhd
