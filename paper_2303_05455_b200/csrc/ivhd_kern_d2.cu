// ivhd_kern_d2.cu — instantiations of the step kernels for target_dim = 2
// (table in ivhd_kernels.h).
#include "ivhd_kernels.h"
#include "ivhd_step_f64.cuh"

namespace ivhd {
namespace {

template <int OPT, bool W, int N, bool P>
KernelInfo info() {
  return KernelInfo{step_kernel<2, OPT, W, N, P>, step_smem_bytes<2, OPT, W, N>()};
}

template <bool W, int N, bool P>
KernelInfo by_opt(int opt) {
  switch (opt) {
    case OPT_ADAM: return KernelInfo{step_kernel_f64<2, W, N>, 0, kBlock};  // fp64, peer mode at run time
    case OPT_FD: return info<OPT_FD, W, N, P>();
    case OPT_SGD: return info<OPT_SGD, W, N, P>();
    case OPT_MOM: return info<OPT_MOM, W, N, P>();
    case OPT_NEST: return info<OPT_NEST, W, N, P>();
    case OPT_ADADELTA: return info<OPT_ADADELTA, W, N, P>();
    default: return info<OPT_NONE, W, N, false>();
  }
}

template <bool W, bool P>
KernelInfo by_norm(int opt, int norm) {
  return norm == 0 ? by_opt<W, 0, P>(opt) : by_opt<W, 1, P>(opt);
}

}  // namespace

KernelInfo kernel_d2(int opt, bool weighted, int norm, bool peer) {
  if (peer) return weighted ? by_norm<true, true>(opt, norm) : by_norm<false, true>(opt, norm);
  return weighted ? by_norm<true, false>(opt, norm) : by_norm<false, false>(opt, norm);
}

}  // namespace ivhd

#ifdef IVHD_TIMELINE
// debug builds (tools/timeline.py): the 2-D step kernels live in this unit,
// so its copy of the timeline buffer is the one they write
extern "C" int ivhd_timeline_dump(long long* out) {
  return cudaMemcpyFromSymbol(out, ivhd::g_tl, sizeof(ivhd::g_tl)) == cudaSuccess ? 0 : 2;
}
#endif
