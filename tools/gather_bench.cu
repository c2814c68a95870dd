// Random-gather microbenchmark (sm_100a): how many random position reads per
// second one B200 serves from L2, through the LSU path (one ld.global per
// gather, what the step kernel does) versus TMA tile::gather4 (one bulk
// instruction fetches four random 16-byte rows into shared memory).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gather_bench tools/gather_bench.cu -lcuda
//   /tmp/gather_bench [M=1400000] [gathers=8400000] [reps=50]
//
// M vertices of 2 floats (the C3 position array: 11.2 MB, L2 resident);
// `gathers` uniformly random vertex ids per pass (the C3 symmetrised entry
// count).  Prints gathers/s for each variant (CUDA events, warm L2).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

// LSU: each thread streams its slice of the id list, 8 gathers in flight.
__global__ void lsu_gather(const float2* __restrict__ Y, const uint32_t* __restrict__ idx, int64_t n, float* out) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    uint32_t j[8];
    float2 p[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) j[q] = __ldcs(idx + i + q * stride);
#pragma unroll
    for (int q = 0; q < 8; ++q) p[q] = __ldg(Y + j[q]);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += p[q].x * p[q].y;
  }
  for (; i < n; i += stride) {
    const float2 p = __ldg(Y + __ldcs(idx + i));
    acc += p.x * p.y;
  }
  if (acc == 1234.5f) *out = acc;  // keep the loads
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// TMA gather4: one warp per block; each lane owns 4 ids per stage and issues
// one gather4 of the 4 rows (row = the 4 vertices v >> 2, 32 bytes = one
// sector; the destination of a tensor copy must be 128-byte aligned) into the
// stage; kStages stages in flight; the same lane then reads its 4 rows back.
constexpr int kStages = 8;
__global__ void __launch_bounds__(32) tma_gather(const __grid_constant__ CUtensorMap tmap,
                                                 const uint32_t* __restrict__ idx, int64_t n, float* out) {
  __shared__ alignas(128) float2 buf[kStages][32][16];  // [lane][row * 4 + v & 3]
  __shared__ alignas(8) uint64_t bar[kStages];
  const int lane = threadIdx.x;
  if (lane < kStages) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[lane])));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t chunk = 128;
  const int64_t n_chunks = n / chunk;
  float acc = 0.f;
  uint32_t phase = 0;
  auto issue = [&](int64_t c, int s) {
    const uint4 j = *reinterpret_cast<const uint4*>(idx + c * chunk + lane * 4);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(128 * 32) : "memory");
    __syncwarp();
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(smem_u32(&buf[s][lane][0])), "l"(&tmap), "r"(0), "r"((int)(j.x >> 2)), "r"((int)(j.y >> 2)),
        "r"((int)(j.z >> 2)), "r"((int)(j.w >> 2)), "r"(smem_u32(&bar[s]))
        : "memory");
  };
  int64_t c = blockIdx.x;
  int64_t ci = c;
  for (int k = 0; k < kStages && ci < n_chunks; ++k, ci += gridDim.x) issue(ci, k);
  int s = 0;
  for (; c < n_chunks; c += gridDim.x) {
    // wait stage s
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(ok) : "r"(smem_u32(&bar[s])), "r"(phase) : "memory");
    }
    const uint4 j = *reinterpret_cast<const uint4*>(idx + c * chunk + lane * 4);
    const float2 r0 = buf[s][lane][0 + (j.x & 3)], r1 = buf[s][lane][4 + (j.y & 3)];
    const float2 r2 = buf[s][lane][8 + (j.z & 3)], r3 = buf[s][lane][12 + (j.w & 3)];
    acc += r0.x * r0.y + r1.x * r1.y + r2.x * r2.y + r3.x * r3.y;
    __syncwarp();
    if (ci < n_chunks) {
      issue(ci, s);
      ci += gridDim.x;
    }
    if (++s == kStages) { s = 0; phase ^= 1; }
  }
  if (acc == 1234.5f) *out = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int64_t M = argc > 1 ? atoll(argv[1]) : 1400000;
  const int64_t N = argc > 2 ? atoll(argv[2]) : 8400000;
  const int reps = argc > 3 ? atoi(argv[3]) : 50;
  std::vector<uint32_t> h(N);
  uint64_t x = 88172645463325252ull;
  for (int64_t i = 0; i < N; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    h[i] = (uint32_t)(x % (uint64_t)M);
  }
  float2* Y; uint32_t* idx; float* out;
  CK(cudaMalloc(&Y, sizeof(float2) * (M + 4)));
  CK(cudaMalloc(&idx, sizeof(uint32_t) * N));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(Y, 0, sizeof(float2) * (M + 4)));
  CK(cudaMemcpy(idx, h.data(), sizeof(uint32_t) * N, cudaMemcpyHostToDevice));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto timeit = [&](const char* name, auto launch) {
    for (int r = 0; r < 3; ++r) launch();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0; CK(cudaEventElapsedTime(&ms, e0, e1));
    const double us = ms * 1e3 / reps;
    printf("%-28s %8.2f us/pass  %7.1f G gathers/s\n", name, us, N / us / 1e3);
  };
  for (int bps : {4, 8, 16}) {
    char nm[64]; snprintf(nm, sizeof nm, "lsu ldg float2 (%d x 256/SM)", bps);
    timeit(nm, [&] { lsu_gather<<<sms * bps, 256>>>(Y, idx, N, out); });
  }
  // tensor map over (M+3)/4 rows of 8 floats (4 vertices, one sector)
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap tm;
  const cuuint64_t dims[2] = {8, (cuuint64_t)((M + 3) / 4)};
  const cuuint64_t strides[1] = {32};
  const cuuint32_t box[2] = {8, 1};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("tensor map encode failed %d\n", (int)r); return 1; }
  for (int bps : {8, 16, 32}) {
    char nm[64]; snprintf(nm, sizeof nm, "tma gather4 (%d warps/SM)", bps);
    timeit(nm, [&] { tma_gather<<<sms * bps, 32>>>(tm, idx, N, out); });
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}
