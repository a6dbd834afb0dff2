// bw_probe.cu -- read-bandwidth ceilings for the projection's frame stream on B200.
// Streams N frames of Q x Q uint16 (>> L2) three ways and reports GB/s:
//   tma2d   2-D TMA boxes of 128 rows x 64 px, SWIZZLE_128B, 8-slot ring per CTA (the projection's
//           load pattern, no compute)
//   bulk    1-D cp.async.bulk of 32 KB contiguous pieces, 8-slot ring per CTA
//   ldg     plain LDG.128 grid-stride reduction
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe tools/bw_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbar_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory"); }

constexpr int NS = 8;

__global__ void __launch_bounds__(128, 1) k_tma(const __grid_constant__ CUtensorMap tm, int64_t n_tiles, int cpt, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * 16384);
  if (threadIdx.x == 0) { for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t acc = 0;
  int64_t job = 0;
  const int64_t jobs = ((n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x) * cpt;
  auto issue = [&](int64_t j) {
    const int64_t t = blockIdx.x + (j / cpt) * gridDim.x;
    const int c = (int)(j % cpt), s = (int)(j % NS);
    mbar_tx(&full[s], 16384);
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(sa(sm + s * 16384)), "l"((uint64_t)&tm), "r"(c * 64), "r"((int)(t * 128)), "r"(sa(&full[s])) : "memory");
  };
  for (; job < NS && job < jobs; ++job) issue(job);
  for (int64_t j = 0; j < jobs; ++j) {
    mbar_wait(&full[j % NS], (uint32_t)((j / NS) & 1));
    acc += *reinterpret_cast<volatile uint32_t*>(sm + (j % NS) * 16384 + 4 * (j & 255));
    if (job < jobs) { issue(job); ++job; }
  }
  if (acc == 0x12345678u) *sink = acc;
}

constexpr int NSB = 6;
__global__ void __launch_bounds__(128, 1) k_bulk(const uint8_t* src, int64_t n_pieces, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int NS = NSB;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * 32768);
  if (threadIdx.x == 0) { for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t acc = 0;
  const int64_t jobs = (n_pieces - blockIdx.x + gridDim.x - 1) / gridDim.x;
  int64_t job = 0;
  auto issue = [&](int64_t j) {
    const int64_t t = blockIdx.x + j * gridDim.x;
    const int s = (int)(j % NS);
    mbar_tx(&full[s], 32768);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(sm + s * 32768)), "l"(src + t * 32768), "r"(32768), "r"(sa(&full[s])) : "memory");
  };
  for (; job < NS && job < jobs; ++job) issue(job);
  for (int64_t j = 0; j < jobs; ++j) {
    mbar_wait(&full[j % NS], (uint32_t)((j / NS) & 1));
    acc += *reinterpret_cast<volatile uint32_t*>(sm + (j % NS) * 32768 + 4 * (j & 255));
    if (job < jobs) { issue(job); ++job; }
  }
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void k_ldg(const uint4* src, int64_t n, unsigned long long* sink) {
  uint32_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(src + i);
    acc += v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  const int Q = 128;
  const int64_t N = 16384;
  const size_t bytes = (size_t)N * Q * Q * 2;
  uint8_t* d;
  unsigned long long* sink;
  CK(cudaMalloc(&d, bytes));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(d, 1, bytes));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // tensor map
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)Q, (cuuint64_t)(N * Q)};
  const cuuint64_t strides[1] = {(cuuint64_t)Q * 2};
  const cuuint32_t box[2] = {64u, 128u}, es[2] = {1u, 1u};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * 16384 + 1024));
  CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, NSB * 32768 + 1024));
  for (int grid_mul = 1; grid_mul <= 2; ++grid_mul) {
    for (int variant = 0; variant < 3; ++variant) {
      float best = 1e9;
      for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0);
        if (variant == 0) k_tma<<<sms * grid_mul, 128, NS * 16384 + 1024>>>(tm, N * Q / 128, 2, sink);
        if (variant == 1 && grid_mul == 1) k_bulk<<<sms, 128, NSB * 32768 + 1024>>>(d, (int64_t)(bytes / 32768), sink);
        if (variant == 2) k_ldg<<<sms * 8 * grid_mul, 512>>>(reinterpret_cast<const uint4*>(d), (int64_t)(bytes / 16), sink);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
      }
      const char* nm[3] = {"tma2d(64px x 128 rows, SW128, 8 x 16KB)", "bulk(32KB, 6 slots)", "ldg128"};
      if (!(variant == 1 && grid_mul == 2))
        printf("%-42s grid=%d x SMs: %.1f GB/s (%.1f us for %.0f MB)\n", nm[variant], grid_mul, bytes / (best * 1e-3) / 1e9,
               best * 1e3, bytes / 1e6);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
