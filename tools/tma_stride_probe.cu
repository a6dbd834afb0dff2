// tma_stride_probe.cu -- TMA read bandwidth for the access patterns of the G / W streams of the
// rank-update GEMM flush: a [rows][2K] fp32 matrix (8 KB rows at K = 1024) read in 16 KB tiles by
// one producer thread per CTA (148 CTAs, ring of NS tiles), with different box shapes:
//   w128x16   box {32 floats (128 B), 16 rows}, 8 boxes per tile (128 rows x 128 B)  [rgemm]
//   w128x128  box {32 floats, 128 rows}, 1 box per tile
//   w256x64   box {64 floats (256 B), 64 rows}, 1 box per tile
//   w512x32   box {128 floats (512 B), 32 rows}, 1 box per tile
//   w1024x16  box {256 floats (1 KB), 16 rows}, 1 box per tile
// Each CTA owns bands of 128 rows and walks the k direction tile by tile (as rgemm does).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tsp tools/tma_stride_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbar_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory"); }

constexpr int NS = 8, TILE = 16384;

// box = {bx floats, by rows}; a tile = 128 rows x (TILE / 512) ... expressed as nbx x nby boxes
__global__ void __launch_bounds__(128, 1) k_probe(const __grid_constant__ CUtensorMap tm, int rows, int cols, int bx,
                                                  int by, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * TILE);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  // tile geometry: trows x tcols floats with trows * tcols * 4 = TILE
  const int tcols = bx >= 32 ? bx : 32;              // floats along k per tile
  const int trows = TILE / (tcols * 4);
  const int nby = trows / by;
  const int bands = rows / trows, ktiles = cols / tcols;
  const int64_t jobs_total = (int64_t)bands * ktiles;
  uint32_t acc = 0;
  auto issue = [&](int64_t j, int s) {
    const int band = (int)(j / ktiles), kt = (int)(j % ktiles);
    mbar_tx(&full[s], TILE);
    for (int b = 0; b < nby; ++b)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(sa(sm + s * TILE + b * by * tcols * 4)), "l"((uint64_t)&tm), "r"(kt * tcols),
                   "r"(band * trows + b * by), "r"(sa(&full[s])) : "memory");
  };
  // CTA walks its bands in k order
  (void)jobs_total;
  const int64_t my_bands = (bands - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int64_t my_jobs = my_bands * ktiles;
  auto job_of = [&](int64_t i) { return (blockIdx.x + (i / ktiles) * gridDim.x) * (int64_t)ktiles + i % ktiles; };
  int64_t issued = 0;
  for (; issued < NS && issued < my_jobs; ++issued) issue(job_of(issued), (int)(issued % NS));
  for (int64_t i = 0; i < my_jobs; ++i) {
    mbar_wait(&full[i % NS], (uint32_t)((i / NS) & 1));
    acc += *reinterpret_cast<volatile uint32_t*>(sm + (i % NS) * TILE + 4 * (i & 255));
    if (issued < my_jobs) { issue(job_of(issued), (int)(issued % NS)); ++issued; }
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  const int K = 1024, rows = 118784, cols = 2 * K;   // Live-like: 118 845 active v x 1024 complex
  float* d;
  CK(cudaMalloc(&d, (size_t)rows * cols * 4));
  CK(cudaMemset(d, 1, (size_t)rows * cols * 4));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * TILE + 1024));
  struct V { const char* name; int bx, by; CUtensorMapSwizzle sw; };
  const V vs[] = {{"w128x16", 32, 16, CU_TENSOR_MAP_SWIZZLE_128B}, {"w128x128", 32, 128, CU_TENSOR_MAP_SWIZZLE_128B},
                  {"w256x64", 64, 64, CU_TENSOR_MAP_SWIZZLE_NONE}, {"w512x32", 128, 32, CU_TENSOR_MAP_SWIZZLE_NONE},
                  {"w1024x16", 256, 16, CU_TENSOR_MAP_SWIZZLE_NONE}};
  for (const V& v : vs) {
    CUtensorMap tm;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    const cuuint32_t box[2] = {(cuuint32_t)v.bx, (cuuint32_t)v.by};
    const cuuint32_t estr[2] = {1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, v.sw,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("%s: encode failed\n", v.name);
      continue;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) k_probe<<<148, 128, NS * TILE + 1024>>>(tm, rows, cols, v.bx, v.by, sink);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    const int reps = 5;
    for (int rep = 0; rep < reps; ++rep) k_probe<<<148, 128, NS * TILE + 1024>>>(tm, rows, cols, v.bx, v.by, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)rows * cols * 4 * reps;
    printf("%-10s %8.1f GB/s\n", v.name, bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
