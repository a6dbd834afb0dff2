// forward.cu -- seeded forward simulator on the GPU (test-input generator; the
// paper's eq:forward P:83-87 and Poisson dose model P:625-630).  Same recipe as synth/generator.py:
//   exit_s[j][i] = P[j][i] * O[(sy + j - Q/2) mod Sy][(sx + i - Q/2) mod Sx]
//   I_s = |centred unitary DFT2(exit_s)|^2,   lambda = dose * I_s / sum(I_s)
//   counts ~ Poisson(lambda)  (Philox4x32-10 keyed by (seed, 1), counter (pixel, s, draw)),
// with the object O and the real-space probe P supplied by the host generator (complex64).  The
// DFT is cuFFT (this is input generation, not the method's path).  Holds none of the
// reconstruction's arithmetic; shares no code with the library or the oracle.
#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdint>

namespace {

// ---- Philox4x32-10 (Salmon et al., SC'11): counter-based, one 4 x 32-bit block per call
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// uniforms in (0, 1) from a per-pixel stream: counter (pixel, s_lo, s_hi, draw block)
struct Stream {
  uint32_t pix, slo, shi, k0, k1, blk = 0;
  int used = 4;
  U4 buf{};
  __device__ double next() {
    if (used == 4) {
      buf = philox(U4{pix, slo, shi, blk++}, k0, k1);
      used = 0;
    }
    const uint32_t v = used == 0 ? buf.x : used == 1 ? buf.y : used == 2 ? buf.z : buf.w;
    ++used;
    return ((double)v + 0.5) * (1.0 / 4294967296.0);
  }
};

// Poisson(lambda): multiplication method below 10, PTRS (Hoermann 1993) above -- the same
// split numpy's legacy-free generator uses (different random streams, same distribution).
__device__ uint32_t poisson(Stream& rs, double lam) {
  if (lam <= 0.0) return 0;
  if (lam < 10.0) {
    const double e = exp(-lam);
    double prod = 1.0;
    uint32_t k = 0;
    while (true) {
      prod *= rs.next();
      if (prod <= e) return k;
      ++k;
    }
  }
  const double slam = sqrt(lam), loglam = log(lam);
  const double b = 0.931 + 2.53 * slam, a = -0.059 + 0.02483 * b;
  const double invalpha = 1.1239 + 1.1328 / (b - 3.4), vr = 0.9277 - 3.6224 / (b - 2.0);
  while (true) {
    const double U = rs.next() - 0.5, V = rs.next();
    const double us = 0.5 - fabs(U);
    const double k = floor((2.0 * a / us + b) * U + lam + 0.43);
    if (us >= 0.07 && V <= vr) return (uint32_t)k;
    if (k < 0.0 || (us < 0.013 && V > us)) continue;
    if (log(V) + log(invalpha) - log(a / (us * us) + b) <= -lam + k * loglam - lgamma(k + 1.0)) return (uint32_t)k;
  }
}

// exit wave of frame f (scan index idx[f]) written ifftshift-ed for the DFT: element (j, i) at
// ((j + Q/2) mod Q, (i + Q/2) mod Q)
__global__ void exit_kernel(const float2* __restrict__ obj, const float2* __restrict__ probe,
                            const int64_t* __restrict__ idx, int Sy, int Sx, int Q, float2* __restrict__ buf) {
  const int f = blockIdx.y;
  const int64_t s = idx[f];
  const int sy = (int)(s / Sx), sx = (int)(s % Sx);
  const int h = Q / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < Q * Q; e += gridDim.x * blockDim.x) {
    const int j = e / Q, i = e % Q;
    const int oy = ((sy + j - h) % Sy + Sy) % Sy, ox = ((sx + i - h) % Sx + Sx) % Sx;
    const float2 o = obj[(int64_t)oy * Sx + ox], p = probe[e];
    const float2 v = make_float2(p.x * o.x - p.y * o.y, p.x * o.y + p.y * o.x);
    buf[(int64_t)f * Q * Q + ((j + h) % Q) * Q + (i + h) % Q] = v;
  }
}

// I = |F|^2 / Q^2 (unitary), fftshift-ed back to DC at (Q/2, Q/2), and the per-frame sum
__global__ void intensity_kernel(const float2* __restrict__ buf, int Q, double* __restrict__ I,
                                 double* __restrict__ sums) {
  const int f = blockIdx.x;
  const int h = Q / 2;
  double acc = 0.0;
  const double inv = 1.0 / ((double)Q * Q);
  for (int e = threadIdx.x; e < Q * Q; e += blockDim.x) {
    const int ky = e / Q, kx = e % Q;
    const float2 z = buf[(int64_t)f * Q * Q + ((ky + h) % Q) * Q + (kx + h) % Q];
    const double v = ((double)z.x * z.x + (double)z.y * z.y) * inv;
    I[(int64_t)f * Q * Q + e] = v;
    acc += v;
  }
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[f] = red[0];
}

template <typename OutT>
__global__ void sample_kernel(const double* __restrict__ I, const double* __restrict__ sums,
                              const int64_t* __restrict__ idx, int Q, double dose, uint32_t seed, int noise,
                              OutT* __restrict__ out, uint32_t* __restrict__ overflow) {
  const int f = blockIdx.y;
  const int64_t s = idx[f];
  const double scale = sums[f] > 0.0 ? dose / sums[f] : 0.0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < Q * Q; e += gridDim.x * blockDim.x) {
    const double lam = I[(int64_t)f * Q * Q + e] * scale;
    double v = lam;
    if (noise) {
      Stream rs{(uint32_t)e, (uint32_t)s, (uint32_t)((uint64_t)s >> 32), seed, 1u};
      const uint32_t k = poisson(rs, lam);
      if (sizeof(OutT) == 2 && k > 65535u) atomicOr(overflow, 1u);
      v = (double)k;
    }
    out[(int64_t)f * Q * Q + e] = (OutT)v;
  }
}

}  // namespace

// frames for n scan indices (host idx), written to out_dev (n x Q x Q, uint16 if dtype == 0 else
// float32; float64 noise-free intensities scaled to the dose if noise == 0 -- out_dev then holds
// doubles).  obj_dev: Sy x Sx complex64, probe_dev: Q x Q complex64 (device).  Synchronous.
// Returns 0, or -1 on a CUDA / cuFFT error, -2 if a count overflowed uint16.
extern "C" int sim_frames(const void* obj_dev, const void* probe_dev, int Sy, int Sx, int Q, const int64_t* idx_host,
                          int64_t n, double dose, uint32_t seed, int dtype, int noise, void* out_dev) {
  const int64_t chunk = 256;
  float2* buf = nullptr;
  double *I = nullptr, *sums = nullptr;
  int64_t* didx = nullptr;
  uint32_t* ovf = nullptr;
  cufftHandle plan = 0;
  int rc = 0;
  int dims[2] = {Q, Q};
  if (cudaMalloc(&buf, chunk * Q * Q * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&I, chunk * Q * Q * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&sums, chunk * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&didx, n * sizeof(int64_t)) != cudaSuccess || cudaMalloc(&ovf, sizeof(uint32_t)) != cudaSuccess ||
      cudaMemcpy(didx, idx_host, n * sizeof(int64_t), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(ovf, 0, sizeof(uint32_t)) != cudaSuccess ||
      cufftPlanMany(&plan, 2, dims, nullptr, 1, Q * Q, nullptr, 1, Q * Q, CUFFT_C2C, (int)chunk) != CUFFT_SUCCESS) {
    rc = -1;
  }
  for (int64_t a = 0; rc == 0 && a < n; a += chunk) {
    const int m = (int)(n - a < chunk ? n - a : chunk);
    exit_kernel<<<dim3((Q * Q + 255) / 256, m), 256>>>(static_cast<const float2*>(obj_dev),
                                                       static_cast<const float2*>(probe_dev), didx + a, Sy, Sx, Q, buf);
    if (cufftExecC2C(plan, reinterpret_cast<cufftComplex*>(buf), reinterpret_cast<cufftComplex*>(buf), CUFFT_FORWARD) !=
        CUFFT_SUCCESS) {
      rc = -1;
      break;
    }
    intensity_kernel<<<m, 256>>>(buf, Q, I, sums);
    const dim3 g((Q * Q + 255) / 256, m);
    if (!noise) {
      sample_kernel<double><<<g, 256>>>(I, sums, didx + a, Q, dose, seed, 0,
                                        static_cast<double*>(out_dev) + a * Q * Q, ovf);
    } else if (dtype == 0) {
      sample_kernel<uint16_t><<<g, 256>>>(I, sums, didx + a, Q, dose, seed, 1,
                                          static_cast<uint16_t*>(out_dev) + a * Q * Q, ovf);
    } else {
      sample_kernel<float><<<g, 256>>>(I, sums, didx + a, Q, dose, seed, 1, static_cast<float*>(out_dev) + a * Q * Q,
                                       ovf);
    }
    if (cudaGetLastError() != cudaSuccess) rc = -1;
  }
  uint32_t h_ovf = 0;
  if (rc == 0 && (cudaDeviceSynchronize() != cudaSuccess ||
                  cudaMemcpy(&h_ovf, ovf, sizeof(uint32_t), cudaMemcpyDeviceToHost) != cudaSuccess))
    rc = -1;
  if (rc == 0 && h_ovf) rc = -2;
  if (plan) cufftDestroy(plan);
  cudaFree(buf);
  cudaFree(I);
  cudaFree(sums);
  cudaFree(didx);
  cudaFree(ovf);
  return rc;
}
