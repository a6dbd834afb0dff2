// fullwdd.cu -- conventional (full) WDD on the GPU, the paper's comparison method as a second
// workload (eq:deconv_mat P:90-95, eq:extract P:97-106, Fig:schematic_WDD):
//   Gf = F_r(I)                         unitary DFT over the scan axes, per detector pixel
//   chi_v = F_q^-1(Gf[v]),  W_P = F_q^-1(Y_v),  Y_v = p_hat(q) conj(p_hat(q + q_hat_v))
//   x_v = sum_r chi_v(r) conj(W_P(r)) / (|W_P(r)|^2 + eps)          (R12: plain sum over r)
//   O = conj(F^-1_unitary(x)) [/ sqrt(x_0)]                         (R13)
// F_q^-1 is centred (fftshift . ifft2 . ifftshift); for even Q that is (-1)^k ifft2((-1)^m x)
// up to a sign common to chi and W_P, and the post-factor (-1)^k cancels in chi conj(W_P) and
// |W_P|^2, so only the pre-modulation (-1)^(my+mx) is applied (folded into the frame load for
// chi).  The transforms are cuFFT (this workload is not the reduced method's path); the frame
// load, Y_v, the Wiener combine + sum and the image step are kernels here.  Memory: S x Q^2
// complex64 twice (Gf in pixel-major and scan-frequency-major order: Medium 4.3 GB, Large 17 GB)
// plus a batch of Y_v.
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <vector>

#include "internal.h"

namespace wdd {
namespace {

// frames [s][m] -> (-1)^(my+mx) I as complex64, transposed to [m][s] (pixel-major: the scan DFT of
// each detector pixel is then a contiguous batch), through 32 x 32 shared-memory tiles
template <typename T>
__global__ void fw_load_kernel(const T* __restrict__ frames, int64_t S, int QQ, int Q, float2* __restrict__ A) {
  __shared__ float tile[32][33];
  const int64_t s0 = (int64_t)blockIdx.y * 32;
  const int m0 = blockIdx.x * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t s = s0 + dy;
    const int m = m0 + threadIdx.x;
    tile[dy][threadIdx.x] = (s < S && m < QQ) ? (float)frames[s * QQ + m] : 0.f;
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int m = m0 + dy;
    const int64_t s = s0 + threadIdx.x;
    if (m < QQ && s < S) {
      const float sg = (((m / Q) + (m % Q)) & 1) ? -1.f : 1.f;
      A[(int64_t)m * S + s] = make_float2(tile[threadIdx.x][dy] * sg, 0.f);
    }
  }
}

// complex64 [rows][cols] -> [cols][rows], 32 x 32 tiles
__global__ void fw_transpose_kernel(const float2* __restrict__ in, int64_t rows, int64_t cols, float2* __restrict__ out) {
  __shared__ float2 tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t r = r0 + dy, c = c0 + threadIdx.x;
    tile[dy][threadIdx.x] = (r < rows && c < cols) ? in[r * cols + c] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t c = c0 + dy, r = r0 + threadIdx.x;
    if (c < cols && r < rows) out[c * rows + r] = tile[threadIdx.x][dy];
  }
}

__device__ __forceinline__ double fw_freq(int v, int S, double step) {
  const int sf = v < (S + 1) / 2 ? v : v - S;
  return (double)sf / __dmul_rn((double)S, step);
}

// (-1)^(my+mx) Y_v for a batch of scan frequencies (flattened v = vy*Sx + vx)
__global__ void fw_y_kernel(const int32_t* __restrict__ vlist, int nb, int Q, double dq, double qa2, double cph,
                            int Sy, int Sx, double step, float2* __restrict__ Y) {
  const int b = blockIdx.y;
  if (b >= nb) return;
  const int v = vlist[b];
  const double sy = fw_freq(v / Sx, Sy, step), sx = fw_freq(v % Sx, Sx, step);
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < Q * Q; m += gridDim.x * blockDim.x) {
    const int my = m / Q, mx = m % Q;
    const double qy = (double)(my - Q / 2) * dq, qx = (double)(mx - Q / 2) * dq;
    const double u2 = __dadd_rn(__dmul_rn(qy, qy), __dmul_rn(qx, qx));
    const double ay = __dadd_rn(qy, sy), ax = __dadd_rn(qx, sx);
    const double s2 = __dadd_rn(__dmul_rn(ay, ay), __dmul_rn(ax, ax));
    float2 y = make_float2(0.f, 0.f);
    if (u2 <= qa2 && s2 <= qa2) {
      double s, c;
      sincos(cph * (s2 - u2), &s, &c);          // p_hat(q) conj(p_hat(q + q_hat)), p_hat = e^{-i cph |q|^2}
      const float sg = ((my + mx) & 1) ? -1.f : 1.f;
      y = make_float2((float)c * sg, (float)s * sg);
    }
    Y[(int64_t)b * Q * Q + m] = y;
  }
}

// x_v = sum_r chi conj(W_P) / (|W_P|^2 + eps); chi = chi_s x (unnormalised transforms of A),
// W_P = wp_s x (unnormalised inverse DFT of Y)
__global__ void fw_combine_kernel(const float2* __restrict__ A, const float2* __restrict__ Y,
                                  const int32_t* __restrict__ vlist, int Q, double chi_s, double wp_s, double eps,
                                  float2* __restrict__ spec) {
  const int b = blockIdx.x;
  const int v = vlist[b];
  const float2* chi = A + (int64_t)v * Q * Q;
  const float2* wp = Y + (int64_t)b * Q * Q;
  double sr = 0.0, si = 0.0;
  for (int m = threadIdx.x; m < Q * Q; m += blockDim.x) {
    const float2 c = chi[m], w = wp[m];
    const double cr = c.x * chi_s, ci = c.y * chi_s, wr = w.x * wp_s, wi = w.y * wp_s;
    const double den = wr * wr + wi * wi + eps;
    sr += (cr * wr + ci * wi) / den;
    si += (ci * wr - cr * wi) / den;
  }
  __shared__ double rr[256], ri[256];
  rr[threadIdx.x] = sr;
  ri[threadIdx.x] = si;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) { rr[threadIdx.x] += rr[threadIdx.x + o]; ri[threadIdx.x] += ri[threadIdx.x + o]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) spec[v] = make_float2((float)rr[0], (float)ri[0]);
}

__global__ void fw_image_kernel(float2* __restrict__ out, int64_t S, float scale, const float2* __restrict__ spec,
                                int normalize) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S) return;
  double xr = out[i].x * (double)scale, xi = -out[i].y * (double)scale;   // conj(F^-1_unitary(x))
  if (normalize) {
    const double a = spec[0].x, b = spec[0].y, r = hypot(a, b);
    if (r > 0) {
      const double s = sqrt(0.5 * (r + fabs(a)));
      double wr, wi;
      if (a >= 0) { wr = s; wi = b / (2 * s); } else { wr = fabs(b) / (2 * s); wi = copysign(s, b); }
      const double d = wr * wr + wi * wi;
      const double yr = (xr * wr + xi * wi) / d, yi = (xi * wr - xr * wi) / d;
      xr = yr;
      xi = yi;
    }
  }
  out[i] = make_float2((float)xr, (float)xi);
}

}  // namespace

// Workspace cached in the plan across calls (the cuFFT plans and the 2 x S x Q^2 scratch cost
// milliseconds to create).
struct FullWddWork {
  float2 *A = nullptr, *B = nullptr, *Y = nullptr, *spec = nullptr;
  int32_t* dv = nullptr;
  cufftHandle scan = 0, det = 0, yplan = 0, img = 0;
  bool ok = false;
};

void full_wdd_release(Plan& p) {
  FullWddWork* w = p.fw;
  if (!w) return;
  if (w->scan) cufftDestroy(w->scan);
  if (w->det) cufftDestroy(w->det);
  if (w->yplan) cufftDestroy(w->yplan);
  if (w->img) cufftDestroy(w->img);
  cudaFree(w->A);
  cudaFree(w->B);
  cudaFree(w->Y);
  cudaFree(w->spec);
  cudaFree(w->dv);
  delete w;
  p.fw = nullptr;
}

static constexpr int kFwYBatch = 512;                   // scan frequencies per Y_v batch

static wdd_status fw_prepare(Plan& p, char* err, size_t errn) {
  if (p.fw && p.fw->ok) return WDD_OK;
  full_wdd_release(p);
  FullWddWork* w = new FullWddWork();
  p.fw = w;
  const int Q = p.Q;
  const int64_t S = p.S, QQ = (int64_t)Q * Q;
  if (cudaMalloc(&w->A, (size_t)S * QQ * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&w->B, (size_t)S * QQ * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&w->Y, (size_t)kFwYBatch * QQ * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&w->spec, (size_t)S * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&w->dv, p.active_v.size() * sizeof(int32_t)) != cudaSuccess) {
    std::snprintf(err, errn, "full WDD: %.1f GB of device scratch not available", 2.0 * S * QQ * 8 / 1e9);
    full_wdd_release(p);
    return WDD_E_NOMEM;
  }
  int sdims[2] = {p.Sy, p.Sx}, ddims[2] = {Q, Q};
  if (cudaMemcpy(w->dv, p.active_v.data(), p.active_v.size() * sizeof(int32_t), cudaMemcpyHostToDevice) !=
          cudaSuccess ||
      cufftPlanMany(&w->scan, 2, sdims, nullptr, 1, (int)S, nullptr, 1, (int)S, CUFFT_C2C, (int)QQ) != CUFFT_SUCCESS ||
      cufftPlanMany(&w->det, 2, ddims, nullptr, 1, (int)QQ, nullptr, 1, (int)QQ, CUFFT_C2C, (int)S) != CUFFT_SUCCESS ||
      cufftPlanMany(&w->yplan, 2, ddims, nullptr, 1, (int)QQ, nullptr, 1, (int)QQ, CUFFT_C2C, kFwYBatch) !=
          CUFFT_SUCCESS ||
      cufftPlan2d(&w->img, p.Sy, p.Sx, CUFFT_C2C) != CUFFT_SUCCESS) {
    std::snprintf(err, errn, "full WDD: cuFFT plan creation failed");
    full_wdd_release(p);
    return WDD_E_CUDA;
  }
  w->ok = true;
  return WDD_OK;
}

wdd_status full_wdd(Plan& p, const void* frames_dev, void* out_dev, char* err, size_t errn) {
  auto fail = [&](const char* what) {
    std::snprintf(err, errn, "full WDD: %s", what);
    return WDD_E_CUDA;
  };
  if ((p.Q & 1) || p.S > INT32_MAX) { std::snprintf(err, errn, "full WDD needs even Q"); return WDD_E_ARG; }
  const wdd_status pr = fw_prepare(p, err, errn);
  if (pr != WDD_OK) return pr;
  FullWddWork* w = p.fw;
  const int Q = p.Q;
  const int64_t S = p.S, QQ = (int64_t)Q * Q;
  cudaStream_t st = p.stream;
  if (cufftSetStream(w->scan, st) != CUFFT_SUCCESS || cufftSetStream(w->det, st) != CUFFT_SUCCESS ||
      cufftSetStream(w->yplan, st) != CUFFT_SUCCESS || cufftSetStream(w->img, st) != CUFFT_SUCCESS)
    return fail("cuFFT stream");
  if (cudaMemsetAsync(w->spec, 0, (size_t)S * sizeof(float2), st) != cudaSuccess) return fail("memset");
  // (a) frames -> (-1)^m I transposed to pixel-major B[m][s]; scan DFT of every pixel (contiguous
  // batches); transpose back to A[v][m] for the detector transforms
  const dim3 tb(32, 8);
  const dim3 tg1((unsigned)((QQ + 31) / 32), (unsigned)((S + 31) / 32));
  if (p.dtype == 0) fw_load_kernel<uint16_t><<<tg1, tb, 0, st>>>(static_cast<const uint16_t*>(frames_dev), S, (int)QQ, Q, w->B);
  else fw_load_kernel<float><<<tg1, tb, 0, st>>>(static_cast<const float*>(frames_dev), S, (int)QQ, Q, w->B);
  if (cufftExecC2C(w->scan, reinterpret_cast<cufftComplex*>(w->B), reinterpret_cast<cufftComplex*>(w->B),
                   CUFFT_FORWARD) != CUFFT_SUCCESS) return fail("scan FFT");
  const dim3 tg2((unsigned)((S + 31) / 32), (unsigned)((QQ + 31) / 32));
  fw_transpose_kernel<<<tg2, tb, 0, st>>>(w->B, QQ, S, w->A);
  // (b) chi_v for every v: inverse detector DFT of each scan-frequency row (the 1/sqrt(S) of the
  // unitary scan DFT is folded into the combine scale)
  if (cufftExecC2C(w->det, reinterpret_cast<cufftComplex*>(w->A), reinterpret_cast<cufftComplex*>(w->A),
                   CUFFT_INVERSE) != CUFFT_SUCCESS) return fail("detector FFT");
  // (c) W_P for the active v in batches, Wiener combine and sum
  const double cph = kPi * p.lambda * p.defocus;
  const double chi_s = 1.0 / ((double)Q * std::sqrt((double)S)), wp_s = 1.0 / Q;   // unitary scales
  for (int64_t a = 0; a < p.n_act; a += kFwYBatch) {
    const int m = (int)std::min<int64_t>(kFwYBatch, p.n_act - a);
    fw_y_kernel<<<dim3((unsigned)((QQ + 255) / 256), kFwYBatch), 256, 0, st>>>(w->dv + a, m, Q, p.dq, p.qa * p.qa, cph,
                                                                              p.Sy, p.Sx, p.step, w->Y);
    if (cufftExecC2C(w->yplan, reinterpret_cast<cufftComplex*>(w->Y), reinterpret_cast<cufftComplex*>(w->Y),
                     CUFFT_INVERSE) != CUFFT_SUCCESS) return fail("probe FFT");
    fw_combine_kernel<<<m, 256, 0, st>>>(w->A, w->Y, w->dv + a, Q, chi_s, wp_s, p.eps, w->spec);
  }
  // (d) O = conj(F^-1_unitary(x)) [/ sqrt(x_0)]
  if (cufftExecC2C(w->img, reinterpret_cast<cufftComplex*>(w->spec), static_cast<cufftComplex*>(out_dev),
                   CUFFT_INVERSE) != CUFFT_SUCCESS) return fail("image FFT");
  fw_image_kernel<<<(unsigned)((S + 255) / 256), 256, 0, st>>>(static_cast<float2*>(out_dev), S,
                                                                (float)(1.0 / std::sqrt((double)S)), w->spec,
                                                                p.normalize);
  if (cudaGetLastError() != cudaSuccess) return fail("kernel launch");
  return WDD_OK;
}

}  // namespace wdd
