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
// complex64 for Gf (Medium 2.1 GB, Large 8.6 GB) plus a batch of Y_v.
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

template <typename T>
__global__ void fw_load_kernel(const T* __restrict__ frames, int64_t S, int Q, float2* __restrict__ A) {
  const int64_t n = S * Q * Q;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(e % (Q * Q));
    const int sgn = (((m / Q) + (m % Q)) & 1) ? -1 : 1;
    A[e] = make_float2((float)frames[e] * (float)sgn, 0.f);
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

wdd_status full_wdd(Plan& p, const void* frames_dev, void* out_dev, char* err, size_t errn) {
  auto fail = [&](const char* what) {
    std::snprintf(err, errn, "full WDD: %s", what);
    return WDD_E_CUDA;
  };
  if ((p.Q & 1) || p.S > INT32_MAX) { std::snprintf(err, errn, "full WDD needs even Q"); return WDD_E_ARG; }
  const int Q = p.Q;
  const int64_t S = p.S, QQ = (int64_t)Q * Q;
  cudaStream_t st = p.stream;
  float2* A = nullptr;
  float2* Y = nullptr;
  float2* spec = nullptr;
  int32_t* dv = nullptr;
  cufftHandle scan_plan = 0, det_plan = 0, img_plan = 0;
  const int nb = 512;                                   // scan frequencies per Y_v batch
  wdd_status rc = WDD_OK;
  do {
    if (cudaMallocAsync(&A, (size_t)S * QQ * sizeof(float2), st) != cudaSuccess) { rc = WDD_E_NOMEM; break; }
    if (cudaMallocAsync(&Y, (size_t)nb * QQ * sizeof(float2), st) != cudaSuccess) { rc = WDD_E_NOMEM; break; }
    if (cudaMallocAsync(&spec, (size_t)S * sizeof(float2), st) != cudaSuccess ||
        cudaMallocAsync(&dv, p.active_v.size() * sizeof(int32_t), st) != cudaSuccess) { rc = WDD_E_NOMEM; break; }
    if (cudaMemcpyAsync(dv, p.active_v.data(), p.active_v.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st) !=
            cudaSuccess ||
        cudaMemsetAsync(spec, 0, (size_t)S * sizeof(float2), st) != cudaSuccess) { rc = fail("upload"); break; }
    // (a) frames -> (-1)^m I, scan DFT per detector pixel (stride Q^2 between scan positions)
    const int blocks = (int)std::min<int64_t>((S * QQ + 255) / 256, 148 * 32);
    if (p.dtype == 0) fw_load_kernel<uint16_t><<<blocks, 256, 0, st>>>(static_cast<const uint16_t*>(frames_dev), S, Q, A);
    else fw_load_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(frames_dev), S, Q, A);
    int sdims[2] = {p.Sy, p.Sx};
    if (cufftPlanMany(&scan_plan, 2, sdims, sdims, (int)QQ, 1, sdims, (int)QQ, 1, CUFFT_C2C, (int)QQ) != CUFFT_SUCCESS ||
        cufftSetStream(scan_plan, st) != CUFFT_SUCCESS ||
        cufftExecC2C(scan_plan, reinterpret_cast<cufftComplex*>(A), reinterpret_cast<cufftComplex*>(A),
                     CUFFT_FORWARD) != CUFFT_SUCCESS) { rc = fail("scan FFT"); break; }
    // (b) chi_v for every v: inverse detector DFT of each scan-frequency row (the 1/sqrt(S) of
    // the unitary scan DFT is folded into the combine scale)
    int ddims[2] = {Q, Q};
    const int64_t vb = 4096;
    if (cufftPlanMany(&det_plan, 2, ddims, nullptr, 1, (int)QQ, nullptr, 1, (int)QQ, CUFFT_C2C, (int)vb) !=
            CUFFT_SUCCESS || cufftSetStream(det_plan, st) != CUFFT_SUCCESS) { rc = fail("detector plan"); break; }
    for (int64_t v0 = 0; v0 < S && rc == WDD_OK; v0 += vb) {
      cufftHandle ph = det_plan, tmp = 0;
      if (S - v0 < vb) {
        if (cufftPlanMany(&tmp, 2, ddims, nullptr, 1, (int)QQ, nullptr, 1, (int)QQ, CUFFT_C2C, (int)(S - v0)) !=
                CUFFT_SUCCESS || cufftSetStream(tmp, st) != CUFFT_SUCCESS) { rc = fail("detector plan"); break; }
        ph = tmp;
      }
      if (cufftExecC2C(ph, reinterpret_cast<cufftComplex*>(A + v0 * QQ), reinterpret_cast<cufftComplex*>(A + v0 * QQ),
                       CUFFT_INVERSE) != CUFFT_SUCCESS) rc = fail("detector FFT");
      if (tmp) cufftDestroy(tmp);
    }
    if (rc != WDD_OK) break;
    // (c) W_P for the active v in batches, Wiener combine and sum
    cufftHandle yplan = 0;
    if (cufftPlanMany(&yplan, 2, ddims, nullptr, 1, (int)QQ, nullptr, 1, (int)QQ, CUFFT_C2C, nb) != CUFFT_SUCCESS ||
        cufftSetStream(yplan, st) != CUFFT_SUCCESS) { rc = fail("probe plan"); break; }
    const double cph = kPi * p.lambda * p.defocus;
    const double chi_s = 1.0 / ((double)Q * std::sqrt((double)S)), wp_s = 1.0 / Q;   // unitary scales
    for (int64_t a = 0; a < p.n_act && rc == WDD_OK; a += nb) {
      const int m = (int)std::min<int64_t>(nb, p.n_act - a);
      fw_y_kernel<<<dim3((unsigned)((QQ + 255) / 256), nb), 256, 0, st>>>(dv + a, m, Q, p.dq, p.qa * p.qa, cph, p.Sy,
                                                                         p.Sx, p.step, Y);
      if (cufftExecC2C(yplan, reinterpret_cast<cufftComplex*>(Y), reinterpret_cast<cufftComplex*>(Y), CUFFT_INVERSE) !=
          CUFFT_SUCCESS) { rc = fail("probe FFT"); break; }
      fw_combine_kernel<<<m, 256, 0, st>>>(A, Y, dv + a, Q, chi_s, wp_s, p.eps, spec);
    }
    cufftDestroy(yplan);
    if (rc != WDD_OK) break;
    // (d) O = conj(F^-1_unitary(x)) [/ sqrt(x_0)]
    if (cufftPlan2d(&img_plan, p.Sy, p.Sx, CUFFT_C2C) != CUFFT_SUCCESS || cufftSetStream(img_plan, st) != CUFFT_SUCCESS ||
        cufftExecC2C(img_plan, reinterpret_cast<cufftComplex*>(spec), static_cast<cufftComplex*>(out_dev),
                     CUFFT_INVERSE) != CUFFT_SUCCESS) { rc = fail("image FFT"); break; }
    fw_image_kernel<<<(unsigned)((S + 255) / 256), 256, 0, st>>>(static_cast<float2*>(out_dev), S,
                                                                  (float)(1.0 / std::sqrt((double)S)), spec,
                                                                  p.normalize);
    if (cudaGetLastError() != cudaSuccess) rc = fail("kernel launch");
  } while (false);
  if (scan_plan) cufftDestroy(scan_plan);
  if (det_plan) cufftDestroy(det_plan);
  if (img_plan) cufftDestroy(img_plan);
  cudaFreeAsync(A, st);
  cudaFreeAsync(Y, st);
  cudaFreeAsync(spec, st);
  cudaFreeAsync(dv, st);
  return rc;
}

}  // namespace wdd
