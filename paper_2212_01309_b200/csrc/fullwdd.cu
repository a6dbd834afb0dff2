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
// float32 (the frames, pixel-major) + S/2 x Q^2 complex64 (Gf's half plane, pixel-major) + n_act x Q^2
// complex64 (the active scan frequencies' rows in scan-frequency-major order); Medium 1.1 + 1.1 +
// 1.0 GB, Large 4.3 + 4.3 + 3.9 GB; plus a batch of Y_v.
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

// frames [s][m] -> (-1)^(my+mx) I as float32, transposed to [m][s] (pixel-major: the scan DFT of
// each detector pixel is then a contiguous real-to-complex batch), through 32 x 32 shared-memory tiles
template <typename T>
__global__ void fw_load_kernel(const T* __restrict__ frames, int64_t S, int QQ, int Q, float* __restrict__ A) {
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
      A[(int64_t)m * S + s] = tile[threadIdx.x][dy] * sg;
    }
  }
}

// The same with two detector pixels per load and two scan positions per store (4-byte u16 / 8-byte
// f32 loads: a warp reads 128 / 256 contiguous bytes of a frame; 8-byte stores: 256 contiguous
// bytes of a pixel's scan row); 64 scan positions x 64 pixels per tile, block 32 x 8, the eight
// loads of a thread issued together.  Needs QQ and S even and a frame pointer aligned to two
// elements (checked by the caller).
template <typename T>
__global__ void fw_load2_kernel(const T* __restrict__ frames, int64_t S, int QQ, int Q, float* __restrict__ A) {
  __shared__ float tile[64][65];
  const int64_t s0 = (int64_t)blockIdx.y * 64;
  const int m0 = blockIdx.x * 64;
  float2 ld[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t s = s0 + threadIdx.y + 8 * i;
    const int m = m0 + 2 * threadIdx.x;
    ld[i] = make_float2(0.f, 0.f);
    if (s < S && m < QQ) {
      if constexpr (sizeof(T) == 2) {
        const ushort2 v = __ldg(reinterpret_cast<const ushort2*>(frames + s * QQ + m));
        ld[i] = make_float2((float)v.x, (float)v.y);
      } else {
        ld[i] = __ldg(reinterpret_cast<const float2*>(frames + s * QQ + m));
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    tile[threadIdx.y + 8 * i][2 * threadIdx.x] = ld[i].x;
    tile[threadIdx.y + 8 * i][2 * threadIdx.x + 1] = ld[i].y;
  }
  __syncthreads();
#pragma unroll
  for (int dm = threadIdx.y; dm < 64; dm += 8) {
    const int m = m0 + dm;
    const int64_t s = s0 + 2 * threadIdx.x;
    if (m < QQ && s < S) {
      const float sg = (((m / Q) + (m % Q)) & 1) ? -1.f : 1.f;
      *reinterpret_cast<float2*>(A + (int64_t)m * S + s) =
          make_float2(tile[2 * threadIdx.x][dm] * sg, tile[2 * threadIdx.x + 1][dm] * sg);
    }
  }
}

// Gf of the real frames is Hermitian per pixel, Gf[m][-v] = conj Gf[m][v], so the scan DFT is a
// real-to-complex transform that stores vx <= Sx/2 only: B[m][vy][vx], Sxh = Sx/2 + 1 columns.
// B (pixel-major) -> A[b][m] = Gf[m][v_b] for the listed scan frequencies only (the inactive v have
// Y_v = 0 and contribute nothing: their detector transforms are never needed), mirror columns read
// as conjugates; 32 x 32 tiles; vlist ascending, so the gathered reads of a tile row are runs of
// consecutive addresses
__global__ void fw_gather_transpose_kernel(const float2* __restrict__ in, int64_t QQ, int Sy, int Sx,
                                           const int32_t* __restrict__ vlist, int64_t nv, float2* __restrict__ out) {
  __shared__ float2 tile[32][33];
  const int Sxh = Sx / 2 + 1;
  const int64_t pitch = (int64_t)Sy * Sxh;
  const int64_t m0 = (int64_t)blockIdx.y * 32, b0 = (int64_t)blockIdx.x * 32;
  const int64_t bl = b0 + threadIdx.x;
  int64_t off = -1;
  float cj = 1.f;
  if (bl < nv) {
    const int v = vlist[bl], vy = v / Sx, vx = v % Sx;
    if (vx <= Sx / 2) off = (int64_t)vy * Sxh + vx;
    else { off = (int64_t)((Sy - vy) % Sy) * Sxh + (Sx - vx); cj = -1.f; }
  }
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t m = m0 + dy;
    float2 z = (m < QQ && off >= 0) ? in[m * pitch + off] : make_float2(0.f, 0.f);
    z.y *= cj;
    tile[dy][threadIdx.x] = z;
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t b = b0 + dy, m = m0 + threadIdx.x;
    if (b < nv && m < QQ) out[b * QQ + m] = tile[threadIdx.x][dy];
  }
}

__device__ __forceinline__ double fw_freq(int v, int S, double step) {
  const int sf = v < (S + 1) / 2 ? v : v - S;
  return (double)sf / __dmul_rn((double)S, step);
}

// (-1)^(my+mx) Y_v for a batch of scan frequencies (flattened v = vy*Sx + vx), one CTA per v.
// Y_v = p_hat(q) conj(p_hat(q + q_hat)) with p_hat = e^{-i cph |q|^2} on the aperture, and
// |q + q_hat|^2 - |q|^2 = 2 q.q_hat + |q_hat|^2 is linear in q: the phase factor separates into a
// constant, a per-row and a per-column factor (2Q float64 sincos per v instead of Q^2), multiplied
// in float64.  The aperture tests are the per-pixel float64 tests of the oracle's Y_v.
__global__ void __launch_bounds__(256) fw_y_kernel(const int32_t* __restrict__ vlist, int nb, int Q, double dq,
                                                   double qa2, double cph, int Sy, int Sx, double step,
                                                   float2* __restrict__ Y) {
  // per row my / column mx: the phase factor (the rows' carrying the constant e^{i cph |q_hat|^2}),
  // q^2 and (q + q_hat)^2, each rounded as in the per-pixel sums u2 = qy^2 + qx^2, s2 = ay^2 + ax^2
  extern __shared__ double2 fw_e[];            // [2Q] factors, then [2Q] (q^2, (q + q_hat)^2)
  double2* fw_q = fw_e + 2 * Q;
  const int b = blockIdx.x;
  if (b >= nb) return;
  const int v = vlist[b];
  const double sy = fw_freq(v / Sx, Sy, step), sx = fw_freq(v % Sx, Sx, step);
  double s0, c0;
  sincos(cph * (sy * sy + sx * sx), &s0, &c0);
  for (int i = threadIdx.x; i < 2 * Q; i += blockDim.x) {
    const bool row = i < Q;
    const double q = (double)((row ? i : i - Q) - Q / 2) * dq;
    const double sh = row ? sy : sx;
    double sn, cs;
    sincos(cph * 2.0 * q * sh, &sn, &cs);
    fw_e[i] = row ? make_double2(c0 * cs - s0 * sn, c0 * sn + s0 * cs) : make_double2(cs, sn);
    const double a = __dadd_rn(q, sh);
    fw_q[i] = make_double2(__dmul_rn(q, q), __dmul_rn(a, a));
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int my = warp; my < Q; my += nw) {
    const double2 ey = fw_e[my], qy = fw_q[my];
    float2* Yr = Y + (int64_t)b * Q * Q + (int64_t)my * Q;
    for (int mx = lane; mx < Q; mx += 32) {
      const double2 qx = fw_q[Q + mx];
      float2 y = make_float2(0.f, 0.f);
      if (__dadd_rn(qy.x, qx.x) <= qa2 && __dadd_rn(qy.y, qx.y) <= qa2) {
        const double2 ex = fw_e[Q + mx];
        const double c = ey.x * ex.x - ey.y * ex.y, sn = ey.x * ex.y + ey.y * ex.x;   // e^{i cph (s2 - u2)}
        const float sg = ((my + mx) & 1) ? -1.f : 1.f;
        y = make_float2((float)c * sg, (float)sn * sg);
      }
      Yr[mx] = y;
    }
  }
}

// x_v = sum_r chi conj(W_P) / (|W_P|^2 + eps); chi = chi_s x (unnormalised transforms of A),
// W_P = wp_s x (unnormalised inverse DFT of Y)
__global__ void fw_combine_kernel(const float2* __restrict__ A, const float2* __restrict__ Y,
                                  const int32_t* __restrict__ vlist, int Q, double chi_s, double wp_s, double eps,
                                  float2* __restrict__ spec) {
  // (A and vlist already offset to the batch: row b of A is chi of vlist[b])
  const int b = blockIdx.x;
  const int v = vlist[b];
  const float2* chi = A + (int64_t)b * Q * Q;
  const float2* wp = Y + (int64_t)b * Q * Q;
  double sr = 0.0, si = 0.0;
  auto term = [&](float cx, float cy, float wx, float wy) {
    const double cr = cx * chi_s, ci = cy * chi_s, wr = wx * wp_s, wi = wy * wp_s;
    const double inv = 1.0 / (wr * wr + wi * wi + eps);
    sr += (cr * wr + ci * wi) * inv;
    si += (ci * wr - cr * wi) * inv;
  };
  // two pixels per 16-byte load (Q even; rows of A and Y are 16-byte aligned), four loads in flight
  const float4* chi4 = reinterpret_cast<const float4*>(chi);
  const float4* wp4 = reinterpret_cast<const float4*>(wp);
  const int n2 = Q * Q / 2;
#pragma unroll 4
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    const float4 c = __ldg(chi4 + i), w = __ldg(wp4 + i);
    term(c.x, c.y, w.x, w.y);
    term(c.z, c.w, w.z, w.w);
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
  float* Bf = nullptr;
  int ybatch = 0;
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
  cudaFree(w->Bf);
  cudaFree(w->Y);
  cudaFree(w->spec);
  cudaFree(w->dv);
  delete w;
  p.fw = nullptr;
}

// Scan frequencies per Y_v batch: three per SM.  cuFFT's 128 x 128 kernel runs one transform per
// CTA, one CTA per SM, so a batch that is a multiple of the SM count wastes no partial wave, and
// 444 x Q^2 x 8 B stays L2-resident at Q = 128 (measured, Medium / Large: 512 -> 5.49 / 21.5 ms,
// 592 -> 5.20 / 20.3, 444 -> 4.75 / 18.7, 296 -> 5.21 / 20.3)
static int fw_ybatch(const Plan& p) { return 3 * std::max(1, p.sm_count); }

static wdd_status fw_prepare(Plan& p, char* err, size_t errn) {
  if (p.fw && p.fw->ok) return WDD_OK;
  full_wdd_release(p);
  FullWddWork* w = new FullWddWork();
  p.fw = w;
  const int Q = p.Q;
  const int64_t S = p.S, QQ = (int64_t)Q * Q;
  const int64_t nv = std::max<int64_t>(1, p.n_act);
  w->ybatch = fw_ybatch(p);
  const int64_t nv_pad = (nv + w->ybatch - 1) / w->ybatch * w->ybatch;   // (whole batches: see full_wdd)
  if (cudaMalloc(&w->A, (size_t)nv_pad * QQ * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&w->Bf, (size_t)S * QQ * sizeof(float)) != cudaSuccess ||
      cudaMalloc(&w->B, (size_t)QQ * p.Sy * (p.Sx / 2 + 1) * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&w->Y, (size_t)w->ybatch * QQ * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&w->spec, (size_t)S * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&w->dv, p.active_v.size() * sizeof(int32_t)) != cudaSuccess) {
    std::snprintf(err, errn, "full WDD: %.1f GB of device scratch not available", (double)(S + nv) * QQ * 8 / 1e9);   // (Bf + B ~ S x Q^2 x 8 bytes)
    full_wdd_release(p);
    return WDD_E_NOMEM;
  }
  cudaMemset(w->A + nv * QQ, 0, (size_t)(nv_pad - nv) * QQ * sizeof(float2));   // pad rows stay zero under the FFT
  int sdims[2] = {p.Sy, p.Sx}, ddims[2] = {Q, Q};
  std::vector<int32_t> vsorted(p.active_v.begin(), p.active_v.end());   // ascending v: gathers in runs of s
  std::sort(vsorted.begin(), vsorted.end());
  if (cudaMemcpy(w->dv, vsorted.data(), vsorted.size() * sizeof(int32_t), cudaMemcpyHostToDevice) !=
          cudaSuccess ||
      cufftPlanMany(&w->scan, 2, sdims, nullptr, 1, (int)S, nullptr, 1, p.Sy * (p.Sx / 2 + 1), CUFFT_R2C, (int)QQ) !=
          CUFFT_SUCCESS ||
      cufftPlanMany(&w->yplan, 2, ddims, nullptr, 1, (int)QQ, nullptr, 1, (int)QQ, CUFFT_C2C, w->ybatch) !=
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
  if (cufftSetStream(w->scan, st) != CUFFT_SUCCESS ||
      cufftSetStream(w->yplan, st) != CUFFT_SUCCESS || cufftSetStream(w->img, st) != CUFFT_SUCCESS)
    return fail("cuFFT stream");
  if (cudaMemsetAsync(w->spec, 0, (size_t)S * sizeof(float2), st) != cudaSuccess) return fail("memset");
  // (a) frames -> (-1)^m I transposed to pixel-major Bf[m][s]; real-to-complex scan DFT of every
  // pixel (contiguous batches, half plane B[m][vy][vx <= Sx/2]); the active scan frequencies' rows
  // gathered and transposed to A[b][m] for the detector transforms (n_act of S rows: ~45% at
  // Medium / Large)
  const dim3 tb(32, 8);
  const dim3 tg1((unsigned)((QQ + 31) / 32), (unsigned)((S + 31) / 32));
  const dim3 tg1v((unsigned)((QQ + 63) / 64), (unsigned)((S + 63) / 64));
  const bool pair_ok = reinterpret_cast<uintptr_t>(frames_dev) % (p.dtype == 0 ? 4 : 8) == 0 && S % 2 == 0;   // (QQ is even)
  if (p.dtype == 0) {
    if (pair_ok) fw_load2_kernel<uint16_t><<<tg1v, tb, 0, st>>>(static_cast<const uint16_t*>(frames_dev), S, (int)QQ, Q, w->Bf);
    else fw_load_kernel<uint16_t><<<tg1, tb, 0, st>>>(static_cast<const uint16_t*>(frames_dev), S, (int)QQ, Q, w->Bf);
  } else {
    if (pair_ok) fw_load2_kernel<float><<<tg1v, tb, 0, st>>>(static_cast<const float*>(frames_dev), S, (int)QQ, Q, w->Bf);
    else fw_load_kernel<float><<<tg1, tb, 0, st>>>(static_cast<const float*>(frames_dev), S, (int)QQ, Q, w->Bf);
  }
  if (cufftExecR2C(w->scan, w->Bf, reinterpret_cast<cufftComplex*>(w->B)) != CUFFT_SUCCESS) return fail("scan FFT");
  const dim3 tg2((unsigned)((p.n_act + 31) / 32), (unsigned)((QQ + 31) / 32));
  if (p.n_act > 0) fw_gather_transpose_kernel<<<tg2, tb, 0, st>>>(w->B, QQ, p.Sy, p.Sx, w->dv, p.n_act, w->A);
  // (b) chi_v: inverse detector DFT of each gathered scan-frequency row, batch by batch in the
  // loop below with the same cuFFT plan as the probe transforms (at this batch size cuFFT runs the
  // 128 x 128 transform as two 1-D passes, measured faster than its one-kernel 2-D form on all
  // n_act rows at once: Medium 1.18 -> 0.75 ms); the 1/sqrt(S) of the unitary scan DFT is folded
  // into the combine scale.  A is padded to whole batches; the pad rows are transformed, never read.
  // (c) W_P for the active v in batches, Wiener combine and sum
  const double cph = kPi * p.lambda * p.defocus;
  const double chi_s = 1.0 / ((double)Q * std::sqrt((double)S)), wp_s = 1.0 / Q;   // unitary scales
  for (int64_t a = 0; a < p.n_act; a += w->ybatch) {
    const int m = (int)std::min<int64_t>(w->ybatch, p.n_act - a);
    fw_y_kernel<<<m, 256, 4 * Q * sizeof(double2), st>>>(w->dv + a, m, Q, p.dq, p.qa * p.qa, cph, p.Sy, p.Sx,
                                                          p.step, w->Y);
    if (cufftExecC2C(w->yplan, reinterpret_cast<cufftComplex*>(w->A + a * QQ),
                     reinterpret_cast<cufftComplex*>(w->A + a * QQ), CUFFT_INVERSE) != CUFFT_SUCCESS)
      return fail("detector FFT");
    if (cufftExecC2C(w->yplan, reinterpret_cast<cufftComplex*>(w->Y), reinterpret_cast<cufftComplex*>(w->Y),
                     CUFFT_INVERSE) != CUFFT_SUCCESS) return fail("probe FFT");
    fw_combine_kernel<<<m, 256, 0, st>>>(w->A + a * QQ, w->Y, w->dv + a, Q, chi_s, wp_s, p.eps, w->spec);
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
