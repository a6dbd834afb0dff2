// Plan-time Wiener bank on the GPU (Algorithm 1):
//   Y_v[my][mx] = p_hat(q_m) conj(p_hat(q_m + q_hat_v))          (R7, R8)
//   H(Y_v)[a][b] = sum_my sum_mx Psi[mx][a] Psi[my][b] Y_v[my][mx] (k = a*L + b, R5)
//   K_v[k] = conj(H[k]) / (|H[k]|^2 + eps)                        (R11)
// for every active v, in float64.  Y_v is non-zero only on the lens where the aperture and the
// shifted aperture overlap; on a detector row both are pixel intervals, so each row of the lens
// is one interval [lo, hi] found by bisection with the same float64 membership test as the
// active-set search (products and sums rounded separately, no FMA contraction: R10).  With
// p_hat = exp(-i pi lambda df |q|^2) the phase of Y_v separates into a row factor and a column
// factor, exp(i c (2 qy sy + sy^2)) exp(i c (2 qx sx + sx^2)) with c = pi lambda df, so for one
// scan-frequency column vx the column factor times Psi is a table E[mx][a] shared by all its vy.
// One CTA = up to 32 active v of one vx column (the flush tiles); 256 threads.
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace wdd {
namespace {

constexpr int kBankThreads = 256;
constexpr int kBankRows = 32;   // detector rows per stage-2 chunk

__device__ __forceinline__ double scan_freq(int v, int S, double step) {
  const int sf = v < (S + 1) / 2 ? v : v - S;   // fftfreq (R15)
  return (double)sf / __dmul_rn((double)S, step);
}

// s2 = (qy + sy)^2 + (qx + sx)^2 <= qa2 with every operation rounded on its own (R10)
__device__ __forceinline__ bool in_shifted(double a, double qx, double sx, double qa2) {
  const double b = __dadd_rn(qx, sx);
  return __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)) <= qa2;
}

template <typename OutT>
__global__ void __launch_bounds__(kBankThreads) bank_kernel(
    const double* __restrict__ psi, const double* __restrict__ q, const int2* __restrict__ apx, int ax_lo,
    int n_axc, const int2* __restrict__ tiles, const int32_t* __restrict__ col_vx,
    const int32_t* __restrict__ col_off, const int32_t* __restrict__ act_vy, int Q, int L, int Sy, int Sx,
    double step, double qa2, double cph, double eps, OutT* __restrict__ W) {
  extern __shared__ __align__(16) double2 bsm[];
  const int K = L * L;
  double2* E = bsm;                                   // n_axc x L
  double2* T = E + (size_t)n_axc * L;                 // kBankRows x L
  double2* rho = T + kBankRows * L;                   // kBankRows
  double* psic = reinterpret_cast<double*>(rho + kBankRows);   // kBankRows x L
  int2* lens = reinterpret_cast<int2*>(psic + kBankRows * L);  // Q
  __shared__ int srange[2][2];   // [v parity][min row, max row] of the lens
  const int tid = threadIdx.x;
  const int2 tile = tiles[blockIdx.x];
  const int j = tile.x;
  const int g0 = col_off[j] + tile.y, g1 = min(col_off[j + 1], g0 + 32);
  const double sx = scan_freq(col_vx[j], Sx, step);
  const double sx2 = __dmul_rn(sx, sx);
  // E[mx][a] = Psi[mx][a] exp(i cph (2 qx sx + sx^2)) over the aperture's column range
  for (int e = tid; e < n_axc * L; e += kBankThreads) {
    const int mx = ax_lo + e / L, a = e % L;
    double s, c;
    sincos(cph * (2.0 * q[mx] * sx + sx2), &s, &c);
    const double ps = psi[(size_t)mx * L + a];
    E[e] = make_double2(ps * c, ps * s);
  }
  constexpr int kMaxAcc = 4;   // K <= 1024 = 4 x 256
  for (int g = g0; g < g1; ++g) {
    const double sy = scan_freq(act_vy[g], Sy, step);
    const double sy2 = __dmul_rn(sy, sy);
    int* rng = srange[g & 1];   // alternating: the previous v's range may still be being read
    if (tid == 0) {
      rng[0] = Q;
      rng[1] = -1;
    }
    __syncthreads();   // E ready; the previous v's use of lens / srange is over
    // lens interval of each detector row
    for (int my = tid; my < Q; my += kBankThreads) {
      int2 iv = make_int2(1, 0);
      const int2 ap = apx[my];
      if (ap.x <= ap.y) {
        const double a = __dadd_rn(q[my], sy);
        // column of minimal |qx + sx| inside [ap.x, ap.y]: first b >= 0, or its left neighbour
        int lo = ap.x, hi = ap.y + 1;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (__dadd_rn(q[mid], sx) >= 0.0) hi = mid; else lo = mid + 1;
        }
        int ms = min(lo, ap.y);
        if (ms > ap.x && fabs(__dadd_rn(q[ms - 1], sx)) <= fabs(__dadd_rn(q[ms], sx))) --ms;
        if (in_shifted(a, q[ms], sx, qa2)) {
          int l0 = ap.x, l1 = ms;            // first member in [ap.x, ms]
          while (l0 < l1) {
            const int mid = (l0 + l1) >> 1;
            if (in_shifted(a, q[mid], sx, qa2)) l1 = mid; else l0 = mid + 1;
          }
          int r0 = ms, r1 = ap.y;            // last member in [ms, ap.y]
          while (r0 < r1) {
            const int mid = (r0 + r1 + 1) >> 1;
            if (in_shifted(a, q[mid], sx, qa2)) r0 = mid; else r1 = mid - 1;
          }
          iv = make_int2(l0 - ax_lo, r0 - ax_lo);
          atomicMin(&rng[0], my);
          atomicMax(&rng[1], my);
        }
      }
      lens[my] = iv;
    }
    __syncthreads();
    const int rmin = rng[0], rmax = rng[1];
    double2 H[kMaxAcc];
#pragma unroll
    for (int u = 0; u < kMaxAcc; ++u) H[u] = make_double2(0.0, 0.0);
    for (int r0 = rmin; r0 <= rmax; r0 += kBankRows) {
      // row factors and the chunk's basis rows
      if (tid < kBankRows) {
        const int my = r0 + tid;
        double2 f = make_double2(0.0, 0.0);
        if (my <= rmax) {
          double s, c;
          sincos(cph * (2.0 * q[my] * sy + sy2), &s, &c);
          f = make_double2(c, s);
        }
        rho[tid] = f;
      }
      for (int e = tid; e < kBankRows * L; e += kBankThreads) {
        const int my = r0 + e / L;
        psic[e] = my <= rmax ? psi[(size_t)my * L + e % L] : 0.0;
      }
      __syncthreads();
      // stage 1: T[r][a] = rho_r sum_{mx in lens row} E[mx][a]
      for (int e = tid; e < kBankRows * L; e += kBankThreads) {
        const int r = e / L, a = e % L, my = r0 + r;
        double2 acc = make_double2(0.0, 0.0);
        if (my <= rmax) {
          const int2 iv = lens[my];
          for (int x = iv.x; x <= iv.y; ++x) {
            const double2 v = E[x * L + a];
            acc.x += v.x;
            acc.y += v.y;
          }
        }
        const double2 f = rho[r];
        T[e] = make_double2(acc.x * f.x - acc.y * f.y, acc.x * f.y + acc.y * f.x);
      }
      __syncthreads();
      // stage 2: H[a][b] += sum_r Psi[my][b] T[r][a]
#pragma unroll
      for (int u = 0; u < kMaxAcc; ++u) {
        const int k = tid + u * kBankThreads;
        if (k < K) {
          const int a = k / L, b = k % L;
          double2 h = H[u];
          for (int r = 0; r < kBankRows; ++r) {
            const double w = psic[r * L + b];
            const double2 t = T[r * L + a];
            h.x = fma(w, t.x, h.x);
            h.y = fma(w, t.y, h.y);
          }
          H[u] = h;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < kMaxAcc; ++u) {
      const int k = tid + u * kBankThreads;
      if (k < K) {
        const double den = H[u].x * H[u].x + H[u].y * H[u].y + eps;
        const double wr = H[u].x / den, wi = -H[u].y / den;
        if constexpr (sizeof(OutT) == sizeof(double2))
          W[(size_t)g * K + k] = OutT{wr, wi};
        else
          W[(size_t)g * K + k] = OutT{__double2float_rn(wr), __double2float_rn(wi)};
      }
    }
  }
}

}  // namespace

// Uploads the float64 tables the kernel needs (basis, detector grid, aperture row intervals),
// runs the bank kernel into W_dev (complex64, or complex128 when f64) and waits for it.
cudaError_t build_bank(const Plan& p, const double* q_host, const int2* apx_host, int ax_lo, int n_axc, void* W_dev,
                       bool f64) {
  if (p.K > kBankThreads * 4) return cudaErrorInvalidValue;
  double *d_psi = nullptr, *d_q = nullptr;
  int2* d_apx = nullptr;
  cudaError_t e = cudaMalloc(&d_psi, p.basis.size() * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_q, (size_t)p.Q * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_apx, (size_t)p.Q * sizeof(int2));
  if (e == cudaSuccess) e = cudaMemcpy(d_psi, p.basis.data(), p.basis.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_q, q_host, (size_t)p.Q * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_apx, apx_host, (size_t)p.Q * sizeof(int2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    const size_t smem = (size_t)n_axc * p.L * sizeof(double2) + kBankRows * p.L * sizeof(double2) +
                        kBankRows * sizeof(double2) + kBankRows * p.L * sizeof(double) + (size_t)p.Q * sizeof(int2);
    const double cph = kPi * p.lambda * p.defocus;   // -(c0) of p_hat's exponent, P:447 with R7
    const dim3 grid((unsigned)p.flush_tiles.size());
    if (f64) {
      e = cudaFuncSetAttribute(bank_kernel<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess)
        bank_kernel<double2><<<grid, kBankThreads, smem>>>(d_psi, d_q, d_apx, ax_lo, n_axc, p.d_flush_tiles,
                                                             p.d_col_vx, p.d_col_off, p.d_act_vy, p.Q, p.L, p.Sy,
                                                             p.Sx, p.step, p.qa * p.qa, cph, p.eps,
                                                             static_cast<double2*>(W_dev));
    } else {
      e = cudaFuncSetAttribute(bank_kernel<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess)
        bank_kernel<float2><<<grid, kBankThreads, smem>>>(d_psi, d_q, d_apx, ax_lo, n_axc, p.d_flush_tiles,
                                                            p.d_col_vx, p.d_col_off, p.d_act_vy, p.Q, p.L, p.Sy,
                                                            p.Sx, p.step, p.qa * p.qa, cph, p.eps,
                                                            static_cast<float2*>(W_dev));
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  cudaFree(d_psi);
  cudaFree(d_q);
  cudaFree(d_apx);
  return e;
}

}  // namespace wdd
