// fft.cuh -- shared-memory FFTs for the scan-frequency transforms of the Live-WDD path.
//
// The unitary scan DFT F_2D = F_y (x) F_x is applied along one scan axis at
// a time to many independent sequences (one per coefficient k, or per image column).  For a
// power-of-two length N = N1 * N2 this is the four-step (Cooley-Tukey) factorisation:
//   step 1  for each n2 < N2:  y[n2][k1] = W_N^{n2 k1} * sum_{n1} x[N2 n1 + n2] W_N1^{n1 k1}
//   step 2  for each k1 < N1:  X[k1 + N1 k2] = sum_{n2} y[n2][k1] W_N2^{n2 k2}
// Each thread owns one short DFT (N1 or N2 <= 32 points) held entirely in registers (radix-2
// DIT, compile-time unrolled), so a length-N transform costs two register passes and one
// shared-memory exchange instead of log2(N) synchronised shared-memory passes.
#pragma once
#include <cstdint>

namespace wdd {
namespace fft {

// Complex arithmetic on packed fp32 pairs (sm_100 FADD2 / FMUL2 / FFMA2: one instruction per
// complex add, two per complex multiply; each lane rounds exactly as the scalar expression in the
// comment, so results are bit-identical to the scalar forms).
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }   // a + b
__device__ __forceinline__ float2 csub(float2 a, float2 b) {                              // a - b
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
// (fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x))
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return __ffma2_rn(make_float2(a.x, a.x), b, __fmul2_rn(make_float2(-b.y, b.x), make_float2(a.y, a.y)));
}

__host__ __device__ constexpr int brev_c(int v, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((v >> i) & 1) << (bits - 1 - i);
  return r;
}

// cos / sin of 2 pi q / 32, q < 16, as compile-time constants (float-rounded exact values)
__host__ __device__ constexpr float cos32(int q) {
  return q == 0 ? 1.f : q == 1 ? 9.807852804e-01f : q == 2 ? 9.238795325e-01f : q == 3 ? 8.314696123e-01f
       : q == 4 ? 7.071067812e-01f : q == 5 ? 5.555702330e-01f : q == 6 ? 3.826834324e-01f : q == 7 ? 1.950903220e-01f
       : q == 8 ? 0.f : q == 9 ? -1.950903220e-01f : q == 10 ? -3.826834324e-01f : q == 11 ? -5.555702330e-01f
       : q == 12 ? -7.071067812e-01f : q == 13 ? -8.314696123e-01f : q == 14 ? -9.238795325e-01f : -9.807852804e-01f;
}
// v * W_32^q = v * exp(-2 pi i q / 32) with q a compile-time constant after unrolling
__device__ __forceinline__ float2 rot32(float2 v, int q) {
  if (q == 0) return v;
  if (q == 8) return make_float2(v.y, -v.x);                        // times -i
  const float c = cos32(q), sn = q < 8 ? cos32(8 - q) : cos32(q - 8);
  // exp(-i t) = cos t - i sin t; sin(2 pi q/32) = cos(2 pi (8 - q)/32) for q < 8, = cos(2 pi (q - 8)/32) for q >= 8
  // (fmaf(v.x, c, v.y * sn), fmaf(v.y, c, -v.x * sn))
  return __ffma2_rn(v, make_float2(c, c), __fmul2_rn(make_float2(v.y, -v.x), make_float2(sn, sn)));
}

// One radix-2 DIT stage (butterfly span LEN) of an in-register DFT of R <= 32 points; recursion
// over LEN keeps every register index and twiddle a compile-time constant.
template <int R, int LEN>
__device__ __forceinline__ void dft_stage(float2 (&v)[R]) {
  if constexpr (LEN <= R) {
#pragma unroll
    for (int i = 0; i < R; i += LEN) {
#pragma unroll
      for (int j = 0; j < LEN / 2; ++j) {
        const float2 a = v[i + j];
        const float2 b = rot32(v[i + j + LEN / 2], j * (32 / LEN));   // W_LEN^j = W_32^{32 j / LEN}
        v[i + j] = cadd(a, b);
        v[i + j + LEN / 2] = csub(a, b);
      }
    }
    dft_stage<R, 2 * LEN>(v);
  }
}

// In-register forward DFT of R = 2^LR <= 32 points (natural order in and out).
template <int LR>
__device__ __forceinline__ void dft_reg(float2 (&v)[1 << LR]) {
  static_assert(LR <= 5, "register DFT up to 32 points");
  constexpr int R = 1 << LR;
  float2 u[R];
#pragma unroll
  for (int i = 0; i < R; ++i) u[i] = v[brev_c(i, LR)];
  dft_stage<R, 2>(u);
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = u[i];
}

template <int LOGN> struct Split {
  static constexpr int L1 = (LOGN + 1) / 2, L2 = LOGN - L1;
  static constexpr int N1 = 1 << L1, N2 = 1 << L2;
};

// Slot holding frequency f after fft_seq<LOGN>.
template <int LOGN>
__device__ __forceinline__ int fslot(int f) {
  using S = Split<LOGN>;
  return S::N2 * (f & (S::N1 - 1)) + (f >> S::L1);
}

// Forward DFT (unnormalised, e^{-2 pi i}) of 2^logc interleaved sequences of length N = 2^LOGN
// stored in shared memory as x[n * cnt + c] (sequence index fastest: a warp touches consecutive
// addresses), plus PAD float2 after every block of N2 positions (pidx below; PAD = 8 makes the
// second step's 8-sequence tiles conflict-free: consecutive blocks then start half a bank row
// apart).  LOGC >= 0 fixes logc at compile time, so every shared-memory address of a thread is
// one base register plus an immediate offset.  Input in natural order; frequency f ends at slot
// fslot<LOGN>(f).  tw = the full table tw[m] = exp(-2 pi i m / N), m < N, in shared memory, or in
// global memory read through the L1 (TWG: no per-CTA copy; only the step-2 twiddles W_N^{n2 k1}
// read it).  Starts and ends with the block synchronised.
template <int LOGN, int PAD = 0>
__device__ __forceinline__ int pidx(int n, int logc) {
  return (n << logc) + (n >> Split<LOGN>::L2) * PAD;
}
template <int LOGN, int LOGC = -1, int PAD = 0, bool TWG = false>
__device__ __forceinline__ void fft_seq(float2* x, const float2* tw, int logc_rt) {
  using S = Split<LOGN>;
  constexpr int N1 = S::N1, N2 = S::N2;
  const int logc = LOGC >= 0 ? LOGC : logc_rt;
  const int cnt = 1 << logc;
  const int bs = (N2 << logc) + PAD;       // stride between blocks of N2 positions
  for (int t = threadIdx.x; t < (N2 << logc); t += blockDim.x) {
    const int c = t & (cnt - 1), n2 = t >> logc;
    float2* xb = x + (n2 << logc) + c;
    float2 v[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) v[n1] = xb[n1 * bs];
    dft_reg<S::L1>(v);
    if (N2 > 1) {
#pragma unroll
      for (int k1 = 1; k1 < N1; ++k1) v[k1] = cmul(v[k1], TWG ? __ldg(tw + n2 * k1) : tw[n2 * k1]);
    }
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) xb[k1 * bs] = v[k1];
  }
  __syncthreads();
  if (N2 > 1) {
    for (int t = threadIdx.x; t < (N1 << logc); t += blockDim.x) {
      const int c = t & (cnt - 1), k1 = t >> logc;
      float2* xb = x + k1 * bs + c;
      float2 v[N2];
#pragma unroll
      for (int n2 = 0; n2 < N2; ++n2) v[n2] = xb[n2 << logc];
      dft_reg<S::L2>(v);
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) xb[k2 << logc] = v[k2];
    }
    __syncthreads();
  }
}

}  // namespace fft
}  // namespace wdd
