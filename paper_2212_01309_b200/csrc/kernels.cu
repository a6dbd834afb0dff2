// kernels.cu -- sm_100a kernels of the Live-WDD hot path (Algorithm 2).
//
//   project_kernel  a1-a3: frame ingest + exact count conversion + Hermite-Gauss projection
//                   H(I) = psi_x^T I^T psi_y.  Stage 1 (contraction over detector
//                   columns) runs on the 5th-gen tensor cores: tcgen05.mma kind::f16, A = frame
//                   rows converted in registers to exact fp16, B = [Psi_hi | Psi_lo] fp16 split,
//                   fp32 accumulation in TMEM.  Stage 2 (contraction over detector rows) is fp32.
//   rowdft_kernel   a4: R[j][sy][k] (+)= sum_sx Fx[j][sx] C[(sy,sx)][k]  (F_2D =
//                   F_y (x) F_x), over the active vx columns j only.
//   flush_kernel    a5: G[(j,vy)][k] += sum_rows Fy[vy][sy] R[j][sy][k]  (eq:outer_prod).
//   readout_kernel  a6: o_v = sum_k G[v][k] K_v[k], one warp per active v.
//   finalize        a8: cuFFT C2C inverse + conj / unitary scale / optional 1/sqrt(o_0).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "internal.h"
#include "tc.cuh"

namespace wdd {

using namespace tc;

// =====================================================================================
// Projection (tcgen05)
// =====================================================================================
constexpr int kProjThreads = 128;
constexpr uint32_t kLBO_A = 2064;  // bytes between K-adjacent core matrices of the A tile:
                                   // 16 row groups x 128 B + 16 B pad (rotates banks of STS)

__host__ __device__ constexpr int pow2_cols(int c) { return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512; }
__host__ __device__ constexpr int align_up(int x, int a) { return (x + a - 1) / a * a; }

template <int Q, int L>
struct ProjCfg {
  static constexpr int kChunks = Q / 8;                 // 16-byte K chunks per row
  static constexpr int kA_bytes = kChunks * (int)kLBO_A;
  static constexpr int kN = 2 * L;                      // MMA N: Psi_hi and Psi_lo columns
  static constexpr int kLBO_B = 16 * kN;
  static constexpr int kB_bytes = kChunks * kLBO_B;
  static constexpr int kFPT = Q >= 128 ? 1 : 128 / Q;  // frames per 128-row tile
  static constexpr int kTPU = Q >= 128 ? Q / 128 : 1;  // tiles per work unit
  static constexpr int kTs = L + 1;                     // padded row stride of the T tile
  static constexpr int kOut = kFPT * L * L;             // C outputs per unit
  static constexpr int kOPT = (kOut + kProjThreads - 1) / kProjThreads;
  static constexpr int kTmemCols = pow2_cols(2 * kN);
  static constexpr int off_A = 0;
  static constexpr int off_B = align_up(kA_bytes, 128);
  static constexpr int off_T = off_B + align_up(kB_bytes, 128);
  static constexpr int off_P = off_T + align_up(128 * kTs * 4, 128);
  static constexpr int off_bar = off_P + align_up(Q * L * 4, 128);
  static constexpr int smem = off_bar + 64;
};

__device__ __forceinline__ uint32_t magic_half2(uint32_t v10) {
  // v10 holds two 10-bit integers (bits 0-9 and 16-25).  (0x6400 | x) is fp16 1024 + x,
  // exact; subtracting 1024 leaves x exactly.
  uint32_t bits = v10 | 0x64006400u;
  const __half2 h = *reinterpret_cast<const __half2*>(&bits);
  const __half2 r = __hsub2(h, __half2half2(__ushort_as_half((unsigned short)0x6400)));
  return *reinterpret_cast<const uint32_t*>(&r);
}

// Convert rows [row0, row0+valid) of the frame matrix (n*Q rows of Q pixels) into the
// K-major no-swizzle fp16 A image.  plane 0: u16 -> low 10 bits (exact), f32 -> fp16(x);
// plane 1: u16 -> bits 10..15, f32 -> fp16(x - fp16(x)).  Returns whether plane 1 is nonzero.
template <int Q, bool U16>
__device__ __forceinline__ bool convert_tile(const void* __restrict__ frames, int64_t row0, int valid,
                                             uint8_t* sA, int plane, int tid) {
  constexpr int kChunks = Q / 8;
  constexpr int kPer = kChunks;  // 128 rows * kChunks chunks / 128 threads
  constexpr int G = kPer < 8 ? kPer : 8;
  bool resid = false;
#pragma unroll 1
  for (int base = 0; base < kPer; base += G) {
    if constexpr (U16) {
      uint4 raw[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int c = tid + kProjThreads * (base + g);
        const int r = c / kChunks, j = c % kChunks;
        raw[g] = make_uint4(0, 0, 0, 0);
        if (r < valid) {
          const uint16_t* src = reinterpret_cast<const uint16_t*>(frames) + (row0 + r) * Q + j * 8;
          raw[g] = __ldg(reinterpret_cast<const uint4*>(src));
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int c = tid + kProjThreads * (base + g);
        const int r = c / kChunks, j = c % kChunks;
        uint32_t w[4] = {raw[g].x, raw[g].y, raw[g].z, raw[g].w};
        uint4 o;
        uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          resid |= (w[q] & 0xFC00FC00u) != 0u;
          op[q] = plane == 0 ? magic_half2(w[q] & 0x03FF03FFu) : magic_half2((w[q] >> 10) & 0x003F003Fu);
        }
        *reinterpret_cast<uint4*>(sA + j * kLBO_A + (r >> 3) * 128 + (r & 7) * 16) = o;
      }
    } else {
      float4 raw[2 * G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int c = tid + kProjThreads * (base + g);
        const int r = c / kChunks, j = c % kChunks;
        raw[2 * g] = raw[2 * g + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < valid) {
          const float4* src = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(frames) + (row0 + r) * Q + j * 8);
          raw[2 * g] = __ldg(src);
          raw[2 * g + 1] = __ldg(src + 1);
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int c = tid + kProjThreads * (base + g);
        const int r = c / kChunks, j = c % kChunks;
        const float* x = reinterpret_cast<const float*>(&raw[2 * g]);
        uint4 o;
        __half* hp = reinterpret_cast<__half*>(&o);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const __half h = __float2half_rn(x[e]);
          const float d = x[e] - __half2float(h);
          resid |= d != 0.f;
          hp[e] = plane == 0 ? h : __float2half_rn(d);
        }
        *reinterpret_cast<uint4*>(sA + j * kLBO_A + (r >> 3) * 128 + (r & 7) * 16) = o;
      }
    }
  }
  return resid;
}

template <int Q, int L>
__device__ __forceinline__ void issue_proj_mmas(const uint8_t* sA, const uint8_t* sB, uint32_t tacc) {
  using Cfg = ProjCfg<Q, L>;
  constexpr uint32_t idesc = idesc_f16(128, Cfg::kN);
  const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
#pragma unroll
  for (int kk = 0; kk < Q / 16; ++kk) {
    const uint64_t ad = smem_desc_noswz(a0 + 2 * kk * kLBO_A, kLBO_A, 128);
    const uint64_t bd = smem_desc_noswz(b0 + 2 * kk * Cfg::kLBO_B, Cfg::kLBO_B, 128);
    mma_f16_ss(tacc, ad, bd, idesc, kk > 0 ? 1u : 0u);
  }
}

template <int Q, int L, bool U16>
__global__ void __launch_bounds__(kProjThreads) project_kernel(const void* __restrict__ frames, int64_t n,
                                                               float* __restrict__ C, const uint4* __restrict__ Bpack,
                                                               const float* __restrict__ psi, float inv_scale) {
  using Cfg = ProjCfg<Q, L>;
  constexpr int K = L * L;
  constexpr float kResScale = U16 ? 1024.f : 1.f;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem + Cfg::off_A;
  uint8_t* sB = smem + Cfg::off_B;
  float* sT = reinterpret_cast<float*>(smem + Cfg::off_T);
  float* sP = reinterpret_cast<float*>(smem + Cfg::off_P);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::off_bar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + Cfg::off_bar + 8);
  const int tid = threadIdx.x, warp = tid >> 5;

  for (int i = tid; i < Cfg::kB_bytes / 16; i += kProjThreads) reinterpret_cast<uint4*>(sB)[i] = __ldg(Bpack + i);
  for (int i = tid; i < Q * L; i += kProjThreads) sP[i] = __ldg(psi + i);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<Cfg::kTmemCols>(tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t tlane = tbase + ((uint32_t)(warp * 32) << 16);
  uint32_t phase = 0;

  const int64_t n_units = (n + Cfg::kFPT - 1) / Cfg::kFPT;
  const int64_t total_rows = n * Q;
  for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
    float cacc[Cfg::kOPT];
#pragma unroll
    for (int i = 0; i < Cfg::kOPT; ++i) cacc[i] = 0.f;
#pragma unroll 1
    for (int tt = 0; tt < Cfg::kTPU; ++tt) {
      const int64_t row0 = u * Cfg::kFPT * Q + (int64_t)tt * 128;
      const int64_t rem = total_rows - row0;
      const int valid = rem < 128 ? (int)rem : 128;
      const bool r = convert_tile<Q, U16>(frames, row0, valid, sA, 0, tid);
      fence_proxy_async_smem();
      const int any = __syncthreads_or(r);
      if (tid == 0) {
        tc_fence_after();
        issue_proj_mmas<Q, L>(sA, sB, tbase);
        mma_commit(bar);
      }
      mbar_wait(bar, phase);
      phase ^= 1u;
      tc_fence_after();
      if (any) {  // counts >= 1024 (u16) or non-fp16 values (f32): second plane
        convert_tile<Q, U16>(frames, row0, valid, sA, 1, tid);
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
          tc_fence_after();
          issue_proj_mmas<Q, L>(sA, sB, tbase + Cfg::kN);
          mma_commit(bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1u;
        tc_fence_after();
      }
      // ---- stage-1 epilogue: T[qy][a] = (acc_hi + acc_lo) / scale
      {
        float acc[Cfg::kN];
        tmem_ld_cols<Cfg::kN>(tlane, acc);
        float t[L];
#pragma unroll
        for (int a = 0; a < L; ++a) t[a] = acc[a] + acc[L + a];
        if (any) {
          tmem_ld_cols<Cfg::kN>(tlane + Cfg::kN, acc);
#pragma unroll
          for (int a = 0; a < L; ++a) t[a] = fmaf(kResScale, acc[a] + acc[L + a], t[a]);
        }
#pragma unroll
        for (int a = 0; a < L; ++a) sT[tid * Cfg::kTs + a] = t[a] * inv_scale;
      }
      tc_fence_before();
      __syncthreads();
      // ---- stage 2: C[f][a][b] += sum_qy Psi[qy][b] T[qy][a]
#pragma unroll
      for (int i = 0; i < Cfg::kOPT; ++i) {
        const int o = tid + kProjThreads * i;
        if (o < Cfg::kOut) {
          const int f = o / K, a = (o / L) % L, b = o % L;
          const int r0 = Q >= 128 ? 0 : f * Q;
          const int rn = Q >= 128 ? 128 : Q;
          const int qy0 = Q >= 128 ? tt * 128 : 0;
          float s = 0.f;
#pragma unroll 8
          for (int rr = 0; rr < rn; ++rr) s = fmaf(sP[(qy0 + rr) * L + b], sT[(r0 + rr) * Cfg::kTs + a], s);
          cacc[i] += s;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < Cfg::kOPT; ++i) {
      const int o = tid + kProjThreads * i;
      if (o < Cfg::kOut) {
        const int64_t fg = u * Cfg::kFPT + o / K;
        if (fg < n) C[fg * K + (o % K)] = cacc[i];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<Cfg::kTmemCols>(tbase);
}

template <int Q, int L, bool U16>
static cudaError_t launch_project_t(const Plan& p, const void* frames, int64_t n, float* C, cudaStream_t st) {
  using Cfg = ProjCfg<Q, L>;
  auto kern = project_kernel<Q, L, U16>;
  static int blocks_per_sm = -1;
  if (blocks_per_sm < 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::smem);
    if (e != cudaSuccess) return e;
    int nb = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kProjThreads, Cfg::smem);
    if (e != cudaSuccess) return e;
    blocks_per_sm = std::max(1, std::min(nb, 512 / Cfg::kTmemCols));
  }
  const int64_t units = (n + Cfg::kFPT - 1) / Cfg::kFPT;
  const int grid = (int)std::min<int64_t>(units, (int64_t)blocks_per_sm * p.sm_count);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, kProjThreads, Cfg::smem, st>>>(frames, n, C, reinterpret_cast<const uint4*>(p.d_Bpack), p.d_psi,
                                              (float)(1.0 / p.b_scale));
  return cudaGetLastError();
}

#define WDD_PROJ_CASE(QQ, LL)                                                          \
  if (p.Q == QQ && p.L == LL)                                                          \
    return p.dtype == 0 ? launch_project_t<QQ, LL, true>(p, frames, n, C, st)          \
                        : launch_project_t<QQ, LL, false>(p, frames, n, C, st);

cudaError_t launch_project(const Plan& p, const void* frames, int64_t n, float* C, cudaStream_t st) {
  WDD_PROJ_CASE(32, 8) WDD_PROJ_CASE(32, 16) WDD_PROJ_CASE(32, 24) WDD_PROJ_CASE(32, 32)
  WDD_PROJ_CASE(64, 8) WDD_PROJ_CASE(64, 16) WDD_PROJ_CASE(64, 24) WDD_PROJ_CASE(64, 32)
  WDD_PROJ_CASE(128, 8) WDD_PROJ_CASE(128, 16) WDD_PROJ_CASE(128, 24) WDD_PROJ_CASE(128, 32)
  WDD_PROJ_CASE(256, 8) WDD_PROJ_CASE(256, 16) WDD_PROJ_CASE(256, 24) WDD_PROJ_CASE(256, 32)
  return cudaErrorInvalidValue;
}

size_t project_smem_bytes(int Q, int L) {
#define WDD_SMEM_CASE(QQ, LL) if (Q == QQ && L == LL) return ProjCfg<QQ, LL>::smem;
  WDD_SMEM_CASE(32, 8) WDD_SMEM_CASE(32, 16) WDD_SMEM_CASE(32, 24) WDD_SMEM_CASE(32, 32)
  WDD_SMEM_CASE(64, 8) WDD_SMEM_CASE(64, 16) WDD_SMEM_CASE(64, 24) WDD_SMEM_CASE(64, 32)
  WDD_SMEM_CASE(128, 8) WDD_SMEM_CASE(128, 16) WDD_SMEM_CASE(128, 24) WDD_SMEM_CASE(128, 32)
  WDD_SMEM_CASE(256, 8) WDD_SMEM_CASE(256, 16) WDD_SMEM_CASE(256, 24) WDD_SMEM_CASE(256, 32)
#undef WDD_SMEM_CASE
  return 0;
}

// B operand image: rows n < L hold fp16(Psi*s) (hi), rows L..2L-1 the fp16 residual (lo),
// s = 2^e chosen so max|Psi|*s ~ 2^14 (keeps the residual out of fp16 subnormals).
void pack_basis_fp16(const Plan& p, std::vector<uint16_t>& out, double& scale) {
  const int Q = p.Q, L = p.L, kN = 2 * L;
  double mx = 0;
  for (double v : p.basis) mx = std::max(mx, std::fabs(v));
  const int e = (int)std::floor(std::log2(16384.0 / mx));
  scale = std::ldexp(1.0, e);
  out.assign((size_t)(Q / 8) * 16 * kN / 2, 0);
  for (int m = 0; m < Q; ++m) {
    for (int nr = 0; nr < kN; ++nr) {
      const int a = nr % L;
      const double v = p.basis[(size_t)m * L + a] * scale;
      const __half hi = __float2half_rn((float)v);
      const __half h = nr < L ? hi : __float2half_rn((float)(v - (double)__half2float(hi)));
      const size_t byte = (size_t)(m / 8) * 16 * kN + (nr / 8) * 128 + (nr % 8) * 16 + (m % 8) * 2;
      out[byte / 2] = __half_as_ushort(h);
    }
  }
}

// =====================================================================================
// Row DFT (a4): R[j][sy][k] (+)= sum_{frames of row sy in chunk} Fx[j][sx] C[p][k]
// =====================================================================================
__global__ void __launch_bounds__(256) rowdft_kernel(const float* __restrict__ C, RowSource rs,
                                                     const float2* __restrict__ Fx, float2* __restrict__ R,
                                                     int Sx, int Sy, int K, int n_vx) {
  __shared__ float Cs[32][64];
  __shared__ float2 Fs[32][33];
  const int t = threadIdx.x, kk = t & 63, jg = t >> 6;
  const int k0 = blockIdx.x * 64, j0 = blockIdx.y * 32, r = blockIdx.z;
  int sy, count, mode, pb = 0, eb = 0, sx0 = 0;
  if (rs.contiguous) {
    const int sy0 = rs.s0 / Sx;
    sx0 = rs.s0 % Sx;
    sy = sy0 + r;
    pb = max(0, r * Sx - sx0);
    const int pe = min(rs.n, (r + 1) * Sx - sx0);
    count = pe - pb;
    mode = r == 0 ? rs.mode_first : (r == rs.n_rows - 1 ? rs.mode_last : 0);
  } else {
    const int4 ri = rs.rows[r];
    sy = ri.x;
    eb = ri.y;
    count = ri.z;
    mode = ri.w;
  }
  float2 acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = make_float2(0.f, 0.f);
  for (int e0 = 0; e0 < count; e0 += 32) {
    const int ne = min(32, count - e0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = t + 256 * i, ee = idx >> 6, kq = idx & 63;
      float v = 0.f;
      if (ee < ne && k0 + kq < K) {
        const int p = rs.contiguous ? pb + e0 + ee : rs.ent[eb + e0 + ee].x;
        v = C[(int64_t)p * K + k0 + kq];
      }
      Cs[ee][kq] = v;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = t + 256 * i, jj = idx >> 5, ee = idx & 31;
      float2 v = make_float2(0.f, 0.f);
      if (ee < ne && j0 + jj < n_vx) {
        const int sx = rs.contiguous ? sx0 + pb + e0 + ee - r * Sx : rs.ent[eb + e0 + ee].y;
        v = Fx[(int64_t)(j0 + jj) * Sx + sx];
      }
      Fs[jj][ee] = v;
    }
    __syncthreads();
    for (int ee = 0; ee < ne; ++ee) {
      const float c = Cs[ee][kk];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float2 f = Fs[jg * 8 + q][ee];
        acc[q].x = fmaf(f.x, c, acc[q].x);
        acc[q].y = fmaf(f.y, c, acc[q].y);
      }
    }
    __syncthreads();
  }
  const int k = k0 + kk;
  if (k >= K) return;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int j = j0 + jg * 8 + q;
    if (j < n_vx) {
      float2* ptr = R + ((int64_t)j * Sy + sy) * K + k;
      if (mode) {
        const float2 o = *ptr;
        *ptr = make_float2(o.x + acc[q].x, o.y + acc[q].y);
      } else {
        *ptr = acc[q];
      }
    }
  }
}

cudaError_t launch_rowdft(const Plan& p, const float* C, const RowSource& rs, cudaStream_t st) {
  if (rs.n_rows <= 0) return cudaSuccess;
  dim3 grid((p.K + 63) / 64, (p.n_vx + 31) / 32, rs.n_rows);
  rowdft_kernel<<<grid, 256, 0, st>>>(C, rs, p.d_Fx, p.d_R, p.Sx, p.Sy, p.K, p.n_vx);
  return cudaGetLastError();
}

// =====================================================================================
// Flush (a5): G[(j,vy)][k] += sum_{staged rows} Fy[vy][sy] R[j][sy][k]
// =====================================================================================
__global__ void __launch_bounds__(256) flush_kernel(const float2* __restrict__ R, const float2* __restrict__ Fy,
                                                    const int32_t* __restrict__ rows, int n_rows,
                                                    const int2* __restrict__ tiles, const int32_t* __restrict__ col_off,
                                                    const int32_t* __restrict__ act_vy, float2* __restrict__ G,
                                                    int Sy, int K) {
  __shared__ float2 Rs[32][64];
  __shared__ float2 Fs[32][33];
  __shared__ int vys[32];
  const int t = threadIdx.x, kk = t & 63, ig = t >> 6;
  const int2 tile = tiles[blockIdx.x];
  const int j = tile.x, i0 = tile.y, k0 = blockIdx.y * 64;
  const int g0 = col_off[j], mj = col_off[j + 1] - g0;
  if (t < 32) vys[t] = (i0 + t < mj) ? act_vy[g0 + i0 + t] : -1;
  __syncthreads();
  float2 acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = make_float2(0.f, 0.f);
  for (int r0 = 0; r0 < n_rows; r0 += 32) {
    const int nr = min(32, n_rows - r0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = t + 256 * i, rr = idx >> 6, kq = idx & 63;
      float2 v = make_float2(0.f, 0.f);
      if (rr < nr && k0 + kq < K) v = R[((int64_t)j * Sy + rows[r0 + rr]) * K + k0 + kq];
      Rs[rr][kq] = v;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = t + 256 * i, ii = idx >> 5, rr = idx & 31;
      float2 v = make_float2(0.f, 0.f);
      if (rr < nr && vys[ii] >= 0) v = Fy[(int64_t)vys[ii] * Sy + rows[r0 + rr]];
      Fs[ii][rr] = v;
    }
    __syncthreads();
    for (int rr = 0; rr < nr; ++rr) {
      const float2 x = Rs[rr][kk];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float2 f = Fs[ig * 8 + q][rr];
        acc[q].x = fmaf(f.x, x.x, fmaf(-f.y, x.y, acc[q].x));
        acc[q].y = fmaf(f.x, x.y, fmaf(f.y, x.x, acc[q].y));
      }
    }
    __syncthreads();
  }
  const int k = k0 + kk;
  if (k >= K) return;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + ig * 8 + q;
    if (i < mj) {
      float2* ptr = G + (int64_t)(g0 + i) * K + k;
      const float2 o = *ptr;
      *ptr = make_float2(o.x + acc[q].x, o.y + acc[q].y);
    }
  }
}

cudaError_t launch_flush(const Plan& p, const int32_t* rows, int n_rows, cudaStream_t st) {
  if (n_rows <= 0) return cudaSuccess;
  dim3 grid((unsigned)p.flush_tiles.size(), (p.K + 63) / 64);
  flush_kernel<<<grid, 256, 0, st>>>(p.d_R, p.d_Fy, rows, n_rows, p.d_flush_tiles, p.d_col_off, p.d_act_vy,
                                     p.d_G, p.Sy, p.K);
  return cudaGetLastError();
}

// =====================================================================================
// Readout (a6): o_v = sum_k G[v][k] W[v][k], one warp per active v
// =====================================================================================
__global__ void __launch_bounds__(256) readout_kernel(const float2* __restrict__ G, const float2* __restrict__ W,
                                                      int64_t n_act, int K, float2* __restrict__ o,
                                                      const int32_t* __restrict__ vpos, float2* __restrict__ spec) {
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= n_act) return;
  const float4* Gr = reinterpret_cast<const float4*>(G + g * K);
  const float4* Wr = reinterpret_cast<const float4*>(W + g * K);
  float re = 0.f, im = 0.f;
  for (int i = lane; i < K / 2; i += 32) {
    const float4 a = __ldg(Gr + i), b = __ldg(Wr + i);
    re = fmaf(a.x, b.x, fmaf(-a.y, b.y, re));
    im = fmaf(a.x, b.y, fmaf(a.y, b.x, im));
    re = fmaf(a.z, b.z, fmaf(-a.w, b.w, re));
    im = fmaf(a.z, b.w, fmaf(a.w, b.z, im));
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, s);
    im += __shfl_xor_sync(0xffffffffu, im, s);
  }
  if (lane == 0) {
    o[g] = make_float2(re, im);
    if (spec) spec[vpos[g]] = make_float2(re, im);
  }
}

cudaError_t launch_readout(const Plan& p, const float2* G, bool scatter, cudaStream_t st) {
  const int64_t threads = p.n_act * 32;
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  readout_kernel<<<blocks, 256, 0, st>>>(G, p.d_W, p.n_act, p.K, p.d_o, p.d_vpos, scatter ? p.d_spec : nullptr);
  return cudaGetLastError();
}

__global__ void scatter_kernel(const float2* __restrict__ o, const int32_t* __restrict__ vpos, int64_t n_act,
                               float2* __restrict__ spec) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < n_act) spec[vpos[g]] = o[g];
}

cudaError_t launch_scatter(const Plan& p, cudaStream_t st) {
  scatter_kernel<<<(unsigned)((p.n_act + 255) / 256), 256, 0, st>>>(p.d_o, p.d_vpos, p.n_act, p.d_spec);
  return cudaGetLastError();
}

// =====================================================================================
// Finalize (a8): out = conj(IDFT2(o)) / sqrt(S) [/ sqrt(o_0)]; the IDFT itself is cuFFT.
// =====================================================================================
__global__ void conj_scale_kernel(float2* __restrict__ out, int64_t S, double inv_sqrt_s,
                                  const float2* __restrict__ spec, int normalize) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S) return;
  double xr = out[i].x * inv_sqrt_s, xi = -out[i].y * inv_sqrt_s;
  if (normalize) {
    // principal sqrt of o_0
    const double a = spec[0].x, b = spec[0].y;
    const double r = hypot(a, b);
    double wr = 0, wi = 0;
    if (r > 0) {
      const double s = sqrt(0.5 * (r + fabs(a)));
      if (a >= 0) { wr = s; wi = b / (2 * s); }
      else { wr = fabs(b) / (2 * s); wi = copysign(s, b); }
    }
    const double d = wr * wr + wi * wi;
    if (d > 0) {
      const double yr = (xr * wr + xi * wi) / d, yi = (xi * wr - xr * wi) / d;
      xr = yr;
      xi = yi;
    }
  }
  out[i] = make_float2((float)xr, (float)xi);
}

cudaError_t launch_finalize(const Plan& p, float2* out, cudaStream_t st) {
  if (cufftSetStream(p.fft, st) != CUFFT_SUCCESS) return cudaErrorUnknown;
  if (cufftExecC2C(p.fft, reinterpret_cast<cufftComplex*>(p.d_spec), reinterpret_cast<cufftComplex*>(out),
                   CUFFT_INVERSE) != CUFFT_SUCCESS)
    return cudaErrorUnknown;
  const int64_t S = p.S;
  conj_scale_kernel<<<(unsigned)((S + 255) / 256), 256, 0, st>>>(out, S, 1.0 / std::sqrt((double)S), p.d_spec,
                                                                 p.normalize);
  return cudaGetLastError();
}

}  // namespace wdd
