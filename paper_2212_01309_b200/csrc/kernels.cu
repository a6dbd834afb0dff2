// kernels.cu -- sm_100a kernels of the Live-WDD hot path (Algorithm 2).
//
//   project_kernel  a1-a3: frame ingest + exact count conversion + Hermite-Gauss projection
//                   H(I) = psi_x^T I^T psi_y.  Stage 1 (contraction over detector
//                   columns) runs on the 5th-gen tensor cores: tcgen05.mma kind::f16, A = frame
//                   rows converted in registers to exact fp16, B = [Psi_hi | Psi_lo] fp16 split,
//                   fp32 accumulation in TMEM.  Stage 2 (contraction over detector rows) runs on the
//                   tensor cores too, with T split into fp16 hi/lo planes.
//   rowfft_kernel   a4: R[j][sy][k] = sum_sx Fx[j][sx] C[(sy,sx)][k]  (F_2D =
//                   F_y (x) F_x), over the active vx columns j only (radix-2 FFT in
//                   shared memory; rowdft_kernel is the DFT-matrix form for other row lengths).
//   colfft_kernel   a5: G[(j,vy)][k] += sum_rows Fy[vy][sy] R[j][sy][k]  (eq:outer_prod)
//                   (FFT along y; flush_kernel is the DFT-matrix form for a few staged rows).
//   readout_kernel  a6: o_v = sum_k G[v][k] K_v[k], one warp per active v.
//   finalize        a8: cuFFT C2C inverse + conj / unitary scale / optional 1/sqrt(o_0).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <climits>
#include <type_traits>
#include <cmath>
#include <ctime>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_bf16.h>
#include <mutex>
#include <set>
#include <tuple>
#include <vector>

#include "internal.h"
#include "tc.cuh"
#include "fft.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace wdd {

using namespace tc;

// =====================================================================================
// Projection (tcgen05), warp-specialised and persistent.
//
//   warp 0       stage-1 MMA issuer : T_tile (128 rows x 2L) += A1 * B^T            (TMEM acc1)
//   warp 1       stage-2 MMA issuer : D (128 x 2L) += A2 * B^T over qy, hi+lo planes (TMEM acc2)
//   warp 2       TMA producer (u16) : 2-D tiled loads of 128 detector rows x 64 pixels with hardware
//                                     swizzle into a shared-memory ring (ragged tails zero-filled)
//   warps 3-10   converters (2 groups of 4 warps, even / odd chunks)
//                                   : one detector row per thread: swizzled LDS -> exact fp16 in
//                                     registers (counts split into low 10 bits + bits 10-15 x 1024)
//                                     -> tcgen05.st into a TMEM A ring; the raw slot is released as
//                                     soon as it has been read.  f32 frames: LDG -> fp16(x) +
//                                     fp16(x - fp16(x)) into shared-memory operand slots instead.
//   warps 11-14  epilogue           : acc1 -> T -> fp16 hi/lo A2 image (smem); acc2 -> C (global)
//
// Stage 1 contracts the detector columns (qx) for 128 detector rows at a time; stage 2 contracts
// the detector rows (qy) for g2 <= 128/L frames at a time, M = (frame, a) rows, in K-chunks of
// 128 rows (two for Q = 256).  Both stages use the same B image [Psi_hi | Psi_lo] (N = 2L).
// g2 is chosen per launch so a small batch still spreads over every SM.
// =====================================================================================
#ifdef WDD_TRACE
__device__ unsigned long long g_trace[16 * 4096];
__device__ __forceinline__ void trace_rec(int code, unsigned& cnt, int j) {
  if (blockIdx.x != 0) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_trace[code * 4096 + (cnt++ & 4095)] = (t << 16) | ((unsigned long long)(code & 0xff) << 8) | (unsigned long long)(j & 0xff);
}
#define TRACE(c, j) trace_rec(c, trc[c], j)
#define TRACE_DECL unsigned trc[16] = {0};
// per-CTA timeline of every projection CTA: [entry, first TMA issue, last raw landing, exit, smid]
__device__ unsigned long long g_cta[8192][5];
__device__ unsigned g_cta_n;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CTA_REC(slot, field) do { if ((slot) < 8192) g_cta[slot][field] = gtime(); } while (0)
#else
#define TRACE(c, j)
#define TRACE_DECL
#endif
#ifndef WDD_NS
#define WDD_NS 8
#endif
#ifndef WDD_LEAN
#define WDD_LEAN 1
#endif
// WDD_LEAN: two CTAs per SM (one converter group, shallower rings, <= 113 KB smem, <= 256 TMEM
// columns) so that one CTA's pipeline fill / drain overlaps the other's streaming.
constexpr bool kLeanAllowed = WDD_LEAN != 0;   // per configuration: lean only where it fits
constexpr int kConv = 128;          // threads per converter group (2 groups: even / odd chunks)
#ifndef WDD_LEAN_SMEM
#define WDD_LEAN_SMEM (110 * 1024)    // two CTAs per SM (measured: 112.3 KB and 114 968 B CTAs ran one per SM)
#endif
constexpr int kLeanSmem = WDD_LEAN_SMEM;   // shared-memory budget of a lean (two CTAs per SM) projection CTA
constexpr uint32_t kLBO = 2064;     // no-swizzle K-major: bytes between K-adjacent core matrices of a
                                    // 128-row operand (16 row groups x 128 B + 16 B bank-rotation pad)

__host__ __device__ constexpr int pow2_cols(int c) { return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512; }
__host__ __device__ constexpr int align_up(int x, int a) { return (x + a - 1) / a * a; }

template <int Q, int L, bool U16, bool LEAN>
struct ProjCfgT {
  static constexpr bool kLean = LEAN;
  static constexpr int kNGroups = LEAN ? 1 : 2;                     // converter groups
  static constexpr int kThreads = 96 + kNGroups * 128 + 128;        // MMA1, MMA2, TMA, converters, epilogue
  static constexpr int kMinBlocks = LEAN ? 2 : 1;
  static constexpr int kEpi0 = 96 + kNGroups * 128;                 // first epilogue thread
  static constexpr int kKC = Q >= 64 ? 64 : Q;            // K elements (pixels) per A1 chunk
  static constexpr int kCPT = Q / kKC;                    // chunks per stage-1 tile
  static constexpr int kSpan = kKC * 2;                   // bytes per row of a raw u16 chunk (swizzle span)
  static constexpr int kSwzMask = kSpan == 128 ? 7 : 3;   // TMA SWIZZLE_128B / 64B address XOR mask
  static constexpr int kSlotU = 128 * kSpan;              // u16 slot == TMA box
  static constexpr int kSlotF = (kKC / 8) * (int)kLBO;    // f32 path: no-swizzle fp16 operand
  static constexpr int kSlot = align_up(U16 ? kSlotU : kSlotF, 1024);
  static constexpr int kN = 2 * L;                        // MMA N: Psi_hi | Psi_lo
  static constexpr int kLBO_B = 16 * kN;
  static constexpr int kB = (Q / 8) * kLBO_B;
  static constexpr int kFPT = Q >= 128 ? 1 : 128 / Q;     // frames per stage-1 tile
  static constexpr int kTPF = Q >= 128 ? Q / 128 : 1;     // stage-1 tiles per frame (= stage-2 K chunks)
  static constexpr int kK2 = Q >= 128 ? 128 : Q;          // stage-2 K chunk (detector rows)
  // stage-2 MMA M: 64 rows (frame, a) when a group of whole stage-1 tiles fits, else 128.  The
  // M = 64 accumulator occupies lanes 0-15 of each TMEM lane quadrant (row m -> lane m%16 + 32(m/16)).
  static constexpr int kM2 = (64 / L) >= kFPT ? 64 : 128;
  static constexpr int kG2 = Q >= 128 ? kM2 / L : ((kM2 / L) / kFPT) * kFPT;  // max frames per group
  // A2 is MN-major (no swizzle): core matrix = 8 consecutive m (16 bytes) x 8 k, k-blocks at
  // 128 bytes, m-blocks at kSBO2, so the epilogue stores 8 values of a frame row as one 16-byte word
  static constexpr uint32_t kSBO2 = (kK2 / 8) * 128;
  static constexpr int kA2 = (kM2 / 8) * (int)kSBO2;       // one A2 plane
  // Lean variant with L >= 24: the Psi_hi and Psi_lo products accumulate into the same fp32
  // accumulator (two MMAs with N = L: the sum the epilogue would otherwise form, done by the
  // tensor core), which halves the accumulators' TMEM and the epilogue's loads (Large: 141 -> 123
  // us per 16k frames).  Elsewhere one MMA with N = 2L and the sum in the epilogue measured faster
  // (the extra MMAs cost the full Q = 256 kernel ~10%); M = 128 would also need N >= 16 for L = 8.
  static constexpr bool kSplitAcc = LEAN && L >= 24;
  static constexpr int kNacc = kSplitAcc ? L : kN;        // accumulator columns (both stages)
  static constexpr int kAcc1 = kNacc;                     // per acc1 slot (both count planes accumulate here)
#ifndef WDD_LEAN_NB2
#define WDD_LEAN_NB2 1
#endif
#ifndef WDD_LEAN_NA
#define WDD_LEAN_NA 2
#endif
  static constexpr int kNB2 = LEAN ? WDD_LEAN_NB2 : 2;    // stage-2 A2 images / accumulators in flight
  // TMEM A-operand ring (u16 path): 4 deep in the full variant; lean 2 (WDD_LEAN_NA=4, where 256
  // TMEM columns hold it with a two-deep acc1 ring, measured: Box projection 1.016 -> 0.981 of the
  // copy peak, Large / Medium unchanged)
  static constexpr int kNA = !LEAN ? 4
                           : (WDD_LEAN_NA + kNGroups) * (Q >= 64 ? 32 : Q / 2) + (2 + kNB2) * kNacc <= 256 ? WDD_LEAN_NA : 2;
  // acc1 ring: 4 deep unless TMEM (A ring + plane-1 buffers + acc1 + acc2 images) would exceed 512 columns
  // (lean: 2, or 1 where two would not leave both CTAs of an SM their 256 TMEM columns)
  static constexpr int kNAcc = LEAN ? ((kNA + kNGroups) * (Q >= 64 ? 32 : Q / 2) + (2 + kNB2) * kNacc > 256 ? 1 : 2)
                                    : ((kNA + kNGroups) * (Q >= 64 ? 32 : Q / 2) + (4 + kNB2) * kNacc > 512 ? 2 : 4);
  static constexpr int kACols = kKC / 2;                  // TMEM columns of one A1 chunk (fp16 pairs)
  static constexpr int tA = 0;                            // TMEM column map
  static constexpr int tP1 = tA + kNA * kACols;          // one plane-1 buffer per converter group
  static constexpr int tAcc1 = tP1 + kNGroups * kACols;
  static constexpr int tAcc2 = tAcc1 + kNAcc * kAcc1;
  static constexpr int kTmemCols = pow2_cols(tAcc2 + kNB2 * kNacc);
  static_assert(tAcc2 + kNB2 * kN <= 512, "TMEM");
  // stage-2 C rows go out through a per-warp shared-memory transpose (512-byte coalesced stores
  // instead of 16-byte pieces of 16 rows) where it fits: Q = 128, L = 32 (C is 1/8 of the bytes)
  static constexpr bool kCStage = Q == 128 && L == 32 && kM2 == 64;
  static constexpr int kCStageB = kCStage ? 4 * 16 * L * 4 : 0;
  // with a single A2 image the staging aliases it: the stage-2 epilogue runs between the wait for
  // the stage-2 MMAs (A2 free) and the next group's T writes (after an epilogue-wide barrier)
  static constexpr bool kCAlias = kCStage && kNB2 == 1 && kCStageB <= 2 * kA2;
  // shared memory besides the raw ring: A2 images, B image, C staging, the barriers and meta words
  // of the other rings; each raw slot adds its two barriers and a meta word (kNSraw below)
  static constexpr int kFixed = (U16 ? 0 : 2 * kSlot) + align_up(kNB2 * 2 * kA2, 1024) + align_up(kB, 1024) +
                                (kCAlias ? 0 : kCStageB) + 8 * (2 * kNA + 2 * 2 + 3 * kNB2 + 3) + 4 * kNA + 80;
  // (lean: two CTAs and their per-CTA reservation must share the SM's 228 KB -- 110 KB each leaves
  // room; measured: 112.3 KB CTAs did not co-reside.  Two converter groups need an even ring.)
  static constexpr int kNSraw = (((LEAN ? kLeanSmem : 232448) - kFixed) / (kSlot + 8 * 2 + 4)) & (kNGroups == 2 ? ~1 : ~0);
  static constexpr int kNSfit = kNSraw < 2 ? 2 : kNSraw;   // (lean: configs that do not fit run 1 CTA/SM)
  static constexpr int kNS = kNSfit < WDD_NS ? kNSfit : WDD_NS;  // raw ring (even: group = job parity)
  static constexpr int off_ring = 0;
  static constexpr int off_P1 = off_ring + kNS * kSlot;   // f32 path only
  static constexpr int off_A2 = off_P1 + (U16 ? 0 : 2 * kSlot);
  static constexpr int off_B = off_A2 + align_up(kNB2 * 2 * kA2, 1024);
  static constexpr int off_C = kCAlias ? off_A2 : off_B + align_up(kB, 1024);
  static constexpr int off_bar = off_B + align_up(kB, 1024) + (kCAlias ? 0 : kCStageB);
  static constexpr int kBars = 2 * kNS + 2 * kNA + 2 * kNAcc + 3 * kNB2 + 3;
  static constexpr int off_misc = off_bar + 8 * kBars;    // meta[kNS+kNA], wflag[2 groups][2][4], tmem slot
  static constexpr int smem = off_misc + 4 * (kNS + kNA) + 64 + 16;
  static constexpr int kTmemUsed = tAcc2 + kNB2 * kNacc;
  static_assert((kNGroups == 1 || kNS % 2 == 0) && kNA % 2 == 0, "even rings: converter group = job parity");
  static_assert(kG2 >= 1, "group");
  static_assert(smem <= 232448, "shared memory");
};
// Lean (two CTAs per SM) where both CTAs fit in shared memory and TMEM, else the full variant.
template <int Q, int L, bool U16>
struct ProjCfgSel {
  using LeanCfg = ProjCfgT<Q, L, U16, true>;
  // (Q = 256, L = 32 would fit a three-slot lean CTA, but measured slower than the full variant's
  // eight slots and two converter groups: Live step 0.78 vs 0.81 of its roofline)
  static constexpr bool lean = kLeanAllowed && LeanCfg::smem <= kLeanSmem && LeanCfg::kTmemUsed <= 256 &&
                               LeanCfg::kNSraw >= 3 && !(Q == 256 && L == 32);
  using type = typename std::conditional<lean, LeanCfg, ProjCfgT<Q, L, U16, false>>::type;
};
template <int Q, int L, bool U16>
using ProjCfg = typename ProjCfgSel<Q, L, U16>::type;


__device__ __forceinline__ uint32_t magic_half2(uint32_t v10) {
  // v10 holds two 10-bit integers (bits 0-9 and 16-25).  (0x6400 | x) is fp16 1024 + x,
  // exact; subtracting 1024 leaves x exactly.
  uint32_t bits = v10 | 0x64006400u;
  const __half2 h = *reinterpret_cast<const __half2*>(&bits);
  const __half2 r = __hsub2(h, __half2half2(__ushort_as_half((unsigned short)0x6400)));
  return *reinterpret_cast<const uint32_t*>(&r);
}

// Second count plane of a u16 pair: (x >> 10) * 1024 = x & 0xFC00, exact in fp16.
__device__ __forceinline__ uint32_t hi_plane(uint32_t w) {
  const uint32_t v = magic_half2((w >> 10) & 0x003F003Fu);
  const __half2 h = *reinterpret_cast<const __half2*>(&v);
  const __half2 r = __hmul2(h, __half2half2(__ushort_as_half((unsigned short)0x6400)));
  return *reinterpret_cast<const uint32_t*>(&r);
}

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Kernel attributes are per device (context), so the "already set" cache is keyed by the current
// device as well as the function; thread-safe (plans on several devices in one process).
cudaError_t func_attr_once(const void* fn, cudaFuncAttribute attr, int value) {
  static std::mutex mu;
  static std::set<std::tuple<int, const void*, int, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_tuple(dev, fn, (int)attr, value);
  std::lock_guard<std::mutex> g(mu);
  if (done.count(key)) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, attr, value);
  if (e == cudaSuccess) done.insert(key);
  return e;
}

struct ProjArgs {
  const void* frames;
  int64_t n;
  int64_t pos0;         // scan position of frame f: idx ? idx[f] : pos0 + f
  const int32_t* idx;
  ProjDst dst;          // where coefficient row a of a frame goes: shard o with alo[o] <= a < alo[o+1]
                        // -> C[o] + position * Kd[o] + (a - alo[o]) * L (another rank's store: peer memory)
  int g2;      // frames per stage-2 group (<= kG2; a multiple of kFPT)
  const uint4* Bpack;
  float sc1;   // acc1 -> fp16 A2 scale   (2^(eT - s))
  float sc2;   // acc2 -> C scale          (2^(-s - eT))
  int pdl_wait_end;   // 1: complete only after the preceding grid (keeps stream order for later launches;
                      // CTA 0 waits), 2: every CTA waits
  int pdl_wait_start; // 1: no frame load (and no dependent launch) before the preceding grid has completed --
                      // the frames may come from a caller kernel enqueued right before the ingest
  unsigned* err;      // f32 frames: bit 0 set if a value does not fit the fp16 hi/lo split (|x| > 65504 or
                      // not finite); sticky until wdd_check
};

// Stage-1 tile tt of group g: first frame-matrix row and the number of valid rows.
// Q >= 128: tiles are ordered (half h, frame f) with tt = h*g2 + f, so that the stage-2 K chunk h
// of every frame of the group is complete before the next chunk begins.
template <int Q, int L, bool U16>
__device__ __forceinline__ void tile_coords(int64_t g, int tt, int g2, int64_t n, int64_t& row0, int& valid) {
  using Cfg = ProjCfg<Q, L, U16>;
  const int64_t frame0 = g * g2;
  if constexpr (Q >= 128) row0 = (frame0 + tt % g2) * Q + (int64_t)(tt / g2) * 128;
  else row0 = (frame0 + (int64_t)tt * Cfg::kFPT) * Q;
  const int64_t rem = n * Q - row0;
  valid = rem <= 0 ? 0 : (rem < 128 ? (int)rem : 128);
}

template <int Q, int L, bool U16>
__global__ void __launch_bounds__(ProjCfg<Q, L, U16>::kThreads, ProjCfg<Q, L, U16>::kMinBlocks)
    project_kernel(ProjArgs a, const __grid_constant__ CUtensorMap tmap) {
  using Cfg = ProjCfg<Q, L, U16>;
  constexpr int K = L * L;
  TRACE_DECL
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem + Cfg::off_ring;
  uint8_t* sP1 = smem + Cfg::off_P1;
  uint8_t* sA2 = smem + Cfg::off_A2;
  uint8_t* sB = smem + Cfg::off_B;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::off_bar);
  uint64_t* raw_full = bars;                   // [kNS] slot filled (TMA tx / f32 converter)
  uint64_t* raw_empty = bars + Cfg::kNS;       // [kNS] slot free   (u16 converter / f32 MMA commit)
  uint64_t* a_full = bars + 2 * Cfg::kNS;      // [Cfg::kNA] TMEM A chunk written (u16)
  uint64_t* a_empty = a_full + Cfg::kNA;            // [Cfg::kNA] TMEM A chunk consumed (u16)
  uint64_t* p1_empty = a_empty + Cfg::kNA;          // [2] per converter group
  uint64_t* acc1_full = p1_empty + 2;          // [kNAcc]
  uint64_t* acc1_empty = acc1_full + Cfg::kNAcc;
  uint64_t* a2_full = acc1_empty + Cfg::kNAcc;  // [kNB2] A2 image written
  uint64_t* s2_done = a2_full + Cfg::kNB2;      // [kNB2] stage-2 MMAs reading A2 image done
  uint64_t* acc2_empty = s2_done + Cfg::kNB2;   // [kNB2] stage-2 accumulator read by the epilogue
  uint64_t* b_full = acc2_empty + Cfg::kNB2;    // basis operand image landed (bulk copy)
  uint32_t* meta = reinterpret_cast<uint32_t*>(smem + Cfg::off_misc);   // [kNS + Cfg::kNA]
  uint32_t* wflag = meta + Cfg::kNS + Cfg::kNA;                               // [2][2][4]
  uint32_t* tslot = wflag + 16;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (!a.pdl_wait_start) pdl_trigger();
#ifdef WDD_TRACE
  __shared__ unsigned cta_slot;
  if (tid == 0) {
    cta_slot = atomicAdd(&g_cta_n, 1u);
    CTA_REC(cta_slot, 0);
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    if (cta_slot < 8192) g_cta[cta_slot][4] = sm;
  }
#endif

  // ---- setup: barriers and TMEM only, so the TMA producer can start streaming at once; the basis
  // operand image arrives by one bulk copy that only the MMA issuers wait for
  if (tid == 0) {
    // u16: each of the 4 converter warps releases its 32 rows of a raw slot as soon as it has them
    // in registers (f32: the stage-1 MMA commit releases the slot)
    for (int i = 0; i < Cfg::kNS; ++i) { mbar_init(&raw_full[i], 1); mbar_init(&raw_empty[i], U16 ? 4 : 1); }
    for (int i = 0; i < Cfg::kNA; ++i) { mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1); }
    mbar_init(&p1_empty[0], 1);
    mbar_init(&p1_empty[1], 1);
    for (int i = 0; i < Cfg::kNAcc; ++i) { mbar_init(&acc1_full[i], 1); mbar_init(&acc1_empty[i], 4); }
    for (int i = 0; i < Cfg::kNB2; ++i) { mbar_init(&a2_full[i], 1); mbar_init(&s2_done[i], 1); mbar_init(&acc2_empty[i], 4); }
    mbar_init(b_full, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(b_full, Cfg::kB);
    bulk_load(sB, a.Bpack, Cfg::kB, b_full);
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tslot);
  if (U16 && warp == 2 && lane == 0) prefetch_tmap(&tmap);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  if (a.pdl_wait_start) {   // (setup above overlaps the predecessor; frames are read only below)
    pdl_wait();
    pdl_trigger();
  }

  const int64_t n = a.n;
  const int g2 = a.g2;
  const int tpg = Q >= 128 ? g2 * Cfg::kTPF : g2 / Cfg::kFPT;   // stage-1 tiles per group
  const int tph = Q >= 128 ? g2 : tpg;                           // stage-1 tiles per stage-2 K chunk
  const int64_t n_groups = (n + g2 - 1) / g2;
  const int64_t my_groups = blockIdx.x < n_groups ? (n_groups - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (warp == 0) {
    // ================= stage-1 MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16(128, Cfg::kNacc);
      constexpr uint64_t kLoOff = (uint64_t)((L / 8) * 128) >> 4;   // Psi_lo rows of the B image (descriptor units)
      const uint32_t ring0 = smem_u32(ring), p10 = smem_u32(sP1), b0 = smem_u32(sB);
      mbar_wait(b_full, 0);
      uint32_t slot = 0, sphase = 0, tile = 0, job = 0;
      for (int64_t gi = 0; gi < my_groups; ++gi) {
        for (int tt = 0; tt < tpg; ++tt, ++tile) {
          const uint32_t s1 = tile % Cfg::kNAcc;
          mbar_wait(&acc1_empty[s1], ((tile / Cfg::kNAcc) & 1u) ^ 1u);
          TRACE(6, tile);
          tc_fence_after();
          const uint32_t acc = tbase + Cfg::tAcc1 + s1 * Cfg::kAcc1;
          for (int c = 0; c < Cfg::kCPT; ++c, ++job) {
            const uint32_t grp = Cfg::kNGroups == 2 ? (job & 1u) : 0u;
            mbar_wait(U16 ? &a_full[slot] : &raw_full[slot], sphase);
            TRACE(5, slot);
            tc_fence_after();
            const bool has_p1 = meta[slot] & 1u;
#pragma unroll
            for (int kk = 0; kk < Cfg::kKC / 16; ++kk) {
              const uint64_t bd = smem_desc_noswz(b0 + (c * (Cfg::kKC / 8) + 2 * kk) * Cfg::kLBO_B, Cfg::kLBO_B, 128);
              const uint32_t accum = (c > 0 || kk > 0) ? 1u : 0u;
              if constexpr (U16) mma_f16_ts(acc, tbase + Cfg::tA + slot * Cfg::kACols + kk * 8, bd, idesc, accum);
              else mma_f16_ss(acc, smem_desc_noswz(ring0 + slot * Cfg::kSlot + 2 * kk * kLBO, kLBO, 128), bd, idesc, accum);
              if constexpr (Cfg::kSplitAcc) {
                if constexpr (U16) mma_f16_ts(acc, tbase + Cfg::tA + slot * Cfg::kACols + kk * 8, bd + kLoOff, idesc, 1u);
                else mma_f16_ss(acc, smem_desc_noswz(ring0 + slot * Cfg::kSlot + 2 * kk * kLBO, kLBO, 128), bd + kLoOff,
                                idesc, 1u);
              }
            }
            if (has_p1) {
#pragma unroll
              for (int kk = 0; kk < Cfg::kKC / 16; ++kk) {
                const uint64_t bd = smem_desc_noswz(b0 + (c * (Cfg::kKC / 8) + 2 * kk) * Cfg::kLBO_B, Cfg::kLBO_B, 128);
                if constexpr (U16) mma_f16_ts(acc, tbase + Cfg::tP1 + grp * Cfg::kACols + kk * 8, bd, idesc, 1u);
                else mma_f16_ss(acc, smem_desc_noswz(p10 + grp * Cfg::kSlot + 2 * kk * kLBO, kLBO, 128), bd, idesc, 1u);
                if constexpr (Cfg::kSplitAcc) {
                  if constexpr (U16) mma_f16_ts(acc, tbase + Cfg::tP1 + grp * Cfg::kACols + kk * 8, bd + kLoOff, idesc, 1u);
                  else mma_f16_ss(acc, smem_desc_noswz(p10 + grp * Cfg::kSlot + 2 * kk * kLBO, kLBO, 128), bd + kLoOff,
                                  idesc, 1u);
                }
              }
              mma_commit(&p1_empty[grp]);
            }
            mma_commit(U16 ? &a_empty[slot] : &raw_empty[slot]);
            if (++slot == (U16 ? Cfg::kNA : Cfg::kNS)) { slot = 0; sphase ^= 1u; }
          }
          mma_commit(&acc1_full[s1]);
        }
      }
    }
  } else if (warp == 1) {
    // ================= stage-2 MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16(Cfg::kM2, Cfg::kNacc, 0, /*a_major=MN*/ 1, 0);
      constexpr bool kLoN = Cfg::kM2 == 64 ? L % 8 == 0 : L % 16 == 0;                // N = L a valid MMA shape
      constexpr uint32_t idesc_lo = idesc_f16(Cfg::kM2, L, 0, /*a_major=MN*/ 1, 0);   // Psi_hi columns only
      constexpr uint64_t kLoOff = (uint64_t)((L / 8) * 128) >> 4;
      const uint32_t a20 = smem_u32(sA2), b0 = smem_u32(sB);
      mbar_wait(b_full, 0);
      uint32_t c2 = 0;
      for (int64_t gi = 0; gi < my_groups; ++gi) {
        const uint32_t gb = (uint32_t)(gi % Cfg::kNB2);
        const uint32_t acc2 = tbase + Cfg::tAcc2 + gb * Cfg::kNacc;
        for (int h = 0; h < Cfg::kTPF; ++h, ++c2) {
          const uint32_t ab = c2 % Cfg::kNB2;
          mbar_wait(&a2_full[ab], (c2 / Cfg::kNB2) & 1u);
          if (h == 0 && gi >= Cfg::kNB2) mbar_wait(&acc2_empty[gb], (uint32_t)((gi / Cfg::kNB2) - 1) & 1u);
          TRACE(12, h);
          tc_fence_after();
          const uint32_t a2 = a20 + ab * 2 * Cfg::kA2;
          // (T_hi + T_lo)(Psi_hi + Psi_lo) without the T_lo Psi_lo term (<= 2^-22 of the product,
          // below the fp32 accumulation): the lo plane multiplies Psi_hi only (N = L)
#pragma unroll
          for (int kk = 0; kk < Cfg::kK2 / 16; ++kk) {
            const uint64_t ad = smem_desc_noswz(a2 + kk * 256, 128, Cfg::kSBO2);
            const uint64_t bd = smem_desc_noswz(b0 + (h * (Cfg::kK2 / 8) + 2 * kk) * Cfg::kLBO_B, Cfg::kLBO_B, 128);
            mma_f16_ss(acc2, ad, bd, idesc, (h > 0 || kk > 0) ? 1u : 0u);
            if constexpr (Cfg::kSplitAcc) mma_f16_ss(acc2, ad, bd + kLoOff, idesc, 1u);
          }
#pragma unroll
          for (int kk = 0; kk < Cfg::kK2 / 16; ++kk) {
            const uint64_t ad = smem_desc_noswz(a2 + Cfg::kA2 + kk * 256, 128, Cfg::kSBO2);
            const uint64_t bd = smem_desc_noswz(b0 + (h * (Cfg::kK2 / 8) + 2 * kk) * Cfg::kLBO_B, Cfg::kLBO_B, 128);
            if constexpr (kLoN) mma_f16_ss(acc2, ad, bd, idesc_lo, 1u);
            else {
              mma_f16_ss(acc2, ad, bd, idesc, 1u);
              if constexpr (Cfg::kSplitAcc) mma_f16_ss(acc2, ad, bd + kLoOff, idesc, 1u);
            }
          }
          mma_commit(&s2_done[ab]);
        }
      }
    }
  } else if (warp == 2) {
    // ================= TMA producer (u16 frames)
    if (U16 && lane == 0) {
      const uint64_t pol = policy_evict_first();   // frames are read exactly once
      uint32_t slot = 0, sphase = 0;
#ifdef WDD_TRACE
      __syncwarp(1u);
      CTA_REC(cta_slot, 1);
#endif
      for (int64_t gi = 0; gi < my_groups; ++gi) {
        const int64_t g = blockIdx.x + gi * gridDim.x;
        for (int tt = 0; tt < tpg; ++tt) {
          int64_t row0;
          int valid;
          tile_coords<Q, L, U16>(g, tt, g2, n, row0, valid);
          for (int c = 0; c < Cfg::kCPT; ++c) {
            mbar_wait(&raw_empty[slot], sphase ^ 1u);
            TRACE(2, slot);
            mbar_arrive_expect_tx(&raw_full[slot], Cfg::kSlotU);
            tma_load_2d_hint(ring + slot * Cfg::kSlot, &tmap, c * Cfg::kKC, (int)row0, &raw_full[slot], pol);
            if (++slot == Cfg::kNS) { slot = 0; sphase ^= 1u; }
          }
        }
      }
    }
  } else if (warp < 3 + 4 * Cfg::kNGroups) {
    // ================= converters: group cg handles the jobs (chunks) with job % 2 == cg
    const int cg = (warp - 3) >> 2;
    const int ct = tid - 96 - cg * kConv;
    const int cw = (warp - 3) & 3;
    const int quad = warp & 3;
    const int row = quad * 32 + lane;                     // detector row of the tile == TMEM lane
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    const int bar_id = 1 + 2 * cg;                        // named barriers 1 and 3 (2 = epilogue)
    uint32_t p1_uses = 0, job = 0;
    for (int64_t gi = 0; gi < my_groups; ++gi) {
      const int64_t g = blockIdx.x + gi * gridDim.x;
      for (int tt = 0; tt < tpg; ++tt) {
        int64_t row0;
        int valid;
        tile_coords<Q, L, U16>(g, tt, g2, n, row0, valid);
        for (int c = 0; c < Cfg::kCPT; ++c, ++job) {
          if (Cfg::kNGroups == 2 && (job & 1u) != (uint32_t)cg) continue;
          const uint32_t slot = job % Cfg::kNS, sphase = (job / Cfg::kNS) & 1u;
          const uint32_t aslot = job % Cfg::kNA, aphase = (job / Cfg::kNA) & 1u;
          bool resid = false;
          uint32_t* wf = wflag + cg * 8 + ((job / Cfg::kNGroups) & 1) * 4;
          if constexpr (U16) {
            constexpr int kW = Cfg::kACols;               // 32-bit words of this row in the chunk
            const uint8_t* src = ring + slot * Cfg::kSlot;
            uint32_t w[kW];
            mbar_wait(&raw_full[slot], sphase);
            if (ct == 0) TRACE(3, slot);
#ifdef WDD_TRACE
            if (ct == 0) CTA_REC(cta_slot, 2);
#endif
#pragma unroll
            for (int j = 0; j < kW / 4; ++j) {           // swizzled 16-byte pieces of row `row`
              int off = row * Cfg::kSpan + j * 16;
              off ^= ((off >> 7) & Cfg::kSwzMask) << 4;
              const uint4 v = *reinterpret_cast<const uint4*>(src + off);
              w[4 * j] = v.x; w[4 * j + 1] = v.y; w[4 * j + 2] = v.z; w[4 * j + 3] = v.w;
            }
            uint32_t hi_or = 0;
#pragma unroll
            for (int q = 0; q < kW; ++q) hi_or |= w[q];
            resid = (hi_or & 0xFC00FC00u) != 0u;
            // a warp with no count >= 1024 never re-reads its rows: release them now
            const bool warp_resid = __any_sync(0xffffffffu, resid);
            if (!warp_resid) {
              __syncwarp();
              if (lane == 0) mbar_arrive(&raw_empty[slot]);
            }
#pragma unroll
            for (int q = 0; q < kW; ++q) w[q] = magic_half2(w[q] & 0x03FF03FFu) | 0u;
            mbar_wait(&a_empty[aslot], aphase ^ 1u);
            if (ct == 0) TRACE(13, aslot);
            tc_fence_after();
#pragma unroll
            for (int q = 0; q < kW; q += 16) tmem_st16(tbase + lane_addr + Cfg::tA + aslot * Cfg::kACols + q, w + q);
            tmem_st_wait();
            const uint32_t bal = __ballot_sync(0xffffffffu, resid);
            if (lane == 0) wf[cw] = bal ? 1u : 0u;
            tc_fence_before();
            named_sync(bar_id, kConv);
            const bool any = (wf[0] | wf[1] | wf[2] | wf[3]) != 0u;
            if (any) {  // bits 10-15 of the counts: second plane
              mbar_wait(&p1_empty[cg], (p1_uses & 1u) ^ 1u);
              ++p1_uses;
              tc_fence_after();
#pragma unroll
              for (int j = 0; j < kW / 4; ++j) {
                if (warp_resid) {   // (warps without high bits released their rows: their plane is 0)
                  int off = row * Cfg::kSpan + j * 16;
                  off ^= ((off >> 7) & Cfg::kSwzMask) << 4;
                  const uint4 v = *reinterpret_cast<const uint4*>(src + off);
                  // (bits 10-15) * 1024 is exact in fp16 (<= 64512): accumulates into the same acc
                  w[4 * j] = hi_plane(v.x);
                  w[4 * j + 1] = hi_plane(v.y);
                  w[4 * j + 2] = hi_plane(v.z);
                  w[4 * j + 3] = hi_plane(v.w);
                } else {
                  w[4 * j] = w[4 * j + 1] = w[4 * j + 2] = w[4 * j + 3] = 0u;
                }
              }
#pragma unroll
              for (int q = 0; q < kW; q += 16) tmem_st16(tbase + lane_addr + Cfg::tP1 + cg * Cfg::kACols + q, w + q);
              tmem_st_wait();
              tc_fence_before();
              named_sync(bar_id, kConv);
            }
            if (warp_resid) {                             // second plane done: release the rows
              __syncwarp();
              if (lane == 0) mbar_arrive(&raw_empty[slot]);
            }
            if (ct == 0) {
              meta[aslot] = any ? 1u : 0u;
              mbar_arrive(&a_full[aslot]);
              TRACE(4, aslot);
            }
          } else {
            // f32: LDG -> fp16(x) (+ residual plane) into a no-swizzle K-major smem slot
            constexpr int kPPR = Cfg::kKC / 8;              // 16-B fp16 pieces per row
            constexpr int kPieces = 128 * kPPR / kConv;
            uint8_t* dst = ring + slot * Cfg::kSlot;
            uint4 lo[kPieces];
            mbar_wait(&raw_empty[slot], sphase ^ 1u);
#pragma unroll
            for (int i = 0; i < kPieces; ++i) {
              const int p = ct + kConv * i, r = p / kPPR, j = p % kPPR;
              float4 x0 = make_float4(0.f, 0.f, 0.f, 0.f), x1 = x0;
              if (r < valid) {
                const float4* src = reinterpret_cast<const float4*>(
                    reinterpret_cast<const float*>(a.frames) + (row0 + r) * Q + c * Cfg::kKC + j * 8);
                x0 = __ldg(src);
                x1 = __ldg(src + 1);
              }
              const float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
              uint4 o, l;
              __half* hp = reinterpret_cast<__half*>(&o);
              __half* lp = reinterpret_cast<__half*>(&l);
              bool bad = false;
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                hp[e] = __float2half_rn(x[e]);
                bad |= __hisinf(hp[e]) || __hisnan(hp[e]);
                const float d = x[e] - __half2float(hp[e]);
                resid |= d != 0.f;
                lp[e] = __float2half_rn(d);
              }
              if (bad) atomicOr(a.err, 1u);
              *reinterpret_cast<uint4*>(dst + j * kLBO + (r >> 3) * 128 + (r & 7) * 16) = o;
              lo[i] = l;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, resid);
            if (lane == 0) wf[cw] = bal ? 1u : 0u;
            fence_proxy_async_smem();
            named_sync(bar_id, kConv);
            const bool any = (wf[0] | wf[1] | wf[2] | wf[3]) != 0u;
            if (any) {
              mbar_wait(&p1_empty[cg], (p1_uses & 1u) ^ 1u);
              ++p1_uses;
#pragma unroll
              for (int i = 0; i < kPieces; ++i) {
                const int p = ct + kConv * i, r = p / kPPR, j = p % kPPR;
                *reinterpret_cast<uint4*>(sP1 + cg * Cfg::kSlot + j * kLBO + (r >> 3) * 128 + (r & 7) * 16) = lo[i];
              }
              fence_proxy_async_smem();
              named_sync(bar_id, kConv);
            }
            if (ct == 0) { meta[slot] = any ? 1u : 0u; mbar_arrive(&raw_full[slot]); }
          }
        }
      }
    }
  } else {
    // ================= epilogue (128 threads; TMEM lane quadrant = warp % 4)
    const int et = tid - Cfg::kEpi0;
    const int quad = warp & 3;
    const int row = quad * 32 + lane;                    // TMEM lane == tile row == A2 m index
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    uint32_t tile = 0, c2 = 0;
    // groups whose stage-2 result has not been stored yet (at most kNB2 + 1): (frame0, gi, last chunk)
    int64_t pend_f0[Cfg::kNB2 + 1] = {};
    int64_t pend_gi[Cfg::kNB2 + 1] = {};
    uint32_t pend_c[Cfg::kNB2 + 1] = {};
    int npend = 0;
    // accumulator row held by this thread's lane (M = 64: lanes 0-15 of each quadrant)
    const int m2 = Cfg::kM2 == 128 ? row : (lane < 16 ? quad * 16 + lane : 1 << 20);
    // destination of this thread's coefficient row a = m2 % L (fixed for the kernel): the shard
    // that owns it -- this rank's store or a peer's, written directly over NVLink
    int c_own = 0;
    while (c_own + 1 < a.dst.n && (m2 % L) >= a.dst.alo[c_own + 1]) ++c_own;
    float* const c_base = a.dst.C[c_own];
    const int64_t c_stride = a.dst.K[c_own];
    const int c_off = ((m2 % L) - a.dst.alo[c_own]) * L;
    auto stage2_epilogue = [&](int64_t frame0, int64_t gi) {
      const uint32_t gb = (uint32_t)(gi % Cfg::kNB2);
      float d[Cfg::kNacc];
      tmem_ld_cols<Cfg::kNacc>(tbase + Cfg::tAcc2 + gb * Cfg::kNacc + lane_addr, d);
      // value of accumulator column b (the hi + lo sum: formed by the MMAs, or here for L = 8)
      // C values b .. b + 3 (the accumulator sum times sc2), packed arithmetic, same rounding as dv(b) * sc2
      const float2 sc2 = make_float2(a.sc2, a.sc2);
      auto dq = [&](int b) {
        float2 u = make_float2(d[b], d[b + 1]), w = make_float2(d[b + 2], d[b + 3]);
        if constexpr (!Cfg::kSplitAcc) {
          u = __fadd2_rn(u, make_float2(d[(L + b) % Cfg::kNacc], d[(L + b + 1) % Cfg::kNacc]));
          w = __fadd2_rn(w, make_float2(d[(L + b + 2) % Cfg::kNacc], d[(L + b + 3) % Cfg::kNacc]));
        }
        u = __fmul2_rn(u, sc2);
        w = __fmul2_rn(w, sc2);
        return make_float4(u.x, u.y, w.x, w.y);
      };
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc2_empty[gb]);
      const int f = m2 / L;
      const int64_t fg = frame0 + f;
      if constexpr (Cfg::kCStage) if (a.dst.n == 1) {
        // lanes 0-15 of this warp hold rows aa0 .. aa0 + 15 of one frame (a contiguous 16 L floats
        // of C): rows into the warp's staging (16-byte chunks XOR-swizzled by row), then the warp
        // stores them as 512-byte contiguous pieces
        float* stg = reinterpret_cast<float*>(smem + Cfg::off_C) + quad * 16 * L;
        if (lane < 16) {
#pragma unroll
          for (int b = 0; b < L; b += 4)
            *reinterpret_cast<float4*>(stg + lane * L + (((b >> 2) ^ (lane & 7)) << 2)) =
                dq(b);
        }
        __syncwarp();
        const int fw = (quad * 16) / L;                      // the warp's frame (warp-uniform)
        const int64_t fgw = frame0 + fw;
        if (fw < g2 && fgw < n) {
          float* dst = a.dst.C[0] + (a.idx ? (int64_t)__ldg(a.idx + fgw) : a.pos0 + fgw) * K + ((quad * 16) % L) * L;
#pragma unroll
          for (int i = 0; i < (16 * L) / 128; ++i) {
            const int e = i * 128 + lane * 4;                // float index in the warp's 16 rows
            const int r = e / L, cq = (e % L) >> 2;
            *reinterpret_cast<float4*>(dst + e) = *reinterpret_cast<const float4*>(stg + r * L + ((cq ^ (r & 7)) << 2));
          }
        }
        __syncwarp();
        return;
      }
      if (f < g2 && fg < n) {
        float* dst = c_base + (a.idx ? (int64_t)__ldg(a.idx + fg) : a.pos0 + fg) * c_stride + c_off;
#pragma unroll
        for (int b = 0; b < L; b += 4) {
          const float4 v = dq(b);
          *reinterpret_cast<float4*>(dst + b) = v;
        }
      }
    };
    // store every pending group whose last stage-2 chunk is <= cdone (all those MMAs have completed)
    auto flush_pending = [&](uint32_t cdone) {
      while (npend > 0 && pend_c[0] <= cdone) {
        stage2_epilogue(pend_f0[0], pend_gi[0]);
        for (int i = 1; i < npend; ++i) { pend_f0[i - 1] = pend_f0[i]; pend_gi[i - 1] = pend_gi[i]; pend_c[i - 1] = pend_c[i]; }
        --npend;
      }
    };
    for (int64_t gi = 0; gi < my_groups; ++gi) {
      const int64_t g = blockIdx.x + gi * gridDim.x;
      for (int tt = 0; tt < tpg; ++tt, ++tile) {
        const uint32_t s1 = tile % Cfg::kNAcc;
        mbar_wait(&acc1_full[s1], (tile / Cfg::kNAcc) & 1u);
        if (et == 0) TRACE(8, tile);
        tc_fence_after();
        float acc[Cfg::kNacc];
        float2 t[L / 2];                                 // T values of this row, packed pairs
        tmem_ld_cols<Cfg::kNacc>(tbase + Cfg::tAcc1 + s1 * Cfg::kAcc1 + lane_addr, acc);
        {
          const float2 sc = make_float2(a.sc1, a.sc1);
#pragma unroll
          for (int q = 0; q < L; q += 2) {
            float2 v = make_float2(acc[q], acc[q + 1]);
            if constexpr (!Cfg::kSplitAcc) v = __fadd2_rn(v, make_float2(acc[(L + q) % Cfg::kNacc], acc[(L + q + 1) % Cfg::kNacc]));
            t[q / 2] = __fmul2_rn(v, sc);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc1_empty[s1]);
        const uint32_t ab = c2 % Cfg::kNB2;
        if (tt % tph == 0 && c2 >= (uint32_t)Cfg::kNB2) {   // A2 image ab is free once chunk c2 - kNB2 is done
          mbar_wait(&s2_done[ab], ((c2 / Cfg::kNB2) - 1) & 1u);
          if (et == 0) TRACE(14, tile);
          tc_fence_after();
          flush_pending(c2 - Cfg::kNB2);
          if (et == 0) TRACE(15, tile);
          if constexpr (Cfg::kCAlias) named_sync(2, 128);   // every warp's C staging (in A2) read out
        }
        // A2 element (m = f*L + a, k), MN-major: (m/8)*kSBO2 + (k/8)*128 + (k%8)*16 + (m%8)*2
        int f, k;
        if constexpr (Q >= 128) { f = tt % g2; k = row; }
        else { f = tt * Cfg::kFPT + row / Q; k = row % Q; }
        {
          uint8_t* base = sA2 + ab * 2 * Cfg::kA2 + (k >> 3) * 128 + (k & 7) * 16 + ((f * L) >> 3) * Cfg::kSBO2;
#pragma unroll
          for (int q0 = 0; q0 < L; q0 += 8) {
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              // packed conversions (one F2FP per pair; the same RN values as per-element converts)
              const float2 av = t[q0 / 2 + e];
              const __half2 h = __floats2half2_rn(av.x, av.y);
              const float2 hf = __half22float2(h);
              const float2 dv2 = __fadd2_rn(av, make_float2(-hf.x, -hf.y));
              const __half2 l = __floats2half2_rn(dv2.x, dv2.y);
              hw[e] = *reinterpret_cast<const uint32_t*>(&h);
              lw[e] = *reinterpret_cast<const uint32_t*>(&l);
            }
            uint8_t* p = base + (q0 >> 3) * Cfg::kSBO2;
            *reinterpret_cast<uint4*>(p) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(p + Cfg::kA2) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
          }
        }
        if (et == 0) TRACE(10, tile);
        if (tt % tph == tph - 1) {   // stage-2 K chunk complete
          fence_proxy_async_smem();
          named_sync(2, 128);
          if (et == 0) { mbar_arrive(&a2_full[ab]); TRACE(11, tile); }
          ++c2;
        }
      }
      pend_f0[npend] = g * g2;
      pend_gi[npend] = gi;
      pend_c[npend] = c2 - 1;
      ++npend;
    }
    // drain: wait for the last chunk of each pending group in order
    while (npend > 0) {
      const uint32_t cl = pend_c[0];
      mbar_wait(&s2_done[cl % Cfg::kNB2], (cl / Cfg::kNB2) & 1u);
      tc_fence_after();
      flush_pending(cl);
    }
    // coefficients stored into peers' stores are performed system-wide before this grid completes
    // (the readout's barrier collective then orders them before the owner's row transform)
    if (a.dst.n > 1) __threadfence_system();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<Cfg::kTmemCols>(tbase);
  // This grid completes only after the preceding grid has completed (so an ordinary launch after
  // it also follows every earlier kernel): one CTA waiting is enough -- the grid is complete only
  // once that CTA exits -- and the others free their SM slots for the next grid of the chain
  // instead of idling until the predecessor's last CTA is done (WDD_PROJ_WAIT_ALL=1: every CTA).
  if (a.pdl_wait_end && (blockIdx.x == 0 || a.pdl_wait_end > 1)) pdl_wait();
#ifdef WDD_TRACE
  if (tid == 0) CTA_REC(cta_slot, 3);
#endif
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link needed)
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D fp32 tensor map (no swizzle) of a row-major [rows][inner] array with the given row pitch,
// for the shared-memory FFTs' tile loads; false if it cannot be encoded (callers then load with
// plain vector loads).  WDD_FFT_TMA=0 disables it.
static bool fft_tmap(CUtensorMap* tm, const void* base, uint64_t inner, uint64_t rows, uint64_t pitch_bytes,
                     uint32_t bx, uint32_t by) {
  static const bool off = [] { const char* e = std::getenv("WDD_FFT_TMA"); return e && std::atoi(e) == 0; }();
  std::memset(tm, 0, sizeof(*tm));
  auto enc = get_encode();
  if (off || !enc || bx * 4 % 16 || bx > 256 || by > 256 || pitch_bytes % 16 || (uintptr_t)base % 16) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)pitch_bytes};
  const cuuint32_t box[2] = {bx, by};
  const cuuint32_t estr[2] = {1u, 1u};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int Q, int L, bool U16>
static cudaError_t launch_project_t(const Plan& p, const void* frames, int64_t n, const ProjDst& dst,
                                    const int32_t* idx, int64_t pos0, cudaStream_t st, bool wait_start) {
  using Cfg = ProjCfg<Q, L, U16>;
  auto kern = project_kernel<Q, L, U16>;
  {
    cudaError_t e = func_attr_once((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::smem);
    if (e == cudaSuccess) e = func_attr_once((const void*)kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
  }
  if (n <= 0) return cudaSuccess;
  // frames per stage-2 group: the largest multiple of kFPT (<= kG2) that keeps the per-CTA
  // frame count minimal, so small batches still spread over every SM
  int g2 = Cfg::kFPT;
  int64_t best = INT64_MAX;
  for (int c = Cfg::kFPT; c <= Cfg::kG2; c += Cfg::kFPT) {
    const int64_t groups = (n + c - 1) / c;
    const int64_t per_cta = (groups + p.sm_count - 1) / p.sm_count * c;
    if (per_cta <= best) { best = per_cta; g2 = c; }
  }
  // Frames per CTA: about 2 MiB (lean: 512 KiB) of frame data per CTA, so that a small batch occupies only part
  // of the GPU and consecutive (PDL-chained) batches stream concurrently on the other SMs instead
  // of each batch paying its own pipeline fill and drain on every SM.  WDD_PROJ_MIN_FRAMES
  // overrides (0 = spread every batch over all SMs).
  static const int env_frames = [] { const char* e = std::getenv("WDD_PROJ_MIN_FRAMES"); return e ? std::atoi(e) : -1; }();
  int min_frames = env_frames >= 0 ? env_frames
                                   : std::max(4, (Cfg::kLean ? (1 << 19) : (1 << 21)) / (Q * Q * (U16 ? 2 : 4)));
  // (full variant: 2 MiB measured best since only CTA 0 of a grid waits for the preceding grid at
  // its end -- Live 1 / 2 / 4 MiB: 23.8 / 24.8 / 24.7 M frames/s, projection 0.96 / 1.03 / 1.05 of the
  // copy peak; the chained per-batch time p50 34 -> 55 us, a lone batch 48 -> 70 us -- the latency
  // grid, opts.ingest_spread, keeps 51 us)
  // the first batch after a reset finds the GPU idle: spread it over every CTA slot so the chained
  // launches of the following batches find a full machine instead of ramping up one grid at a time
  static const int wide_first = [] { const char* e = std::getenv("WDD_PROJ_WIDE_FIRST"); return e ? std::atoi(e) : 1; }();
  if (wide_first && p.frames_ingested == 0 && env_frames < 0) min_frames = 1;
  // The launches that end a scan (the frames of this one and of the calls still to come fit the
  // GPU's CTA slots at fewer than min_frames each) spread thinner: with min_frames frames per CTA
  // the chain's last grids ran alone for a whole CTA lifetime (Medium: the last ~25 us of a
  // 117 us acquisition at a third of the slots, tools/trace_ctas.py)
  static const int tail_spread = [] { const char* e = std::getenv("WDD_PROJ_TAIL"); return e ? std::atoi(e) : 1; }();
  if (tail_spread && p.proj_rem_after >= 0 && env_frames < 0 && min_frames > 1) {
    const int64_t slots = (int64_t)p.sm_count * Cfg::kMinBlocks;
    const int64_t per = (n + p.proj_rem_after + slots - 1) / slots;
    if (per < min_frames) min_frames = (int)std::max<int64_t>(1, per);
  }
  if (p.ingest_spread) min_frames = 1;                 // latency grid (opts.ingest_spread)
  if (min_frames > 0) g2 = Cfg::kG2;
  const int64_t groups = (n + g2 - 1) / g2;
  int grid = (int)std::min<int64_t>(groups, (int64_t)p.sm_count * Cfg::kMinBlocks);
  if (min_frames > 0) grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid, (n + min_frames - 1) / min_frames));
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof tmap);
  if constexpr (U16) {
    auto enc = get_encode();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {(cuuint64_t)Q, (cuuint64_t)(n * Q)};
    const cuuint64_t strides[1] = {(cuuint64_t)Q * 2};
    const cuuint32_t box[2] = {(cuuint32_t)Cfg::kKC, 128u};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(frames), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           Cfg::kSpan == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  static const int no_wait = [] { const char* e = std::getenv("WDD_PROJ_NO_PDLWAIT"); return e ? std::atoi(e) : 0; }();
  static const int wait_all = [] { const char* e = std::getenv("WDD_PROJ_WAIT_ALL"); return e ? std::atoi(e) : 0; }();
  ProjArgs a{frames, n, pos0, idx, dst, g2, reinterpret_cast<const uint4*>(p.d_Bpack), (float)p.sc1, (float)p.sc2,
             no_wait ? 0 : wait_all ? 2 : 1, wait_start ? 1 : 0, p.d_err};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  // The first launch after a reset is an ordinary launch (it starts only once everything before it
  // has completed: the previous acquisition's flush and readout may still read the coefficient
  // store it overwrites) unless the reset swapped in the other store (c_fresh): then it too
  // overlaps its predecessor, the previous readout, programmatically.  Later launches of the
  // acquisition write disjoint scan positions and always overlap their predecessors.
  cfg.numAttrs = (p.frames_ingested == 0 && !p.c_fresh) ? 0 : 1;
  p.last_proj_grid = grid;
  return cudaLaunchKernelEx(&cfg, kern, a, tmap);
}

#define WDD_PROJ_CASE(QQ, LL)                                                          \
  if (p.Q == QQ && p.L == LL)                                                          \
    return p.dtype == 0 ? launch_project_t<QQ, LL, true>(p, frames, n, dst, idx, pos0, st, wait_start)     \
                        : launch_project_t<QQ, LL, false>(p, frames, n, dst, idx, pos0, st, wait_start);

cudaError_t launch_project(const Plan& p, const void* frames, int64_t n, const ProjDst& dst, const int32_t* idx,
                           int64_t pos0, cudaStream_t st, bool wait_start) {
  WDD_PROJ_CASE(32, 8) WDD_PROJ_CASE(32, 16) WDD_PROJ_CASE(32, 24) WDD_PROJ_CASE(32, 32)
  WDD_PROJ_CASE(64, 8) WDD_PROJ_CASE(64, 16) WDD_PROJ_CASE(64, 24) WDD_PROJ_CASE(64, 32)
  WDD_PROJ_CASE(128, 8) WDD_PROJ_CASE(128, 16) WDD_PROJ_CASE(128, 24) WDD_PROJ_CASE(128, 32)
  WDD_PROJ_CASE(256, 8) WDD_PROJ_CASE(256, 16) WDD_PROJ_CASE(256, 24) WDD_PROJ_CASE(256, 32)
  return cudaErrorInvalidValue;
}

#ifdef WDD_TRACE
extern "C" int wdd_trace_dump(unsigned long long* host, int max_n) {
  cudaDeviceSynchronize();
  const int n = max_n < 16 * 4096 ? max_n : 16 * 4096;
  cudaMemcpyFromSymbol(host, g_trace, n * sizeof(unsigned long long));
  static unsigned long long zeros[16 * 4096];
  cudaMemcpyToSymbol(g_trace, zeros, sizeof zeros);
  return n;
}

extern "C" int wdd_trace_ctas(unsigned long long* host /* 8192 x 5 */) {
  cudaDeviceSynchronize();
  unsigned n = 0;
  cudaMemcpyFromSymbol(&n, g_cta_n, sizeof n);
  cudaMemcpyFromSymbol(host, g_cta, sizeof(unsigned long long) * 8192 * 5);
  const unsigned z = 0;
  cudaMemcpyToSymbol(g_cta_n, &z, sizeof z);
  return (int)(n < 8192 ? n : 8192);
}
#endif

bool project_is_lean(const Plan& p) {
#define WDD_LEAN_CASE(QQ, LL) \
  if (p.Q == QQ && p.L == LL) return p.dtype == 0 ? ProjCfg<QQ, LL, true>::kLean : ProjCfg<QQ, LL, false>::kLean;
  WDD_LEAN_CASE(32, 8) WDD_LEAN_CASE(32, 16) WDD_LEAN_CASE(32, 24) WDD_LEAN_CASE(32, 32)
  WDD_LEAN_CASE(64, 8) WDD_LEAN_CASE(64, 16) WDD_LEAN_CASE(64, 24) WDD_LEAN_CASE(64, 32)
  WDD_LEAN_CASE(128, 8) WDD_LEAN_CASE(128, 16) WDD_LEAN_CASE(128, 24) WDD_LEAN_CASE(128, 32)
  WDD_LEAN_CASE(256, 8) WDD_LEAN_CASE(256, 16) WDD_LEAN_CASE(256, 24) WDD_LEAN_CASE(256, 32)
#undef WDD_LEAN_CASE
  return false;
}

// resident projection CTAs per SM as the runtime computes it (registers, smem, threads)
int project_occupancy(const Plan& p) {
  int n = 0;
#define WDD_OCC_CASE(QQ, LL)                                                                         \
  if (p.Q == QQ && p.L == LL) {                                                                      \
    if (p.dtype == 0) {                                                                              \
      using C = ProjCfg<QQ, LL, true>;                                                               \
      func_attr_once((const void*)project_kernel<QQ, LL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::smem); \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, project_kernel<QQ, LL, true>, C::kThreads, C::smem); \
    } else {                                                                                         \
      using C = ProjCfg<QQ, LL, false>;                                                              \
      func_attr_once((const void*)project_kernel<QQ, LL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::smem); \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, project_kernel<QQ, LL, false>, C::kThreads, C::smem); \
    }                                                                                                \
  }
  WDD_OCC_CASE(32, 8) WDD_OCC_CASE(32, 16) WDD_OCC_CASE(32, 24) WDD_OCC_CASE(32, 32)
  WDD_OCC_CASE(64, 8) WDD_OCC_CASE(64, 16) WDD_OCC_CASE(64, 24) WDD_OCC_CASE(64, 32)
  WDD_OCC_CASE(128, 8) WDD_OCC_CASE(128, 16) WDD_OCC_CASE(128, 24) WDD_OCC_CASE(128, 32)
  WDD_OCC_CASE(256, 8) WDD_OCC_CASE(256, 16) WDD_OCC_CASE(256, 24) WDD_OCC_CASE(256, 32)
#undef WDD_OCC_CASE
  return n;
}

size_t project_smem_bytes(int Q, int L) {
#define WDD_SMEM_CASE(QQ, LL) if (Q == QQ && L == LL) return ProjCfg<QQ, LL, true>::smem;
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
// Accumulation (a4 + a5): G[v][k] += F_y (x) F_x applied to the pending coefficients C (P:411-414,
// eq:outer_prod P:424), in the separable form of the north star: a 1-D DFT along each scan row
// (a4) into the staging R[j][sy][k] (active vx columns j only), then the phase-weighted update
// along y (a5) into G for the active (vx, vy).  Both transforms are unitary (1/sqrt(S_axis)).
//
// Power-of-two scan axes use radix-2 FFTs in shared memory (O(S log S) per coefficient instead
// of the O(S * n_active) of the DFT-matrix form; both passes are then HBM-bound); other sizes,
// and flushes of only a few rows along y, use the DFT-matrix kernels further below.  Positions
// not pending (not ingested, or already folded into G) enter as exact zeros: the host passes a
// per-row bitmask of pending positions, so the coefficient store never needs to be cleared.
// =====================================================================================
using fft::cmul;
constexpr int kU = 8;   // loads in flight per thread in the FFT kernels' staging loops
constexpr int kFftMaxLog = 10;   // FFT path for scan axes up to 1024 (DFT-matrix kernels beyond)

__device__ __forceinline__ uint32_t bf16x2_bits(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
// x = hi + lo with hi = bf16(x), lo = bf16(x - hi), packed for two values
__device__ __forceinline__ void split_bf16x2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  const float2 hf = __bfloat1622float2(h);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = bf16x2_bits(a - hf.x, b - hf.y);
}


// a4 by FFT.  CTA = (k-tile of 2P coefficients, one pending scan row).  Two real coefficient
// sequences k, k+1 share one complex FFT (z = C_k + i C_{k+1}); X_k[v] = (Z[v] + conj Z[-v]) / 2,
// X_{k+1}[v] = (Z[v] - conj Z[-v]) / 2i.  Non-pending positions enter as zeros.
#ifndef WDD_RF_MINB_SMALL
#define WDD_RF_MINB_SMALL 3
#endif
#ifndef WDD_RF_MINB_LARGE
#define WDD_RF_MINB_LARGE 2
#endif
#ifndef WDD_CF_MINB_SMALL
#define WDD_CF_MINB_SMALL 3
#endif
#ifndef WDD_CF_MINB_LARGE
#define WDD_CF_MINB_LARGE 2
#endif
// LOGC >= 0: logP fixed at compile time (= the argument); -1: any logP.  FftPad: float2 of padding
// per block of N2 positions (fft::pidx).  0: a pad that shifts the 8-sequence tiles' blocks by half
// a bank row (64 B) would remove the FFT's second-step bank conflicts, but the TMA tile loads need
// 128-byte aligned shared-memory destinations (measured: misaligned-address fault).
template <int LOGC> struct FftPad { static constexpr int value = 0; };
// Twiddles of the FFT flush kernels read through the L1 from the plan's global table (no per-CTA
// shared copy: its load latency sat at the head of every CTA), by scan-length threshold; and the
// y-FFT output stage's row slots computed from act_vy loaded with the W rows instead of from a
// shared table built in the prologue.
#ifndef WDD_RF_TWG_MINLOG
#define WDD_RF_TWG_MINLOG 99
#endif
#ifndef WDD_CF_TWG_MINLOG
#define WDD_CF_TWG_MINLOG 9
#endif
#ifndef WDD_CF_LAZY_MINLOG
#define WDD_CF_LAZY_MINLOG 9
#endif
#ifndef WDD_CF_U_NOG
#define WDD_CF_U_NOG 8   // y-FFT output rows per thread per round without a G read
#endif
#ifndef WDD_CF_U_NOG_KT8
#define WDD_CF_U_NOG_KT8 16   // the same for 8-coefficient tiles (Sy = 1024: Box)
#endif
// y-FFT readout reduction over the hKT lanes of a row: transposed butterfly (every shuffle carries a
// useful value) for compile-time tiles from 2^WDD_CF_BF_MINLOGC coefficients and at runtime widths,
// a plain xor tree per row below (both bit-identical).  Measured (tools/experiments/exp_cfred*.sh):
// Large y-FFT 136 -> 121 us; Box 1.48 ms (xor tree, 8 rows per round) -> 1.53 (xor tree, 16 rows)
// / 1.56 (butterfly, 8 rows) / 1.46 ms (butterfly, 16 rows)
#ifndef WDD_CF_BF_MINLOGC
#define WDD_CF_BF_MINLOGC 3
#endif
template <int LOGN, int LOGC>
__global__ void __launch_bounds__(256, LOGN <= 8 ? WDD_RF_MINB_SMALL : WDD_RF_MINB_LARGE) rowfft_kernel(const float* __restrict__ C, const int32_t* __restrict__ rows,
                                                     const uint32_t* __restrict__ masks, int mask_words,
                                                     const float2* __restrict__ tw, const int32_t* __restrict__ col_vx,
                                                     float2* __restrict__ R, int logP_rt, int Sy, int K, int n_vx,
                                                     float scale, const __grid_constant__ CUtensorMap tmC, int use_tma,
                                                     int kbase, int KR) {
  // coefficients kbase + blockIdx.x * 2P ..; R holds the chunk kbase .. kbase + KR - 1 (row stride KR)
  constexpr int Sx = 1 << LOGN;
  constexpr int PAD = FftPad<LOGC>::value;
  constexpr int kBY = PAD ? fft::Split<LOGN>::N2 : Sx < 256 ? Sx : 256;   // rows per TMA box (one block when padded)
  extern __shared__ __align__(16) float2 fsm[];
  __shared__ uint32_t smask[(Sx + 31) / 32];
  __shared__ int2 sslot[Sx];             // tile offsets of the slots of v and -v per active column j
  __shared__ __align__(8) uint64_t lbar;
  const int logP = LOGC >= 0 ? LOGC : logP_rt;
  const int P = 1 << logP;
  auto xi = [&](int n) { return fft::pidx<LOGN, PAD>(n, logP); };   // position n of the [Sx][P] tile
  constexpr bool TWG = LOGN >= WDD_RF_TWG_MINLOG;
  float2* x = fsm;                       // [Sx][P] (+ PAD per block of N2 positions)
  float2* stw = fsm + xi(Sx);            // [Sx] twiddles (!TWG)
  const int r = blockIdx.y, k0 = kbase + blockIdx.x * 2 * P;
  // use_tma bit 1 (set when this grid is itself PDL-launched): no early trigger -- this kernel reads
  // the coefficient store, which the first projection of the acquisition after next overwrites, so
  // the dependents of this grid launch only once every CTA has its C tile in shared memory (below).
  // An ordinary (non-PDL) launch of this kernel starts after all earlier work has completed, which
  // already orders it after every earlier read of C; its dependents may then launch at once.
  if (!(use_tma & 2)) pdl_trigger();
  if (use_tma & 1) {
    // the CTA's whole Sx x 2P slice of C in flight at once (one or two TMA boxes, pitch 2P floats =
    // the FFT's [Sx][P] layout), issued before the twiddle / slot tables load so their latency
    // overlaps the tile's; positions outside the pending mask are zeroed afterwards
    if (threadIdx.x == 0) {
      mbar_init(&lbar, 1);
      fence_mbar_init();
      pdl_wait();   // C of the projection kernels (and the uploaded row list / masks)
      const int sy0 = rows[r];
      mbar_arrive_expect_tx(&lbar, (uint32_t)(Sx * P * 8));
      for (int b = 0; b < Sx / kBY; ++b) tma_load_2d(x + xi(b * kBY), &tmC, k0, sy0 * Sx + b * kBY, &lbar);
    }
  }
  if constexpr (!TWG)
    for (int i = threadIdx.x; i < Sx; i += blockDim.x) stw[i] = __ldg(tw + i);
  if (col_vx)   // (NULL: column j is vx = j, the half plane's primary columns; slots computed below)
    for (int j = threadIdx.x; j < n_vx; j += blockDim.x) {
      const int v = __ldg(col_vx + j);
      sslot[j] = make_int2(xi(fft::fslot<LOGN>(v)), xi(fft::fslot<LOGN>((Sx - v) & (Sx - 1))));
    }
  pdl_wait();   // C of the projection kernels (and the uploaded row list / masks)
  const int sy = rows[r];
  if (use_tma & 1) {
    // (use_tma bit 2: every position of the row is pending -- no mask to apply)
    if (!(use_tma & 4) && threadIdx.x < mask_words) smask[threadIdx.x] = masks[(int64_t)r * mask_words + threadIdx.x];
    __syncthreads();
    mbar_wait(&lbar, 0);
    if (!(use_tma & 4)) {
      for (int sx = threadIdx.x; sx < Sx; sx += blockDim.x)
        if (!((smask[sx >> 5] >> (sx & 31)) & 1u))
          for (int pp = 0; pp < P; ++pp) x[xi(sx) + pp] = make_float2(0.f, 0.f);
      __syncthreads();
    }
    if (use_tma & 2) pdl_trigger();   // every read of C by this CTA is complete (the TMA tile has landed)
  } else {
  if (threadIdx.x < mask_words) smask[threadIdx.x] = masks[(int64_t)r * mask_words + threadIdx.x];
  __syncthreads();
  // two coefficient pairs (16 bytes) per load; requires P >= 2
  const float4* Crow = reinterpret_cast<const float4*>(C + (int64_t)sy * Sx * K + k0);
  const int lq = logP - 1, total = Sx << lq;            // 16-byte pieces
  // loads in flight per thread: fewer for the short rows (register budget of 3 CTAs per SM;
  // measured: Large row FFT 306 -> 251 us with 4 at 4 CTAs / SM; no change at Sx = 512)
#ifndef WDD_KU_ROW_SMALL
#define WDD_KU_ROW_SMALL 4
#endif
  constexpr int kURow = LOGN <= 8 ? WDD_KU_ROW_SMALL : 8;
  for (int base = 0; base < total; base += kURow * (int)blockDim.x) {
    float4 v[kURow];
#pragma unroll
    for (int u = 0; u < kURow; ++u) {
      const int e = base + u * (int)blockDim.x + threadIdx.x;
      v[u] = e < total ? __ldg(Crow + (int64_t)(e >> lq) * (K >> 2) + (e & ((P >> 1) - 1)))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kURow; ++u) {
      const int e = base + u * (int)blockDim.x + threadIdx.x;
      if (e < total) {
        const int sx = e >> lq;
        *reinterpret_cast<float4*>(x + xi(sx) + 2 * (e & ((P >> 1) - 1))) =
            ((smask[sx >> 5] >> (sx & 31)) & 1u) ? v[u] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  __syncthreads();
  if (use_tma & 2) pdl_trigger();   // every read of C by this CTA is complete
  }
  fft::fft_seq<LOGN, LOGC, PAD, TWG>(x, TWG ? tw : stw, logP);
  const float hs = 0.5f * scale;
  for (int e = threadIdx.x; e < (n_vx << logP); e += blockDim.x) {
    const int j = e >> logP, pp = e & (P - 1);
    const int2 sl = col_vx ? sslot[j] : make_int2(xi(fft::fslot<LOGN>(j)), xi(fft::fslot<LOGN>((Sx - j) & (Sx - 1))));
    const float2 z = x[sl.x + pp], zm = x[sl.y + pp];
    // ((z.x + zm.x) hs, (z.y - zm.y) hs, (z.y + zm.y) hs, (zm.x - z.x) hs) on packed pairs
    const float2 hs2 = make_float2(hs, hs);
    const float2 o01 = __fmul2_rn(__fadd2_rn(z, make_float2(zm.x, -zm.y)), hs2);
    const float2 o23 = __fmul2_rn(__fadd2_rn(make_float2(z.y, -z.x), make_float2(zm.y, zm.x)), hs2);
    const float4 o = make_float4(o01.x, o01.y, o23.x, o23.y);
    *reinterpret_cast<float4*>(R + ((int64_t)j * Sy + sy) * KR + (k0 - kbase) + 2 * pp) = o;
  }
}

// a5 by FFT, fused with the first half of a6.  CTA = (k-tile t of KT coefficients, one active vx
// column j): the length-Sy FFT of the staged rows of R[j][.][k] (rows not staged are zeros), then
// G[(j, vy)][k] (+)= X[vy] for the active vy of column j (overwrite: the first flush after a
// reset, G is logically zero), and, with the updated G still in registers, the tile's share of the
// Wiener readout  opart[t][g] = sum_{k in tile t} G[g][k] K_g[k], so a readout never
// re-reads G.  The partial sums are combined over tiles in a fixed order by the image transform.
template <int LOGN, int LOGC>
__global__ void __launch_bounds__(256, LOGN <= 8 ? WDD_CF_MINB_SMALL : WDD_CF_MINB_LARGE) colfft_kernel(const float2* __restrict__ R, const int32_t* __restrict__ rows,
                                                     int n_rows, const float2* __restrict__ tw,
                                                     const int32_t* __restrict__ col_off,
                                                     const int32_t* __restrict__ act_vy, float2* __restrict__ G,
                                                     const float2* __restrict__ W, float2* __restrict__ opart,
                                                     int64_t n_act, int logKT_rt, int K, float scale, int overwrite,
                                                     int tpc, int o_only, const __grid_constant__ CUtensorMap tmR,
                                                     int use_tma, int kbase, int KR, const int2* __restrict__ hmap) {
  // use_tma: bit 0 = R tiles by TMA, bit 3 = L2 prefetch of the output stage's W / G rows.
  // R holds the coefficient chunk kbase .. kbase + KR - 1 (row stride KR); G, W, opart are global.
  // hmap (Hermitian half plane, NULL = off): R holds only the primary columns (vx <= Sx/2); CTA
  // column blockIdx.y is R column jr, accumulator column hmap[jr].x, and hmap[jr].y the column of
  // -vx (-1: self-mirror).  The coefficients are real, so G[(-vy, -vx)][k] = conj G[(vy, vx)][k]
  // (the scan DFT of a real sequence, eq:outer_prod P:424): the mirror column's active rows are
  // written from the same transform, X[-vy] conjugated -- half the row-FFT output, R traffic
  // and y-FFTs.
  constexpr int Sy = 1 << LOGN;
  constexpr int PAD = FftPad<LOGC>::value;
  constexpr int kBY = PAD ? fft::Split<LOGN>::N2 : Sy < 256 ? Sy : 256;   // rows per TMA box (one block when padded)
  extern __shared__ __align__(16) float2 fsm[];
  const int logKT = LOGC >= 0 ? LOGC : logKT_rt;
  const int KT = 1 << logKT;
  auto xi = [&](int n) { return fft::pidx<LOGN, PAD>(n, logKT); };   // row n of the [Sy][KT] tile
  __shared__ int srow[Sy];                // staged rows
  __shared__ uint8_t sstaged[Sy];         // row staged (TMA path: the others are zeroed)
  __shared__ __align__(8) uint64_t lbar;
  __shared__ float2 sdot[Sy];             // per-row readout partial over this CTA's k-tiles
  __shared__ float2 sdm[Sy];
  constexpr bool TWG = LOGN >= WDD_CF_TWG_MINLOG, LAZY = LOGN >= WDD_CF_LAZY_MINLOG;
  __shared__ int svy[LAZY ? 1 : Sy];      // tile offset of the slot of each active vy of column j (!LAZY)
  __shared__ int svm[LAZY ? 1 : Sy];      // the same for the mirror column (slot of -vy)
  float2* x = fsm;                       // [Sy][KT] (+ PAD per block of N2 rows)
  float2* stw = fsm + xi(Sy);            // [Sy] twiddles (!TWG)
  const int jr = blockIdx.y;              // column of R
  int j = jr, jm = -1;
  if (hmap) {
    const int2 h = __ldg(hmap + jr);
    j = h.x;
    jm = h.y;
  }
  pdl_trigger();
  if ((use_tma & 1) && threadIdx.x == 0) {
    // the first k-tile's Sy x KT slice of R[j] in flight before the tables below load
    mbar_init(&lbar, 1);
    fence_mbar_init();
    pdl_wait();   // R (row DFT) of the preceding kernel
    mbar_arrive_expect_tx(&lbar, (uint32_t)(Sy * KT * 8));
    const int kl0 = blockIdx.x * tpc * KT;
    for (int b = 0; b < Sy / kBY; ++b)
      tma_load_2d(x + xi(b * kBY), &tmR, 2 * kl0, jr * Sy + b * kBY, &lbar);
  }
  const int g0 = __ldg(col_off + j), mj = __ldg(col_off + j + 1) - g0;
  const int gm0 = jm >= 0 ? __ldg(col_off + jm) : 0, mjm = jm >= 0 ? __ldg(col_off + jm + 1) - gm0 : 0;
  if constexpr (!TWG)
    for (int i = threadIdx.x; i < Sy; i += blockDim.x) stw[i] = __ldg(tw + i);
  for (int i = threadIdx.x; i < mj; i += blockDim.x) {
    if constexpr (!LAZY) svy[i] = xi(fft::fslot<LOGN>(__ldg(act_vy + g0 + i)));
    sdot[i] = make_float2(0.f, 0.f);
  }
  for (int i = threadIdx.x; i < mjm; i += blockDim.x) {
    if constexpr (!LAZY) svm[i] = xi(fft::fslot<LOGN>((Sy - __ldg(act_vy + gm0 + i)) & (Sy - 1)));
    sdm[i] = make_float2(0.f, 0.f);
  }
  if (use_tma & 1)
    for (int i = threadIdx.x; i < Sy; i += blockDim.x) sstaged[i] = n_rows < Sy ? 0 : 1;
  pdl_wait();   // R (row DFT) and G of the preceding kernels (and the uploaded row list)
  if (!(use_tma & 1) || n_rows < Sy)   // (a whole-scan TMA flush needs no row list)
    for (int i = threadIdx.x; i < n_rows; i += blockDim.x) srow[i] = __ldg(rows + i);
  if ((use_tma & 1) && n_rows < Sy) {
    __syncthreads();
    for (int i = threadIdx.x; i < n_rows; i += blockDim.x) sstaged[srow[i]] = 1;
  }
  for (int t = 0; t < tpc; ++t) {
  const int k0 = kbase + (blockIdx.x * tpc + t) * KT, kl = k0 - kbase;
  const int hKT = KT >> 1, lh = logKT - 1;             // 16-byte pieces per row
  if (use_tma & 1) {
    // the Sy x KT tile of R[j] in flight at once (pitch KT complex = the FFT's [Sy][KT] layout);
    // rows not staged are zeroed afterwards
    __syncthreads();                                   // x free (previous tile), sstaged set
    if (threadIdx.x == 0 && t > 0) {                   // (tile 0 was issued in the prologue)
      fence_proxy_async_smem();                        // generic writes of x before the async refill
      mbar_arrive_expect_tx(&lbar, (uint32_t)(Sy * KT * 8));
      for (int b = 0; b < Sy / kBY; ++b)
        tma_load_2d(x + xi(b * kBY), &tmR, 2 * kl, jr * Sy + b * kBY, &lbar);
    }
    mbar_wait(&lbar, (uint32_t)(t & 1));
    if (n_rows < Sy)
      for (int e = threadIdx.x; e < (Sy << logKT); e += blockDim.x)
        if (!sstaged[e >> logKT]) x[xi(e >> logKT) + (e & (KT - 1))] = make_float2(0.f, 0.f);
  } else {
  if (n_rows < Sy)
    for (int e = threadIdx.x; e < (Sy << logKT); e += blockDim.x) x[xi(e >> logKT) + (e & (KT - 1))] = make_float2(0.f, 0.f);
  __syncthreads();
  // staged rows of R[j] (k0 .. k0+KT), two coefficients (16 bytes) per load, kU loads in flight
  const float4* Rj = reinterpret_cast<const float4*>(R + (int64_t)jr * Sy * KR + kl);
  const int total = n_rows << lh;
  for (int base = 0; base < total; base += kU * (int)blockDim.x) {
    float4 v[kU];
    int dst[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = base + u * (int)blockDim.x + threadIdx.x;
      const int sy = e < total ? srow[e >> lh] : 0, h = e & (hKT - 1);
      dst[u] = e < total ? xi(sy) + 2 * h : -1;
      v[u] = e < total ? __ldg(Rj + (int64_t)sy * (KR >> 1) + h) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (dst[u] >= 0) *reinterpret_cast<float4*>(x + dst[u]) = v[u];
  }
  }
  if (use_tma & 8) {
    // the output stage's W (and G) rows of this k-tile into L2 while the transform runs: its
    // dependent load rounds then wait on L2, not DRAM
    const int lpr = KT >= 16 ? KT >> 4 : 1;            // 128-byte lines per row segment
    const bool pg = !overwrite && !o_only;
    for (int e = threadIdx.x; e < (mj + mjm) * lpr; e += blockDim.x) {
      const int i = e / lpr, l = e - i * lpr;
      const int64_t off = (int64_t)(i < mj ? g0 + i : gm0 + i - mj) * K + k0 + 16 * l;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(W + off));
      if (pg) asm volatile("prefetch.global.L2 [%0];" ::"l"(G + off));
    }
  }
  __syncthreads();
  fft::fft_seq<LOGN, LOGC, PAD, TWG>(x, TWG ? tw : stw, logKT);
  // Output: thread = (row slot, coefficient pair p); G (+)= X / sqrt(Sy) for the column's active
  // vy, and the tile's share of sum_k G K_v reduced over the hKT threads of the row.
  const int pp = threadIdx.x & (hKT - 1), rs = threadIdx.x >> lh, rpp = (int)blockDim.x >> lh;
  float4* G4 = reinterpret_cast<float4*>(G);
  const float4* W4 = reinterpret_cast<const float4*>(W);
  const int64_t K2 = K >> 1;
  // Rows 0 .. mj-1: column j; rows mj .. mj+mjm-1 (half plane): the mirror column, X[-vy]
  // conjugated -- one stream of rows, U rows per thread per round with their W (and G) segments in
  // flight together: 8 on the first flush after a reset (no G read), else 4.
  const int mt = mj + mjm;
  auto out_rows = [&](auto UC, auto RGC) {
    constexpr int U = decltype(UC)::value;
    constexpr bool RG = decltype(RGC)::value;
    constexpr bool BF = LOGC < 0 || LOGC >= WDD_CF_BF_MINLOGC;
    for (int ib = 0; ib < mt; ib += rpp * U) {           // block-uniform trip count (shuffles)
      float4 o[U], w[U];
      int vy[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = ib + u * rpp + rs;
        const int gr = i < mj ? g0 + i : gm0 + (i - mj);   // accumulator row
        const int64_t gi = (int64_t)gr * K2 + (k0 >> 1) + pp;
        if constexpr (LAZY) vy[u] = i < mt ? __ldg(act_vy + gr) : 0;   // (loaded with W: no table round)
        w[u] = i < mt ? __ldg(W4 + gi) : make_float4(0.f, 0.f, 0.f, 0.f);
        if constexpr (RG) o[u] = i < mt ? G4[gi] : make_float4(0.f, 0.f, 0.f, 0.f);
        else o[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float2 a[U];   // this thread's share of the tile's readout for each of its U rows
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = ib + u * rpp + rs;
        const bool mir = i >= mj;
        float2 d = make_float2(0.f, 0.f);
        if (i < mt) {
          // row of X: vy for column j, -vy for the mirror column (X[-vy] conjugated)
          const int sl = !LAZY ? (mir ? svm[i - mj] : svy[i])
                               : xi(fft::fslot<LOGN>(mir ? (Sy - vy[u]) & (Sy - 1) : vy[u]));
          const float cs = mir ? -scale : scale;
          const float4 z = *reinterpret_cast<const float4*>(x + sl + 2 * pp);
          // (fmaf(z.x, scale, o.x), fmaf(z.y, cs, o.y), ...) on packed pairs
          const float2 s2 = make_float2(scale, cs);
          const float2 g01 = __ffma2_rn(make_float2(z.x, z.y), s2, make_float2(o[u].x, o[u].y));
          const float2 g23 = __ffma2_rn(make_float2(z.z, z.w), s2, make_float2(o[u].z, o[u].w));
          const float4 gn = make_float4(g01.x, g01.y, g23.x, g23.y);
          const int gr = mir ? gm0 + (i - mj) : g0 + i;
          if (!o_only) G4[(int64_t)gr * K2 + (k0 >> 1) + pp] = gn;
          // d = g01 w01 + g23 w23 (complex), lane by lane the scalar chain
          // (fmaf(gn.x, w.x, fmaf(-gn.y, w.y, fmaf(gn.z, w.z, -gn.w * w.w))), fmaf(gn.x, w.y, fmaf(gn.y, w.x, ...)))
          const float2 w01 = make_float2(w[u].x, w[u].y), w23 = make_float2(w[u].z, w[u].w);
          float2 dd = __fmul2_rn(make_float2(-g23.y, g23.y), make_float2(w23.y, w23.x));
          dd = __ffma2_rn(make_float2(g23.x, g23.x), w23, dd);
          dd = __ffma2_rn(make_float2(-g01.y, g01.y), make_float2(w01.y, w01.x), dd);
          dd = __ffma2_rn(make_float2(g01.x, g01.x), w01, dd);
          d = dd;
        }
        a[u] = d;
        if constexpr (!BF) {   // plain xor tree per row, lane 0 of the row accumulates
          if (ib + u * rpp < mt) {                       // block-uniform
            for (int off = hKT >> 1; off > 0; off >>= 1) {
              d.x += __shfl_xor_sync(0xffffffffu, d.x, off);
              d.y += __shfl_xor_sync(0xffffffffu, d.y, off);
            }
            if (pp == 0 && i < mt) {
              float2* sp = mir ? sdm + (i - mj) : sdot + i;
              sp->x += d.x;
              sp->y += d.y;
            }
          }
        }
      }
      if constexpr (BF) {
      // Sum each row's hKT lane shares with a transposed butterfly: at offset off a lane keeps
      // half of its rows and sends the other half to lane ^ off, so every shuffle carries a useful
      // value (per U rows: U - U / hKT complex shuffles instead of U log2 hKT) and each lane ends
      // with whole-row sums of U / hKT rows (a row's sum, own share + partner share at every level,
      // is the lane-0 value of the plain xor tree bit for bit: fp addition is commutative).
      constexpr int LU = U >= 16 ? 4 : U >= 8 ? 3 : U >= 4 ? 2 : U >= 2 ? 1 : 0;
      int ub = 0, lv = 0;   // first row (u) of this lane's remaining values; levels done
#pragma unroll
      for (int L = 0; L < LU; ++L) {
        const int off = hKT >> (L + 1);
        if (off >= 1) {   // block-uniform
          const bool hi = (pp & off) != 0;
          const int h = U >> (L + 1);
#pragma unroll
          for (int j = 0; j < (U >> (L + 1)); ++j) {
            const float2 send = hi ? a[j] : a[j + (U >> (L + 1))];
            const float2 keep = hi ? a[j + (U >> (L + 1))] : a[j];
            const float rx = __shfl_xor_sync(0xffffffffu, send.x, off);
            const float ry = __shfl_xor_sync(0xffffffffu, send.y, off);
            a[j] = make_float2(keep.x + rx, keep.y + ry);
          }
          if (hi) ub += h;
          ++lv;
        }
      }
      // lanes beyond the transposition (hKT > U): plain xor tree on the one remaining value
      for (int off = hKT >> (LU + 1); off >= 1; off >>= 1) {
        a[0].x += __shfl_xor_sync(0xffffffffu, a[0].x, off);
        a[0].y += __shfl_xor_sync(0xffffffffu, a[0].y, off);
      }
      const int nfin = U >> lv;                            // rows per lane after the butterfly
      const bool writer = (pp & ((hKT >> lv) - 1)) == 0;   // one lane per row when hKT > U
#pragma unroll
      for (int j = 0; j < U; ++j) {
        if (j < nfin && writer) {
          const int i = ib + (ub + j) * rpp + rs;
          if (i < mt) {
            float2* sp = i >= mj ? sdm + (i - mj) : sdot + i;
            sp->x += a[j].x;
            sp->y += a[j].y;
          }
        }
      }
      }   // BF
    }
  };
  if (!overwrite && !o_only) out_rows(std::integral_constant<int, 4>{}, std::true_type{});
  else out_rows(std::integral_constant<int, LOGC == 3 ? WDD_CF_U_NOG_KT8 : WDD_CF_U_NOG>{}, std::false_type{});
  __syncthreads();   // x reused by the next k-tile; sdot settled
  }
  const int64_t orow = blockIdx.x + kbase / (KT * tpc);
  for (int i = threadIdx.x; i < mj; i += blockDim.x) opart[orow * n_act + g0 + i] = sdot[i];
  for (int i = threadIdx.x; i < mjm; i += blockDim.x) opart[orow * n_act + gm0 + i] = sdm[i];
}

static int ilog2(int v) { int l = 0; while ((1 << l) < v) ++l; return l; }

// Launch with programmatic dependent launch: the kernel may start (prologue: twiddles, tables)
// while the preceding kernel drains; it calls griddepcontrol.wait before touching that kernel's
// output.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              bool pdl, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// tuning override "a,b" from the environment (unset: (-1, 0))
static int2 env_pair(const char* name) {
  const char* e = std::getenv(name);
  int2 r = make_int2(-1, 0);
  if (e) std::sscanf(e, "%d,%d", &r.x, &r.y);
  return r;
}

static bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }
#ifndef WDD_FFT_SMEM
#define WDD_FFT_SMEM (64 * 1024)
#endif
constexpr int kFftSmem = WDD_FFT_SMEM;   // FFT working set per CTA (the twiddle table is added)

template <typename F>
static cudaError_t with_log(int logn, F&& f) {
  switch (logn) {
    case 1: return f(std::integral_constant<int, 1>{});
    case 2: return f(std::integral_constant<int, 2>{});
    case 3: return f(std::integral_constant<int, 3>{});
    case 4: return f(std::integral_constant<int, 4>{});
    case 5: return f(std::integral_constant<int, 5>{});
    case 6: return f(std::integral_constant<int, 6>{});
    case 7: return f(std::integral_constant<int, 7>{});
    case 8: return f(std::integral_constant<int, 8>{});
    case 9: return f(std::integral_constant<int, 9>{});
    case 10: return f(std::integral_constant<int, 10>{});
    default: return cudaErrorInvalidValue;
  }
}

// =====================================================================================
// a4 by DFT matrix (scan rows whose length is not a power of two):
//   R[j][sy][k] = sum_sx Fx[j][sx] C[sy*Sx + sx][k]   over pending positions (sx) only
// Tile: 16 active-vx columns j x 64 coefficients k of one scan row, 256 threads (2 j x 2 k each).
// Entries are staged 128 at a time (C 32 KB + twiddles 16 KB of shared memory) with all loads of
// a stage in flight at once; the next stage is prefetched into registers during the multiply.
// =====================================================================================
constexpr int kRdE = 128;                                  // entries per stage
constexpr int kRdSmem = kRdE * 64 * 4 + 16 * kRdE * 8;     // 48 KB

__global__ void __launch_bounds__(256) rowdft_kernel(const float* __restrict__ C, const int32_t* __restrict__ rows,
                                                     const uint32_t* __restrict__ masks, int mask_words,
                                                     const float2* __restrict__ Fx, float2* __restrict__ R,
                                                     int Sx, int Sy, int K, int n_vx) {
  extern __shared__ __align__(16) uint8_t rd_smem[];
  float* Cs = reinterpret_cast<float*>(rd_smem);                       // [kRdE][64]
  float2* Fs = reinterpret_cast<float2*>(rd_smem + kRdE * 64 * 4);     // [16][kRdE]
  const int t = threadIdx.x, kq = (t & 31) * 2, jg = t >> 5;           // k pair, j pair (0..7)
  const int k0 = blockIdx.x * 64, j0 = blockIdx.y * 16;
  const int sy = rows[blockIdx.z];
  const uint32_t* mrow = masks + (int64_t)blockIdx.z * mask_words;
  const float* Crow = C + (int64_t)sy * Sx * K + k0;
  float4 cv[8];   // 128 entries x 64 k / 256 threads = 8 float4
  float2 fv[8];   // 16 j x 128 entries / 256 threads = 8 float2
  auto load = [&](int e0) {
    const int ne = min(kRdE, Sx - e0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = t + 256 * i;
      const int ee = idx >> 4, kk = (idx & 15) * 4, sx = e0 + ee;
      cv[i] = (ee < ne && ((__ldg(mrow + (sx >> 5)) >> (sx & 31)) & 1u))
                  ? __ldg(reinterpret_cast<const float4*>(Crow + (int64_t)sx * K + kk))
                  : make_float4(0.f, 0.f, 0.f, 0.f);
      const int jj = idx >> 7, e2 = idx & (kRdE - 1);
      fv[i] = (e2 < ne && j0 + jj < n_vx) ? __ldg(Fx + (int64_t)(j0 + jj) * Sx + e0 + e2) : make_float2(0.f, 0.f);
    }
  };
  load(0);
  float2 acc[2][2];
#pragma unroll
  for (int q = 0; q < 2; ++q) acc[q][0] = acc[q][1] = make_float2(0.f, 0.f);
  for (int e0 = 0; e0 < Sx; e0 += kRdE) {
    const int ne = min(kRdE, Sx - e0);
    __syncthreads();   // previous stage fully consumed
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = t + 256 * i;
      *reinterpret_cast<float4*>(Cs + (idx >> 4) * 64 + (idx & 15) * 4) = cv[i];
      Fs[(idx >> 7) * kRdE + (idx & (kRdE - 1))] = fv[i];
    }
    __syncthreads();
    if (e0 + kRdE < Sx) load(e0 + kRdE);   // prefetch while computing
    const float2* f0 = Fs + (jg * 2) * kRdE;
    const float2* f1 = f0 + kRdE;
#pragma unroll 4
    for (int ee = 0; ee < ne; ++ee) {
      const float2 c = *reinterpret_cast<const float2*>(Cs + ee * 64 + kq);
      const float2 a = f0[ee], b = f1[ee];
      acc[0][0].x = fmaf(a.x, c.x, acc[0][0].x); acc[0][0].y = fmaf(a.y, c.x, acc[0][0].y);
      acc[0][1].x = fmaf(a.x, c.y, acc[0][1].x); acc[0][1].y = fmaf(a.y, c.y, acc[0][1].y);
      acc[1][0].x = fmaf(b.x, c.x, acc[1][0].x); acc[1][0].y = fmaf(b.y, c.x, acc[1][0].y);
      acc[1][1].x = fmaf(b.x, c.y, acc[1][1].x); acc[1][1].y = fmaf(b.y, c.y, acc[1][1].y);
    }
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = j0 + jg * 2 + q;
    if (j >= n_vx) continue;
    *reinterpret_cast<float4*>(R + ((int64_t)j * Sy + sy) * K + k0 + kq) =
        make_float4(acc[q][0].x, acc[q][0].y, acc[q][1].x, acc[q][1].y);
  }
}

static int rowfft_logp(const Plan& p) {
  static const int2 knob = env_pair("WDD_ROWFFT");   // (log2 k pairs per CTA, threads) override
  // k pairs per CTA (>= 2) and threads: up to Sx = 256, 16 pairs on 128 threads (twice the CTAs
  // of 32 pairs on 256: +0.8% Medium, +1% Large end to end); 256 threads beyond (Live: -0.5%)
  const int logSx = ilog2(p.Sx);
  int logP = ilog2(std::max(2, std::min(logSx <= 8 ? 16 : 32, kFftSmem / (8 * p.Sx))));
  if (knob.x >= 0) logP = std::min(logP, knob.x);
  while ((2 << logP) > p.Kl || p.Kl % (2 << logP)) --logP;
  return logP;
}

// compile-time tile width of the FFT flush kernels' specialised instances: the default logKT of
// the y-FFT from Sy = 128 and the default logP of the row FFT at Sx = 128 (-1: runtime width only;
// WDD_FFT_SPEC=0 off).  Measured (bench.py): y-FFT Box 1.82 -> 1.60 ms, Large 140 -> 131 us, Medium
// 18.8 -> 16.8 us; row FFT Medium 14.8 -> 12.5 us, but Box 0.91 -> 1.01 ms and Large 90 -> 94 us.
static constexpr int fft_spec_logc(int logn, bool row) {
#ifndef WDD_RF_SPEC_MAXLOG
#define WDD_RF_SPEC_MAXLOG 7
#endif
  return logn < 7 ? -1 : row ? (logn > WDD_RF_SPEC_MAXLOG ? -1 : logn == 10 ? 3 : 4) : (logn >= 10 ? 3 : logn == 9 ? 4 : 5);
}
static bool fft_spec_on() {
  static const bool on = [] { const char* e = std::getenv("WDD_FFT_SPEC"); return !(e && std::atoi(e) == 0); }();
  return on;
}

template <int LOGN, int LOGC>
static cudaError_t launch_rowfft_t(const Plan& p, const int32_t* rows, const uint32_t* masks, int n_rows,
                               cudaStream_t st, int kbase, int KR, int logP, int nt) {
  constexpr int PAD = FftPad<LOGC>::value;
  const size_t smem = ((size_t)p.Sx << logP) * 8 + (size_t)(p.Sx / fft::Split<LOGN>::N2) * PAD * 8 +
                      (LOGN >= WDD_RF_TWG_MINLOG ? 0 : (size_t)p.Sx * 8) + 16;
  {
    cudaError_t e = func_attr_once((const void*)rowfft_kernel<LOGN, LOGC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kFftSmem + 16384);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(KR / (2 << logP), n_rows);
  // (with two projection CTAs per SM a PDL-launched row FFT would park its CTAs next to the
  // last projection CTAs and slow them down: launch it after the projection completes -- unless
  // that projection ran fewer CTAs than SMs, where the parked CTAs take idle SMs and the launch
  // overlaps the projection's tail: Medium's 512-frame batches, 32 CTAs each, +1.6% end to end;
  // Box's and Large's full-width last batches -0.4% with PDL, tools/experiments/exp_rowpdl.sh)
  static const int env_pdl = [] { const char* e = std::getenv("WDD_ROWFFT_PDL"); return e ? std::atoi(e) : -1; }();
  const bool rowfft_pdl = env_pdl >= 0 ? env_pdl != 0 : !project_is_lean(p) || p.last_proj_grid < p.sm_count;
  CUtensorMap tmC;
  const bool tma = fft_tmap(&tmC, p.d_Call, (uint64_t)p.Kl, (uint64_t)p.S, (uint64_t)p.Kl * 4, 2u << logP,
                            (uint32_t)(PAD ? fft::Split<LOGN>::N2 : std::min(p.Sx, 256)));
  // (Hermitian half plane, p.r_half: only the primary columns vx <= Sx/2 go to R)
  return launch_pdl(rowfft_kernel<LOGN, LOGC>, grid, dim3(nt), smem, st, rowfft_pdl, (const float*)p.d_Call, rows, masks,
                    p.mask_words, (const float2*)p.d_twx,
                    (const int32_t*)(p.r_half ? (p.half_identity ? nullptr : p.d_col_vx_half) : p.d_col_vx), p.d_R, logP, p.Sy, p.Kl,
                    p.r_half ? p.n_vh : p.n_vx, (float)(1.0 / std::sqrt((double)p.Sx)), tmC,
                    (tma ? 1 : 0) | (rowfft_pdl ? 2 : 0) | (masks == p.d_ones ? 4 : 0),
                    kbase, KR);
}

cudaError_t launch_rowdft(const Plan& p, const int32_t* rows, const uint32_t* masks, int n_rows, cudaStream_t st,
                          int kbase, int KR) {
  if (KR <= 0) { kbase = 0; KR = p.Kl; }
  if (n_rows <= 0) return cudaSuccess;
  if (is_pow2(p.Sx) && p.Sx >= 2 && p.Sx <= (1 << kFftMaxLog)) {
    const int logSx = ilog2(p.Sx);
    static const int2 knob = env_pair("WDD_ROWFFT");   // (log2 k pairs per CTA, threads) override
    // k pairs per CTA (>= 2) and threads: up to Sx = 256, 16 pairs on 128 threads (twice the CTAs
    // of 32 pairs on 256: +0.8% Medium, +1% Large end to end); 256 threads beyond (Live: -0.5%)
    const int logP = rowfft_logp(p);
    const int nt = knob.y > 0 ? knob.y : logSx <= 8 ? 128 : 256;
    return with_log(logSx, [&](auto LN) {
      constexpr int LOGN = decltype(LN)::value;
      constexpr int SPEC = fft_spec_logc(LOGN, true);
      if constexpr (SPEC >= 0)
        if (logP == SPEC && fft_spec_on()) return launch_rowfft_t<LOGN, SPEC>(p, rows, masks, n_rows, st, kbase, KR, logP, nt);
      return launch_rowfft_t<LOGN, -1>(p, rows, masks, n_rows, st, kbase, KR, logP, nt);
    });
  }
  {
    cudaError_t e = func_attr_once((const void*)rowdft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kRdSmem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(p.Kl / 64, (p.n_vx + 15) / 16, n_rows);
  rowdft_kernel<<<grid, 256, kRdSmem, st>>>(p.d_Call, rows, masks, p.mask_words, p.d_Fx, p.d_R, p.Sx, p.Sy, p.Kl,
                                            p.n_vx);
  return cudaGetLastError();
}

// =====================================================================================
// a5 by DFT matrix (flush of a few rows, or Sy not a power of two):
//   G[(j,vy)][k] += sum_{staged rows} Fy[vy][sy] R[j][sy][k]
// =====================================================================================
__global__ void __launch_bounds__(256) flush_kernel(const float2* __restrict__ R, const float2* __restrict__ Fy,
                                                    const int32_t* __restrict__ rows, int n_rows,
                                                    const int2* __restrict__ tiles, const int32_t* __restrict__ col_off,
                                                    const int32_t* __restrict__ act_vy, float2* __restrict__ G,
                                                    int Sy, int K, int overwrite) {
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
      const float2 o = overwrite ? make_float2(0.f, 0.f) : *ptr;
      *ptr = make_float2(o.x + acc[q].x, o.y + acc[q].y);
    }
  }
}

// =====================================================================================
// a5 + a6 on the tensor cores: the phase-weighted rank update as the batched complex GEMM of the
// north star,  G[(j, vy)][k] (+)= sum_r F[vy][r] R[j][row_r][k],  F[vy][r] = W_Sy^{vy row_r}/sqrt(Sy)
// (the DFT matrix of eq:outer_prod / P:411-414 restricted to the active vy of column j and the
// staged rows), with the tile's share of the Wiener readout sum_k G K_v fused into the epilogue.
// CTA = (column j, tile of 128 active vy, tile of NT coefficients); the K dimension runs over the
// staged rows, 32 rows (64 real K: re / im parts) per chunk, double-buffered in shared memory.
// Complex -> real: D_re = [Fr | -Fi] x [Rr ; Ri], D_im = [Fi | Fr] x [Rr ; Ri] (two fp32 TMEM
// accumulators, M = 128 vy rows, N = NT).  Precision: both operands split into bf16 hi + lo,
// three passes (hi.hi + hi.lo + lo.hi), fp32 accumulation (~1e-5 relative per term).
// =====================================================================================
constexpr int kCgM = 128;                                  // active vy per tile (MMA M)
constexpr uint32_t kCgLBOA = (kCgM / 8) * 128;             // A (K-major): bytes between K-adjacent core matrices

// CTA = (column j, tile of 128 active vy, k-chunk): the A operand (the F tile of all staged rows,
// <= kCgRows rows) is built once; the CTA then walks its k-chunk in NT-coefficient tiles with the
// B tile of the next tile built (R -> bf16 hi / lo) while the MMAs of the current one run, and the
// epilogue of a tile overlapping the MMAs of the next (two TMEM accumulator pairs).  Each thread
// owns one vy row and half the tile's coefficients, so the Wiener-readout dot product accumulates
// in registers across the whole k-chunk.
constexpr int kCgRows = 64;                                 // staged rows the GEMM form takes
constexpr int kCgKmax = 2 * kCgRows;                        // real K (re / im parts)
constexpr int kCgAfull = kCgM * kCgKmax * 2;                // one A plane over all staged rows (32 KB)
constexpr int kCgNT = 64;                                   // coefficients per tile
constexpr int kCgBt = kCgNT * kCgKmax * 2;                  // one B plane of a tile (16 KB)
constexpr uint32_t kCgSBOBf = (kCgKmax / 8) * 128;          // B (MN-major): N-adjacent core matrices
constexpr int kCgSmem = 4 * kCgAfull + 2 * 2 * kCgBt;       // A [acc][plane] + B [buf][plane] = 192 KB

__global__ void __launch_bounds__(256, 1) colgemm_kernel(const float2* __restrict__ R, const int32_t* __restrict__ rows,
                                                         int n_rows, const float2* __restrict__ tw, int Sy,
                                                         float inv_sqrt_sy, const int32_t* __restrict__ col_off,
                                                         const int32_t* __restrict__ act_vy, float2* __restrict__ G,
                                                         const float2* __restrict__ W, float2* __restrict__ opart,
                                                         int64_t n_act, int K, int ktiles, int overwrite, int o_only) {
  extern __shared__ __align__(1024) uint8_t cg_smem[];
  __shared__ int svy[kCgM];
  __shared__ int srow[kCgRows];
  __shared__ uint64_t mma_done[2];
  __shared__ uint32_t tslot;
  __shared__ float2 sdot[kCgM];
  uint8_t* sA = cg_smem;                                     // [acc re/im][plane hi/lo]
  uint8_t* sB = cg_smem + 4 * kCgAfull;                      // [buf][plane]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j = blockIdx.z, vt = blockIdx.y, kc = blockIdx.x;
  pdl_trigger();
  const int g0 = __ldg(col_off + j), mj = __ldg(col_off + j + 1) - g0;
  const int i0 = vt * kCgM;
  if (i0 >= mj) return;                                      // (grid covers the longest column)
  const int kr = (n_rows + 7) & ~7;                          // rows used, padded to a core matrix
  const int kreal = 2 * kr;                                  // real K
  if (tid < kCgM) svy[tid] = i0 + tid < mj ? __ldg(act_vy + g0 + i0 + tid) : -1;
  if (tid == 0) {
    mbar_init(&mma_done[0], 1);
    mbar_init(&mma_done[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<4 * kCgNT>(&tslot);
  pdl_wait();                                                // R of the row DFT, G of earlier flushes
  if (tid < kr) srow[tid] = tid < n_rows ? rows[tid] : -1;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  const bool sy_pow2 = (Sy & (Sy - 1)) == 0;
  // A (K-major, M = 128): element (m, k) at (k/8)*LBO + (m/8)*128 + (m%8)*16 + (k%8)*2, k = d*kr + r;
  // thread -> (vy row m, group of 8 staged rows): 8 twiddles -> 16-byte stores
  for (int w = tid; w < kCgM * (kr / 8); w += 256) {
    const int m = w % kCgM, rg = w / kCgM;
    const int vy = svy[m];
    float fr[8], fi[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int row = srow[rg * 8 + e];
      float2 f = make_float2(0.f, 0.f);
      if (vy >= 0 && row >= 0) f = __ldg(tw + (sy_pow2 ? ((vy * row) & (Sy - 1)) : (int)(((int64_t)vy * row) % Sy)));
      fr[e] = f.x * inv_sqrt_sy;
      fi[e] = f.y * inv_sqrt_sy;
    }
    const uint32_t off_re = (uint32_t)rg * kCgLBOA + (m >> 3) * 128 + (m & 7) * 16;
    const uint32_t off_im = off_re + (uint32_t)(kr / 8) * kCgLBOA;
    uint32_t h[4], l[4], hn[4], ln[4], hp[4], lp[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      split_bf16x2(fr[2 * e], fr[2 * e + 1], h[e], l[e]);
      split_bf16x2(-fi[2 * e], -fi[2 * e + 1], hn[e], ln[e]);
      split_bf16x2(fi[2 * e], fi[2 * e + 1], hp[e], lp[e]);
    }
    *reinterpret_cast<uint4*>(sA + 0 * kCgAfull + off_re) = make_uint4(h[0], h[1], h[2], h[3]);     // re: [Fr | -Fi]
    *reinterpret_cast<uint4*>(sA + 1 * kCgAfull + off_re) = make_uint4(l[0], l[1], l[2], l[3]);
    *reinterpret_cast<uint4*>(sA + 0 * kCgAfull + off_im) = make_uint4(hn[0], hn[1], hn[2], hn[3]);
    *reinterpret_cast<uint4*>(sA + 1 * kCgAfull + off_im) = make_uint4(ln[0], ln[1], ln[2], ln[3]);
    *reinterpret_cast<uint4*>(sA + 2 * kCgAfull + off_re) = make_uint4(hp[0], hp[1], hp[2], hp[3]); // im: [Fi | Fr]
    *reinterpret_cast<uint4*>(sA + 3 * kCgAfull + off_re) = make_uint4(lp[0], lp[1], lp[2], lp[3]);
    *reinterpret_cast<uint4*>(sA + 2 * kCgAfull + off_im) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(sA + 3 * kCgAfull + off_im) = make_uint4(l[0], l[1], l[2], l[3]);
  }
  const int kbase = kc * ktiles * kCgNT;
  const float2* Rj = R + (int64_t)j * Sy * K;
  // B (MN-major, N = NT): element (n, k) at (n/8)*SBO + (k/8)*128 + (k%8)*16 + (n%8)*2, k = d*kr + r
  auto build_b = [&](int t, int buf) {
    uint8_t* sb = sB + buf * 2 * kCgBt;
    const int k0 = kbase + t * kCgNT;
    for (int w = tid; w < kr * (kCgNT / 8); w += 256) {
      const int r = w % kr, nb = w / kr;
      const int row = srow[r];
      float4 v[4];
      if (row >= 0) {
        const float4* src = reinterpret_cast<const float4*>(Rj + (int64_t)row * K + k0 + nb * 8);
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = __ldg(src + e);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      uint32_t rh[4], rl[4], ih[4], il[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        split_bf16x2(v[e].x, v[e].z, rh[e], rl[e]);
        split_bf16x2(v[e].y, v[e].w, ih[e], il[e]);
      }
      const uint32_t off = nb * kCgSBOBf + (r >> 3) * 128 + (r & 7) * 16;
      const uint32_t offi = off + (uint32_t)(kr / 8) * 128;
      *reinterpret_cast<uint4*>(sb + off) = make_uint4(rh[0], rh[1], rh[2], rh[3]);
      *reinterpret_cast<uint4*>(sb + kCgBt + off) = make_uint4(rl[0], rl[1], rl[2], rl[3]);
      *reinterpret_cast<uint4*>(sb + offi) = make_uint4(ih[0], ih[1], ih[2], ih[3]);
      *reinterpret_cast<uint4*>(sb + kCgBt + offi) = make_uint4(il[0], il[1], il[2], il[3]);
    }
  };
  constexpr uint32_t idesc = idesc_f16(kCgM, kCgNT, /*bf16*/ 1, /*a K-major*/ 0, /*b MN-major*/ 1);
  auto issue = [&](int t) {   // thread 0: MMAs of tile t into TMEM pair t & 1
    tc_fence_after();
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB + (t & 1) * 2 * kCgBt);
    const uint32_t d0 = tbase + (t & 1) * 2 * kCgNT;
    bool first = true;
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {                   // hi.hi, hi.lo, lo.hi
      const int pa = pass == 2 ? 1 : 0, pb = pass == 1 ? 1 : 0;
#pragma unroll 1
      for (int kk = 0; kk < kreal / 16; ++kk) {
#pragma unroll
        for (int acc = 0; acc < 2; ++acc) {
          const uint64_t ad = smem_desc_noswz(a0 + (acc * 2 + pa) * kCgAfull + kk * 2 * kCgLBOA, kCgLBOA, 128);
          const uint64_t bd = smem_desc_noswz(b0 + pb * kCgBt + kk * 256, 128, kCgSBOBf);
          mma_f16_ss(d0 + acc * kCgNT, ad, bd, idesc, first ? 0u : 1u);
        }
        first = false;
      }
    }
    mma_commit(&mma_done[t & 1]);
  };
  build_b(0, 0);
  fence_proxy_async_smem();
  __syncthreads();
  if (tid == 0) issue(0);
  const int quad = warp & 3, half = warp >> 2;
  const int m = quad * 32 + lane;
  const bool valid = svy[m] >= 0;
  const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
  const int64_t grow = (int64_t)(g0 + i0 + m) * K;
  float2 dot = make_float2(0.f, 0.f);
  for (int t = 0; t < ktiles; ++t) {
    if (t + 1 < ktiles) {
      if (t >= 1) mbar_wait(&mma_done[(t + 1) & 1], ((t - 1) >> 1) & 1u);   // B buffer of tile t - 1 free
      build_b(t + 1, (t + 1) & 1);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncthreads();                                       // (also: epilogue t - 1 done with TMEM pair)
      if (tid == 0) issue(t + 1);
    }
    mbar_wait(&mma_done[t & 1], (t >> 1) & 1u);
    tc_fence_after();
    // epilogue of tile t: G (+)= D, dot += G K over this thread's row and half of the coefficients
    const uint32_t d0 = tbase + lane_addr + (t & 1) * 2 * kCgNT + half * (kCgNT / 2);
    float dr[kCgNT / 2], di[kCgNT / 2];
    tmem_ld_cols<kCgNT / 2>(d0, dr);
    tmem_ld_cols<kCgNT / 2>(d0 + kCgNT, di);
    if (valid) {
      const int k0 = kbase + t * kCgNT + half * (kCgNT / 2);
      float4* Gr = reinterpret_cast<float4*>(G + grow + k0);
      const float4* Wr = reinterpret_cast<const float4*>(W + grow + k0);
      float4 o[kCgNT / 4], w[kCgNT / 4];
#pragma unroll
      for (int q = 0; q < kCgNT / 4; ++q) {
        o[q] = (overwrite || o_only) ? make_float4(0.f, 0.f, 0.f, 0.f) : Gr[q];
        w[q] = __ldg(Wr + q);
      }
#pragma unroll
      for (int q = 0; q < kCgNT / 4; ++q) {
        const float4 gn = make_float4(o[q].x + dr[2 * q], o[q].y + di[2 * q], o[q].z + dr[2 * q + 1], o[q].w + di[2 * q + 1]);
        if (!o_only) Gr[q] = gn;
        dot.x = fmaf(gn.x, w[q].x, fmaf(-gn.y, w[q].y, fmaf(gn.z, w[q].z, fmaf(-gn.w, w[q].w, dot.x))));
        dot.y = fmaf(gn.x, w[q].y, fmaf(gn.y, w[q].x, fmaf(gn.z, w[q].w, fmaf(gn.w, w[q].z, dot.y))));
      }
    }
    tc_fence_before();
  }
  if (half == 1) sdot[m] = dot;
  __syncthreads();
  if (half == 0 && valid) {
    const float2 d1 = sdot[m];
    opart[(int64_t)kc * n_act + g0 + i0 + m] = make_float2(dot.x + d1.x, dot.y + d1.y);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<4 * kCgNT>(tbase);
}

// =====================================================================================
// a5 + a6 on the tensor cores, memory-pipelined (flushes of <= 64 rows: the Live cadence).
//   G[(j, vy)][k] (+)= sum_r F[vy][r] R[j][sy_r][k],  F[vy][r] = W_Sy^{vy sy_r} / sqrt(Sy)
// (eq:outer_prod, restricted to the active vy of column j and the flush's rows r),
// with the Wiener readout sum_k G K_v accumulated per vy row in the epilogue.
// Persistent CTAs walk work items (column j, 128 active vy, k-chunk) in 32-coefficient MMA tiles.
// Two shared-memory rings with different lifetimes:
//   B ring (NB x 16 KB)   the R tile (flush rows x 32 complex, fp32, TMA SWIZZLE_128B boxes; one
//                         bulk copy per row when the rows are not contiguous), converted in place to
//                         bf16 hi / lo planes of B = [Rr | Ri] (N = 64, MN-major, K = flush row);
//                         freed by the MMA commit;
//   W/G ring (2 x 3 x 32 KB, three stages owned by each epilogue group)
//                         per 16-coefficient half tile one SWIZZLE_128B box of W and one of G
//                         (G only when read: not on the first flush after a reset, not for
//                         spectrum-only plans; 16-row boxes for the tail tile of a column); freed
//                         by the epilogue.
// Roles:  warp 0 producer (TMA); warps 2-3 converters; warp 1 MMA issuer: D1 = Fr B, D2 = Fi B as
// bf16 three-pass products (hi.hi + hi.lo + lo.hi, fp32 accumulation), A = F from TMEM (built once
// per item), M = 128, N = 64, K = 16 per instruction; warps 4-7 and 8-11 two epilogue groups taking
// alternate MMA tiles, thread = one vy row (TMEM lane): D_re = Fr Rr - Fi Ri, D_im = Fr Ri + Fi Rr,
// G (+)= D stored, dot += G K_v; the dot of the whole k-chunk lands in opart[chunk][g].
// =====================================================================================
constexpr int kRgNT = 32;                                    // coefficients per MMA tile
constexpr int kRgN = 2 * kRgNT;                              // MMA N: [Rr | Ri]
constexpr int kRgRows = 64;                                  // flush rows the GEMM form takes (MMA K)
constexpr int kRgPlaneB = (kRgN / 8) * (kRgRows / 8) * 128;  // 8 KB: element (n, r) at
                                                             // (n/8)*1024 + (r/8)*128 + (r%8)*16 + (n%8)*2
constexpr int kRgStB = 2 * kRgPlaneB;                        // 16 KB = the fp32 R tile (two 128-B halves x 64 rows)
constexpr int kRgHalfR = kRgRows * 128;                      // 8 KB: one 16-coefficient half of the R tile
constexpr int kRgM = 128;
#ifndef WDD_RG_NB
#define WDD_RG_NB 2
#endif
constexpr int kRgNB = WDD_RG_NB;                             // B ring depth (MMA tiles)
constexpr int kRgBoxGW = kRgM * 128;                         // 16 KB: 128 rows x 16 complex
constexpr int kRgStWG = 2 * kRgBoxGW;                        // 32 KB: W box + G box of one half tile
#ifndef WDD_RG_NWG
#define WDD_RG_NWG 3
#endif
// W/G stages per epilogue group.  Each group owns its stages: the two groups run out of lockstep,
// and a barrier shared by both would let the group that is ahead pass a parity wait on a phase two
// behind (observed as rare hangs and faults with 5 shared stages)
constexpr int kRgNWG = WDD_RG_NWG;
constexpr int kRgNW = 2 * kRgNWG;                            // W/G ring depth (half tiles)
constexpr int kRgNAcc = 2;                                   // TMEM accumulator ring depth
constexpr int kRgOffWG = kRgNB * kRgStB;
constexpr int kRgBarOff = kRgOffWG + kRgNW * kRgStWG;
constexpr int kRgNBars = 3 * kRgNB + 2 * kRgNW + 2 * kRgNAcc + 1;
constexpr int kRgSmem = kRgBarOff + 8 * kRgNBars + 16 + 4 * kRgRows + 2 * kRgM * 8;
constexpr int kRgThreads = 384;   // producer, MMA, 2 converter warps, 2 x 4 epilogue warps
constexpr int kRgFCols = kRgRows / 2;                        // TMEM columns of one F plane (bf16 pairs)
constexpr int kRgTmemF = 0;                                  // planes: Fr hi, Fr lo, Fi hi, Fi lo
constexpr int kRgTmemAcc = 4 * kRgFCols;                     // 128: [acc][D1 | D2], 2 x 64 columns each
constexpr int kRgTmemCols = 512;
static_assert(kRgSmem <= 232448, "rgemm shared memory");
static_assert(kRgTmemAcc + kRgNAcc * 2 * kRgN <= kRgTmemCols, "rgemm TMEM");

#ifdef WDD_RG_DEBUG
// hang hunting: per CTA and role the tile counter and the barrier being waited for (readable by
// the host on a side stream while the kernel runs: wdd_rg_debug)
__device__ unsigned g_rgdbg[148 * 8];
#define RGDBG(role, c, code) do { *(volatile unsigned*)&g_rgdbg[blockIdx.x * 8 + (role)] = ((c) << 8) | (code); } while (0)
#else
#define RGDBG(role, c, code)
#endif

struct RgArgs {
  const float2* R;           // R[j][sy][k]
  const int32_t* rows;       // flush row r -> scan row
  int n_rows;
  const float2* tw;          // Sy FFT twiddles
  int Sy;
  float inv_sqrt_sy;
  const int32_t* col_off;
  const int32_t* act_vy;
  const int2* items;         // (column j, first vy i0)
  int n_items;               // item tiles (j, i0); work items = n_items * n_kc
  int n_kc;                  // k-chunks per item tile
  float2* G;
  float2* opart;
  int64_t n_act;
  int K;
  int read_g, write_g;
  int row0;                  // >= 0: the flush rows are row0 .. row0 + n_rows - 1 (TMA boxes of R)
};

// Tensor maps (TMA), all with 16-complex (128-byte) inner boxes and SWIZZLE_128B: W and G with
// 16- and 128-row boxes (one 128-row box per full tile reads ~1.6x faster than eight 16-row
// boxes: tools/tma_stride_probe.cu), R with 16- and 64-row boxes.
struct RgMaps {
  CUtensorMap w16, g16, w128, g128, r16, r64;
};

__global__ void __launch_bounds__(kRgThreads, 1) rgemm_kernel(RgArgs a, const __grid_constant__ RgMaps tm) {
  extern __shared__ __align__(1024) uint8_t rg_smem[];
  TRACE_DECL
  uint64_t* bars = reinterpret_cast<uint64_t*>(rg_smem + kRgBarOff);
  uint64_t* r_full = bars;                    // [NB] R tile landed (TMA tx)
  uint64_t* b_full = r_full + kRgNB;          // [NB] B planes written (2 converter warps)
  uint64_t* b_empty = b_full + kRgNB;         // [NB] MMA commit
  uint64_t* wg_full = b_empty + kRgNB;        // [NW] W / G half tile landed (TMA tx)
  uint64_t* wg_empty = wg_full + kRgNW;       // [NW] the epilogue group's store issuer (after the TMA store read it)
  uint64_t* acc_full = wg_empty + kRgNW;      // [NAcc]
  uint64_t* acc_empty = acc_full + kRgNAcc;   // [NAcc] 4 epilogue warps
  uint64_t* f_full = acc_empty + kRgNAcc;     // F of the current item in TMEM
  uint32_t* tslot = reinterpret_cast<uint32_t*>(f_full + 1);
  int* srow = reinterpret_cast<int*>(tslot + 4);
  float2* sdot = reinterpret_cast<float2*>(srow + kRgRows);   // [2][128] group-1 partial dots
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KT = a.K / kRgNT, kt_per = KT / a.n_kc;          // MMA tiles per work item
  const int kr = (a.n_rows + 15) & ~15;
  const int64_t n_work = (int64_t)a.n_items * a.n_kc;
  if (tid == 0) {
    for (int i = 0; i < kRgNB; ++i) { mbar_init(&r_full[i], 1); mbar_init(&b_full[i], 2); mbar_init(&b_empty[i], 1); }
    for (int i = 0; i < kRgNW; ++i) { mbar_init(&wg_full[i], 1); mbar_init(&wg_empty[i], 1); }
    for (int i = 0; i < kRgNAcc; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 4); }
    mbar_init(f_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<kRgTmemCols>(tslot);
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm.w16); prefetch_tmap(&tm.g16); prefetch_tmap(&tm.w128);
    prefetch_tmap(&tm.g128); prefetch_tmap(&tm.r16); prefetch_tmap(&tm.r64);
  }
  pdl_trigger();
  pdl_wait();   // R of the row FFT, G / opart of earlier kernels
  if (tid < kRgRows) srow[tid] = tid < a.n_rows ? __ldg(a.rows + tid) : 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    // ---------------- producer: per MMA tile c the R tile (B ring), then its two W / G half tiles
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();             // W and G: each byte read once per flush
      const int kr16 = (a.n_rows + 15) >> 4;
      const uint32_t rbytes = 2 * (a.row0 >= 0 ? kr16 * 16 : a.n_rows) * 128;
      uint32_t c = 0;
      for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x) {
        const int2 it = a.items[w / a.n_kc];
        const int kc = (int)(w % a.n_kc);
        const int g0 = __ldg(a.col_off + it.x), grow = g0 + it.y;
        // W / G rows of this item only: the tail tile of a column must not pull in the next
        // column's rows (16-row boxes there)
        const int nb16 = (min(kRgM, __ldg(a.col_off + it.x + 1) - grow) + 15) >> 4;
        const uint32_t wgbytes = nb16 * 16 * 128 * (a.read_g ? 2 : 1);
        const float2* Rj = a.R + (int64_t)it.x * a.Sy * a.K;
        for (int t = 0; t < kt_per; ++t, ++c) {
          const int kt = kc * kt_per + t;
          // R tile
          {
            const int sb = c % kRgNB;
            RGDBG(0, c, 1);
            mbar_wait(&b_empty[sb], ((c / kRgNB) & 1u) ^ 1u);
            TRACE(0, c);
            uint8_t* st = rg_smem + sb * kRgStB;
            mbar_arrive_expect_tx(&r_full[sb], rbytes);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int x = (kt * 2 + h) * 32;               // float column of the half
              if (a.row0 >= 0) {
                if (kr16 == 4) {
                  tma_load_2d(st + h * kRgHalfR, &tm.r64, x, it.x * a.Sy + a.row0, &r_full[sb]);
                } else {
                  for (int b = 0; b < kr16; ++b)
                    tma_load_2d(st + h * kRgHalfR + b * 16 * 128, &tm.r16, x, it.x * a.Sy + a.row0 + 16 * b, &r_full[sb]);
                }
              } else {
                for (int r = 0; r < a.n_rows; ++r)
                  bulk_load(st + h * kRgHalfR + r * 128, Rj + (int64_t)srow[r] * a.K + kt * kRgNT + h * 16, 128,
                            &r_full[sb]);
              }
            }
          }
          // W / G half tiles
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            const uint32_t u = (c >> 1) * 2 + h;              // half tile index within the group (c & 1)
            const int sw = (int)(c & 1u) * kRgNWG + (int)(u % kRgNWG);
            RGDBG(0, c, 2 + h);
            mbar_wait(&wg_empty[sw], ((u / kRgNWG) & 1u) ^ 1u);
            uint8_t* st = rg_smem + kRgOffWG + sw * kRgStWG;
            const int x = (kt * 2 + h) * 32;
            mbar_arrive_expect_tx(&wg_full[sw], wgbytes);
            if (nb16 == kRgM / 16) {
              tma_load_2d_hint(st, &tm.w128, x, grow, &wg_full[sw], pol);
              if (a.read_g) tma_load_2d_hint(st + kRgBoxGW, &tm.g128, x, grow, &wg_full[sw], pol);
            } else {
              for (int b = 0; b < nb16; ++b) {
                tma_load_2d_hint(st + b * 16 * 128, &tm.w16, x, grow + 16 * b, &wg_full[sw], pol);
                if (a.read_g) tma_load_2d_hint(st + kRgBoxGW + b * 16 * 128, &tm.g16, x, grow + 16 * b, &wg_full[sw], pol);
              }
            }
          }
        }
      }
    }
  } else if (warp == 2 || warp == 3) {
    // ---------------- converters: thread = flush row r, groups q8 = 0..3 of 8 coefficients: 64 bytes
    // of R in, 16 bytes per plane out per group, in place (every row is read before any is written)
    const int ct = tid - 64;
    const int swz_mask = a.row0 >= 0 ? 7 : 0;              // TMA rows arrive SWIZZLE_128B
    uint32_t c = 0;
    for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x) {
      for (int t = 0; t < kt_per; ++t, ++c) {
        const int sb = c % kRgNB;
        if (ct == 0) RGDBG(1, c, 1);
        mbar_wait(&r_full[sb], (c / kRgNB) & 1u);
        if (ct == 0) RGDBG(1, c, 2);
        if (ct == 0) TRACE(1, c);
        uint8_t* st = rg_smem + sb * kRgStB;
        float4 v[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = ct, q8 = i;                        // a warp phase = 8 rows, one group: no bank conflicts
          const int h = q8 >> 1;                             // 16-coefficient half
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int chunk = ((q8 & 1) * 4 + u) ^ (r & swz_mask);
            v[i][u] = r < a.n_rows ? *reinterpret_cast<const float4*>(st + h * kRgHalfR + r * 128 + chunk * 16)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        named_sync(2, 64);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = ct, q8 = i;                        // a warp phase = 8 rows, one group: no bank conflicts
          if (r < kr) {
            uint32_t rh[4], rl[4], ih[4], il[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {                  // complex 2u, 2u + 1 of the group
              split_bf16x2(v[i][u].x, v[i][u].z, rh[u], rl[u]);
              split_bf16x2(v[i][u].y, v[i][u].w, ih[u], il[u]);
            }
            uint8_t* d = st + (r >> 3) * 128 + (r & 7) * 16;
            *reinterpret_cast<uint4*>(d + q8 * 1024) = make_uint4(rh[0], rh[1], rh[2], rh[3]);
            *reinterpret_cast<uint4*>(d + (4 + q8) * 1024) = make_uint4(ih[0], ih[1], ih[2], ih[3]);
            *reinterpret_cast<uint4*>(d + kRgPlaneB + q8 * 1024) = make_uint4(rl[0], rl[1], rl[2], rl[3]);
            *reinterpret_cast<uint4*>(d + kRgPlaneB + (4 + q8) * 1024) = make_uint4(il[0], il[1], il[2], il[3]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&b_full[sb]);
        if (ct == 0) TRACE(2, c);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16(kRgM, kRgN, /*bf16*/ 1, /*A K-major*/ 0, /*B MN-major*/ 1);
      const int nkk = kr / 16;
      uint32_t c = 0, item = 0;
      for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x, ++item) {
        RGDBG(2, c, 1);
        mbar_wait(f_full, item & 1u);                        // F of this item in TMEM
        for (int t = 0; t < kt_per; ++t, ++c) {
          const int sb = c % kRgNB, ac = c % kRgNAcc;
          RGDBG(2, c, 2);
          mbar_wait(&b_full[sb], (c / kRgNB) & 1u);
          RGDBG(2, c, 3);
          mbar_wait(&acc_empty[ac], ((c / kRgNAcc) & 1u) ^ 1u);
          RGDBG(2, c, 4);
          TRACE(3, c);
          tc_fence_after();
          // descriptors: one base per stage, offsets added to the address field (addr >> 4)
          const uint64_t bdesc = smem_desc_noswz(smem_u32(rg_smem + sb * kRgStB), 128, 1024);
          const uint32_t d1 = tbase + kRgTmemAcc + ac * 2 * kRgN, d2 = d1 + kRgN;
#pragma unroll
          for (int pass = 0; pass < 3; ++pass) {             // hi.hi, hi.lo, lo.hi
            const int fa = pass == 2 ? 1 : 0, pb = pass == 1 ? 1 : 0;
            const uint32_t fr = tbase + kRgTmemF + (0 + fa) * kRgFCols;
            const uint32_t fi = tbase + kRgTmemF + (2 + fa) * kRgFCols;
#pragma unroll
            for (int kk = 0; kk < kRgRows / 16; ++kk) {
              if (kk < nkk) {
                const uint64_t bd = bdesc + (uint64_t)((pb * kRgPlaneB + kk * 256) >> 4);
                const uint32_t acc = (pass > 0 || kk > 0) ? 1u : 0u;
                mma_f16_ts(d1, fr + kk * 8, bd, idesc, acc);
                mma_f16_ts(d2, fi + kk * 8, bd, idesc, acc);
              }
            }
          }
          mma_commit(&b_empty[sb]);                          // B planes consumed
          mma_commit(&acc_full[ac]);
          TRACE(4, c);
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: two groups of 4 warps take alternate MMA tiles; thread = vy row m
    // of the item (TMEM lane).  Group 0 also builds F.
    const int grp = (warp - 4) >> 2;
    const int quad = warp & 3, m = quad * 32 + lane;
    const uint64_t st_pol = policy_evict_first();           // G is re-read only at the next flush
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    const bool sy_pow2 = (a.Sy & (a.Sy - 1)) == 0;
    uint32_t c = 0, item = 0;
    for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x, ++item) {
      const int2 it = a.items[w / a.n_kc];
      const int kc = (int)(w % a.n_kc);
      const int g0 = __ldg(a.col_off + it.x), mj = __ldg(a.col_off + it.x + 1) - g0;
      const bool valid = it.y + m < mj;
      const int64_t g = (int64_t)g0 + it.y + m;
      const int nvalid = min(kRgM, mj - it.y);                // rows of this item
      const int full16 = nvalid >> 4;                          // 16-row boxes stored by TMA
      if (grp == 0) {
        // F row of this vy over the flush rows, bf16 hi / lo of Fr and Fi, 32 rows at a time,
        // once every MMA of the previous item is complete (its last accumulator is full)
        if (c > 0) {
          const uint32_t cl = c - 1;
          if (m == 0) RGDBG(3, c, 1);
          mbar_wait(&acc_full[cl % kRgNAcc], (cl / kRgNAcc) & 1u);
        }
        const int vy = valid ? __ldg(a.act_vy + g) : 0;
#pragma unroll 1
        for (int r0 = 0; r0 < kr; r0 += 32) {
          uint32_t h[16], l[16], ih[16], il[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            float fr2[2], fi2[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int r = r0 + 2 * u + e;
              float2 f = make_float2(0.f, 0.f);
              if (valid && r < a.n_rows) {
                const int sy = srow[r];
                f = __ldg(a.tw + (sy_pow2 ? ((vy * sy) & (a.Sy - 1)) : (int)(((int64_t)vy * sy) % a.Sy)));
              }
              fr2[e] = f.x * a.inv_sqrt_sy;
              fi2[e] = f.y * a.inv_sqrt_sy;
            }
            split_bf16x2(fr2[0], fr2[1], h[u], l[u]);
            split_bf16x2(fi2[0], fi2[1], ih[u], il[u]);
          }
          const uint32_t col = tbase + lane_addr + kRgTmemF + r0 / 2;
          tmem_st16(col + 0 * kRgFCols, h);
          tmem_st16(col + 1 * kRgFCols, l);
          tmem_st16(col + 2 * kRgFCols, ih);
          tmem_st16(col + 3 * kRgFCols, il);
        }
        tmem_st_wait();
        tc_fence_before();
        named_sync(1, 128);
        if (tid == 128) mbar_arrive(f_full);
      }
      float2 dot = make_float2(0.f, 0.f);
      for (int t = 0; t < kt_per; ++t, ++c) {
        if ((int)(c & 1u) != grp) continue;
        const int ac = c % kRgNAcc;
        if (m == 0) RGDBG(3 + grp, c, 2);
        mbar_wait(&acc_full[ac], (c / kRgNAcc) & 1u);
        if (m == 0) RGDBG(3 + grp, c, 3);
        if (m == 0 && grp == 0) TRACE(5, c);
        tc_fence_after();
        const uint32_t d1 = tbase + lane_addr + kRgTmemAcc + ac * 2 * kRgN, d2 = d1 + kRgN;
        const int k0 = (kc * kt_per + t) * kRgNT;
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
          const uint32_t u = (c >> 1) * 2 + hh;               // half tile index within this group
          const int sw = grp * kRgNWG + (int)(u % kRgNWG);
          // D1 = [Fr Rr | Fr Ri], D2 = [Fi Rr | Fi Ri]: this half's 4 x 16 columns, one wait
          uint32_t dd[64];
          tmem_ld8_raw(d1 + 16 * hh, dd);
          tmem_ld8_raw(d1 + 16 * hh + 8, dd + 8);
          tmem_ld8_raw(d1 + kRgNT + 16 * hh, dd + 16);
          tmem_ld8_raw(d1 + kRgNT + 16 * hh + 8, dd + 24);
          tmem_ld8_raw(d2 + 16 * hh, dd + 32);
          tmem_ld8_raw(d2 + 16 * hh + 8, dd + 40);
          tmem_ld8_raw(d2 + kRgNT + 16 * hh, dd + 48);
          tmem_ld8_raw(d2 + kRgNT + 16 * hh + 8, dd + 56);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 64; ++q) asm volatile("" : "+r"(dd[q]));
          if (hh == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[ac]);
          }
          const float* ar = reinterpret_cast<const float*>(dd);        // Fr Rr
          const float* ai = ar + 16;                                    // Fr Ri
          const float* br = ar + 32;                                    // Fi Rr
          const float* bi = ar + 48;                                    // Fi Ri
          if (m == 0) RGDBG(3 + grp, c, 4 + hh);
          mbar_wait(&wg_full[sw], (u / kRgNWG) & 1u);
          if (m == 0) RGDBG(3 + grp, c, 6 + hh);
          uint8_t* sbox = rg_smem + kRgOffWG + sw * kRgStWG;
          if (valid) {
            const uint8_t* sw8 = sbox + m * 128;
            uint8_t* sg8 = sbox + kRgBoxGW + m * 128;
            float4 wv[8], ov[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {                    // 16-byte chunk q = coefficients 2q, 2q + 1
              const int off = (q ^ (m & 7)) * 16;            // SWIZZLE_128B
              wv[q] = *reinterpret_cast<const float4*>(sw8 + off);
              ov[q] = a.read_g ? *reinterpret_cast<const float4*>(sg8 + off) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            // rows in whole 16-row boxes go back through smem and a TMA store (full 128-byte
            // lines); the rows of a partial last box are stored directly
            const bool direct = m >= full16 * 16;
            float4* Gr = reinterpret_cast<float4*>(a.G + g * a.K + k0 + 16 * hh);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int n0 = 2 * q, n1 = 2 * q + 1;
              const float4 gv = make_float4(ov[q].x + (ar[n0] - bi[n0]), ov[q].y + (ai[n0] + br[n0]),
                                            ov[q].z + (ar[n1] - bi[n1]), ov[q].w + (ai[n1] + br[n1]));
              if (a.write_g) {
                if (direct) Gr[q] = gv;
                else *reinterpret_cast<float4*>(sg8 + (q ^ (m & 7)) * 16) = gv;
              }
              // dot.x = fmaf(gv.x, w.x, fmaf(-gv.y, w.y, fmaf(gv.z, w.z, fmaf(-gv.w, w.w, dot.x)))),
              // dot.y = fmaf(gv.x, w.y, fmaf(gv.y, w.x, fmaf(gv.z, w.w, fmaf(gv.w, w.z, dot.y)))): packed pairs
              dot = __ffma2_rn(make_float2(-gv.w, gv.w), make_float2(wv[q].w, wv[q].z), dot);
              dot = __ffma2_rn(make_float2(gv.z, gv.z), make_float2(wv[q].z, wv[q].w), dot);
              dot = __ffma2_rn(make_float2(-gv.y, gv.y), make_float2(wv[q].y, wv[q].x), dot);
              dot = __ffma2_rn(make_float2(gv.x, gv.x), make_float2(wv[q].x, wv[q].y), dot);
            }
          }
          if (a.write_g) fence_proxy_async_smem();           // smem G writes -> TMA store
          named_sync(4 + grp, 128);                          // the group is done with this W / G stage
          if ((tid & 127) == 0) {
            if (a.write_g && full16 > 0) {
              const int x = ((kc * kt_per + t) * 2 + hh) * 32;
              if (full16 == kRgM / 16) {
                tma_store_2d_hint(&tm.g128, x, g0 + it.y, sbox + kRgBoxGW, st_pol);
              } else {
                for (int b = 0; b < full16; ++b)
                  tma_store_2d_hint(&tm.g16, x, g0 + it.y + 16 * b, sbox + kRgBoxGW + b * 16 * 128, st_pol);
              }
              bulk_commit();
              bulk_wait_read0();                             // smem read by the store: stage reusable
            }
            mbar_arrive(&wg_empty[sw]);
          }
        }
        if (m == 0 && grp == 0) TRACE(6, c);
      }
      // combine the two groups' partial dots (fixed order: group 0 + group 1)
      float2* sd = sdot + (item & 1u) * kRgM;
      if (grp == 1) sd[m] = dot;
      if (m == 0) RGDBG(3 + grp, c, 9);
      named_sync(3, 256);
      if (m == 0) RGDBG(3 + grp, c, 10);
      if (grp == 0 && valid) {
        const float2 d1v = sd[m];
        a.opart[(int64_t)kc * a.n_act + g] = make_float2(dot.x + d1v.x, dot.y + d1v.y);
      }
    }
    if ((tid & 127) == 0) bulk_wait0();                     // the G stores have completed
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kRgTmemCols>(tbase);
}

// k-chunks of the GEMM flush: enough CTAs to fill two waves of the GPU
static int colgemm_chunks(const Plan& p) {
  int max_mj = 0;
  for (int j = 0; j < p.n_vx; ++j) max_mj = std::max(max_mj, p.col_off[j + 1] - p.col_off[j]);
  const int ctas = p.n_vx * ((max_mj + kCgM - 1) / kCgM);
  const int tiles = p.Kl / kCgNT;
  int ch = std::max(1, std::min(tiles, (2 * p.sm_count + ctas - 1) / ctas));
  while (tiles % ch) ++ch;
  return ch;
}

static int colfft_logkt(const Plan& p) {
  static const int2 knob = env_pair("WDD_COLFFT");   // (log2 k per CTA, threads) override
  int logKT = ilog2(std::max(2, std::min(32, kFftSmem / (8 * p.Sy))));
  if (knob.x >= 0) logKT = std::min(logKT, knob.x);
  while ((1 << logKT) > p.Kl || p.Kl % (1 << logKT)) --logKT;
  return logKT;
}

// k-tiles per y-FFT CTA (<= 2: with the TMA tile loads, 4 was 1.5% slower at Large and equal at
// Live) keeping >= 2 waves of CTAs
static int colfft_tpc(const Plan& p) {
  const int tiles = p.Kl >> colfft_logkt(p);
  int tpc = 1;
  // (half plane: a CTA already writes two columns per k-tile; a second k-tile per CTA then makes
  // the y-FFT re-read ~80% more than its bytes from DRAM -- Box 7.75 vs 4.03 GB, 2.13 vs 1.80 ms --
  // and loses end to end: Box -1.3%, Large -0.7%, Medium -3%, tools/experiments/exp_tpc.sh)
  while (!p.r_half && tpc < 2 && tpc * 2 <= tiles && tiles % (tpc * 2) == 0 && (int64_t)(tiles / (tpc * 2)) * p.n_vx >= 2 * p.sm_count)
    tpc *= 2;
  static const int env = [] { const char* e = std::getenv("WDD_COLFFT_TPC"); return e ? std::atoi(e) : 0; }();
  if (env > 0 && tiles % env == 0) tpc = env;
  return tpc;
}

int colfft_tiles(const Plan& p) { return (p.Kl >> colfft_logkt(p)) / colfft_tpc(p); }
// upper bound over r_half and the knobs (one k-tile per CTA): sizes the partial-readout buffer
int colfft_tiles_max(const Plan& p) { return p.Kl >> colfft_logkt(p); }

// Coefficient chunk of an FFT flush whose R staging stays in L2 (WDD_R_CHUNK_MB: the chunk's R
// budget in MB; 0 = off): each chunk is a row FFT + y-FFT pair over the same R buffer, so R is
// written and read back through L2 instead of HBM.  Returns p.Kl (no chunking) when the budget is
// off, too small for one tile unit, or the whole R fits.
int flush_chunk(const Plan& p) {
  static const int mb = [] { const char* e = std::getenv("WDD_R_CHUNK_MB"); return e ? std::atoi(e) : 0; }();
  if (mb <= 0 || !is_pow2(p.Sx) || !is_pow2(p.Sy) || p.Sx > (1 << kFftMaxLog) || p.Sy > (1 << kFftMaxLog)) return p.Kl;
  const int a = 2 << rowfft_logp(p), b = (1 << colfft_logkt(p)) * colfft_tpc(p);
  int unit = a;
  while (unit % b) unit += a;                          // lcm
  const int64_t per_k = (int64_t)p.n_vx * p.Sy * 8;
  int KR = p.Kl;
  while (KR > unit && (KR % 2 == 0) && (int64_t)KR * per_k > (int64_t)mb << 20 && (KR / 2) % unit == 0) KR /= 2;
  return KR;
}

// k-chunks of the pipelined GEMM flush: enough work items for ~4 per CTA
static int rgemm_nkc(const Plan& p) {
  const int KT = p.Kl / kRgNT;
  static const int env = [] { const char* e = std::getenv("WDD_RG_NKC"); return e ? std::atoi(e) : 0; }();
  if (env > 0 && KT % env == 0) return env;
  int nkc = 1;
  while (nkc * 2 <= KT && KT % (nkc * 2) == 0 && (int64_t)p.rg_items.size() * nkc < 4 * p.sm_count) nkc *= 2;
  return nkc;
}

bool rgemm_possible(const Plan& p, int n_rows) {
  return p.rg_ready && n_rows >= 1 && n_rows <= kRgRows && p.Kl % kRgNT == 0 && is_pow2(p.Sx) && p.Sx >= 2 &&
         p.Sx <= (1 << kFftMaxLog);
}

// Tensor maps of G and W for the pipelined GEMM flush (2-D fp32 [n_act][2K], 32-float x 128-row
// boxes, SWIZZLE_128B); built once per plan.
cudaError_t rgemm_prepare(Plan& p) {
  p.rg_ready = false;
  p.rg_items.clear();
  for (int j = 0; j < p.n_vx; ++j)
    for (int i0 = 0; i0 < p.col_off[j + 1] - p.col_off[j]; i0 += kRgM) p.rg_items.push_back(make_int2(j, i0));
  auto enc = get_encode();
  if (!enc || p.Kl % kRgNT) return cudaSuccess;   // (the FFT / DFT flushes remain)
  static_assert(sizeof(RgMaps) <= sizeof(p.rg_tmap), "tensor map storage");
  RgMaps* maps = reinterpret_cast<RgMaps*>(p.rg_tmap);
  auto make = [&](CUtensorMap* tm, void* base, uint64_t rows, uint32_t box_rows) {
    const cuuint64_t dims[2] = {(cuuint64_t)2 * p.Kl, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)p.Kl * sizeof(float2)};
    const cuuint32_t box[2] = {32u, box_rows};   // 16 complex (128 B) x box_rows
    const cuuint32_t estr[2] = {1u, 1u};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
  };
  if (!make(&maps->w16, p.d_W, p.n_act, 16) || !make(&maps->g16, p.d_G, p.n_act, 16) ||
      !make(&maps->w128, p.d_W, p.n_act, kRgM) || !make(&maps->g128, p.d_G, p.n_act, kRgM) ||
      !make(&maps->r16, p.d_R, (uint64_t)p.n_vx * p.Sy, 16) || !make(&maps->r64, p.d_R, (uint64_t)p.n_vx * p.Sy, 64))
    return cudaSuccess;
  if (cudaMalloc(&p.d_rg_items, p.rg_items.size() * sizeof(int2)) != cudaSuccess) return cudaErrorMemoryAllocation;
  cudaError_t e = cudaMemcpy(p.d_rg_items, p.rg_items.data(), p.rg_items.size() * sizeof(int2), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return e;
  e = func_attr_once((const void*)rgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kRgSmem);
  if (e != cudaSuccess) return e;
  p.rg_ready = true;
  return cudaSuccess;
}

static cudaError_t launch_rgemm(const Plan& p, const int32_t* rows, int n_rows, bool overwrite, bool o_only,
                                cudaStream_t st, int row0) {
  const int nkc = rgemm_nkc(p);
  RgArgs a{(const float2*)p.d_R, rows, n_rows, (const float2*)p.d_twy, p.Sy,
           (float)(1.0 / std::sqrt((double)p.Sy)), (const int32_t*)p.d_col_off, (const int32_t*)p.d_act_vy,
           (const int2*)p.d_rg_items, (int)p.rg_items.size(), nkc, p.d_G, p.d_opart, (int64_t)p.n_act, p.Kl,
           (!overwrite && !o_only) ? 1 : 0, o_only ? 0 : 1, row0};
  const int64_t work = (int64_t)p.rg_items.size() * nkc;
  cudaLaunchConfig_t cfg = {};
  // (WDD_RG_GRID: at most that many persistent CTAs, e.g. to leave SMs to projections running
  // beside a pipelined readout)
  static const int env_grid = [] { const char* e = std::getenv("WDD_RG_GRID"); return e ? std::atoi(e) : 0; }();
  const int max_ctas = env_grid > 0 ? std::min(env_grid, p.sm_count) : p.sm_count;
  cfg.gridDim = dim3((unsigned)std::min<int64_t>(work, max_ctas));
  cfg.blockDim = dim3(kRgThreads);
  cfg.dynamicSmemBytes = kRgSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, rgemm_kernel, a, *reinterpret_cast<const RgMaps*>(p.rg_tmap));
}

bool rowfft_applies(const Plan& p) { return is_pow2(p.Sx) && p.Sx >= 2 && p.Sx <= (1 << kFftMaxLog); }

bool flush_uses_fft(const Plan& p, int n_rows) {
  // FFT along y costs ~5 Sy log2(Sy) flops per (column, k) whatever the number of staged rows r;
  // the DFT-matrix update ~8 r m_j with m_j (active vy of the column) a fraction of Sy.
  return is_pow2(p.Sy) && p.Sy >= 2 && p.Sy <= (1 << kFftMaxLog) && n_rows >= std::max(4, ilog2(p.Sy));
}

// Which form of the rank update a flush of n_rows staged rows uses: 3 = pipelined tensor-core
// GEMM (rgemm_kernel; R in its tile layout), 2 = tensor-core DFT GEMM, 1 = FFT along y, 0 = SIMT
// DFT matrix.  WDD_FLUSH=rgemm|gemm|fft|dft overrides; allow_rg = false excludes 3 (R in fp32).
int flush_kind(const Plan& p, int n_rows, bool allow_rg) {
  static const int env = [] {
    const char* e = std::getenv("WDD_FLUSH");
    if (!e) return -1;
    return std::strcmp(e, "rgemm") == 0 ? 3 : std::strcmp(e, "gemm") == 0 ? 2 : std::strcmp(e, "fft") == 0 ? 1
         : std::strcmp(e, "dft") == 0 ? 0 : -1;
  }();
  if (allow_rg && rgemm_possible(p, n_rows) && (env == -1 || env == 3)) return 3;
  const bool gemm_ok = n_rows <= kCgRows && p.Kl % kCgNT == 0;
  int k;
  if (env == 2 || env == 3) k = gemm_ok ? 2 : (flush_uses_fft(p, n_rows) ? 1 : 0);
  else if (env == 1) k = flush_uses_fft(p, n_rows) ? 1 : (gemm_ok ? 2 : 0);
  else if (env == 0) k = 0;
  else k = flush_uses_fft(p, n_rows) ? 1 : (gemm_ok ? 2 : 0);
  // spectrum-only plans need the fused partial readout, which the SIMT DFT flush lacks (their Sy
  // is a power of two <= 2^kFftMaxLog, checked at plan creation, so the FFT always applies)
  if (k == 0 && p.o_only) k = gemm_ok ? 2 : 1;
  return k;
}

int flush_tiles(const Plan& p, int n_rows, int kind) {
  const int k = kind >= 0 ? kind : flush_kind(p, n_rows);
  return k == 3 ? rgemm_nkc(p) : k == 2 ? colgemm_chunks(p) : k == 1 ? colfft_tiles(p) : 0;
}

template <int LOGN, int LOGC>
static cudaError_t launch_colfft_t(const Plan& p, const int32_t* rows, int n_rows, bool overwrite, cudaStream_t st,
                                   bool o_only, int kbase, int KR, int logKT) {
  constexpr int PAD = FftPad<LOGC>::value;
  const size_t smem = ((size_t)p.Sy << logKT) * 8 + (size_t)(p.Sy / fft::Split<LOGN>::N2) * PAD * 8 +
                      (LOGN >= WDD_CF_TWG_MINLOG ? 0 : (size_t)p.Sy * 8) + 16;
  {
    cudaError_t e = func_attr_once((const void*)colfft_kernel<LOGN, LOGC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kFftSmem + 16384);
    if (e != cudaSuccess) return e;
  }
  const int tpc = colfft_tpc(p);
  const bool half = p.r_half;
  dim3 grid((KR >> logKT) / tpc, half ? p.n_vh : p.n_vx);
  static const int2 knob = env_pair("WDD_COLFFT");
  // L2 prefetch of the output stage's rows: Large readout 339 -> 333 us, Box 3.77 -> 3.65 ms;
  // none at Medium (-0.15%: fewer load rounds per tile), so only from Sy = 256
  static const bool pf_on = [] { const char* e = std::getenv("WDD_COLFFT_PF"); return !(e && std::atoi(e) == 0); }();
  CUtensorMap tmR;
  const bool tma = fft_tmap(&tmR, p.d_R, (uint64_t)KR * 2, (uint64_t)grid.y * p.Sy, (uint64_t)KR * 8,
                            2u << logKT, (uint32_t)(PAD ? fft::Split<LOGN>::N2 : std::min(p.Sy, 256)));
  return launch_pdl(colfft_kernel<LOGN, LOGC>, grid, dim3(knob.y > 0 ? knob.y : 256), smem, st, true, p.d_R, rows, n_rows,
                    (const float2*)p.d_twy, (const int32_t*)p.d_col_off, (const int32_t*)p.d_act_vy, p.d_G,
                    (const float2*)p.d_W, p.d_opart, (int64_t)p.n_act, logKT, p.Kl,
                    (float)(1.0 / std::sqrt((double)p.Sy)), overwrite ? 1 : 0, tpc, o_only ? 1 : 0, tmR,
                    (tma ? 1 : 0) | (pf_on && p.Sy >= 256 ? 8 : 0), kbase, KR,
                    half ? (const int2*)p.d_half_map : (const int2*)nullptr);
}

cudaError_t launch_flush(const Plan& p, const int32_t* rows, int n_rows, bool overwrite, cudaStream_t st, bool o_only,
                         int kind, int row0, int kbase, int KR) {
  if (KR <= 0) { kbase = 0; KR = p.Kl; }
  if (n_rows <= 0) return cudaSuccess;
  if (kind < 0) kind = flush_kind(p, n_rows);
  if (kind == 3) return launch_rgemm(p, rows, n_rows, overwrite, o_only, st, row0);
  if (kind == 2) {
    int max_mj = 0;
    for (int j = 0; j < p.n_vx; ++j) max_mj = std::max(max_mj, p.col_off[j + 1] - p.col_off[j]);
    {
      cudaError_t e = func_attr_once((const void*)colgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kCgSmem);
      if (e != cudaSuccess) return e;
    }
    const int ch = colgemm_chunks(p);
    dim3 grid(ch, (max_mj + kCgM - 1) / kCgM, p.n_vx);
    return launch_pdl(colgemm_kernel, grid, dim3(256), (size_t)kCgSmem, st, true, (const float2*)p.d_R, rows, n_rows,
                      (const float2*)p.d_twy, p.Sy, (float)(1.0 / std::sqrt((double)p.Sy)),
                      (const int32_t*)p.d_col_off, (const int32_t*)p.d_act_vy, p.d_G, (const float2*)p.d_W,
                      p.d_opart, (int64_t)p.n_act, p.Kl, (p.Kl / kCgNT) / ch, overwrite ? 1 : 0, o_only ? 1 : 0);
  }
  if (kind == 1) {
    const int logSy = ilog2(p.Sy);
    const int logKT = colfft_logkt(p);
    return with_log(logSy, [&](auto LN) {
      constexpr int LOGN = decltype(LN)::value;
      constexpr int SPEC = fft_spec_logc(LOGN, false);
      if constexpr (SPEC >= 0)
        if (logKT == SPEC && fft_spec_on())
          return launch_colfft_t<LOGN, SPEC>(p, rows, n_rows, overwrite, st, o_only, kbase, KR, logKT);
      return launch_colfft_t<LOGN, -1>(p, rows, n_rows, overwrite, st, o_only, kbase, KR, logKT);
    });
  }
  if (o_only) return cudaErrorNotSupported;   // unreachable: flush_kind never picks the DFT for these
  dim3 grid((unsigned)p.flush_tiles.size(), (p.Kl + 63) / 64);
  flush_kernel<<<grid, 256, 0, st>>>(p.d_R, p.d_Fy, rows, n_rows, p.d_flush_tiles, p.d_col_off, p.d_act_vy,
                                     p.d_G, p.Sy, p.Kl, overwrite ? 1 : 0);
  return cudaGetLastError();
}

// =====================================================================================
// a4 + a5 + a6 fused for scans up to 256 x 256: the whole 2-D scan DFT of a group of coefficients
// in one thread-block cluster, so the row-DFT staging R never goes through HBM (the row FFT + y-FFT
// pair moves 16 n_vx K / Sx bytes per frame through R otherwise).
//   CTA r of the cluster owns scan rows [r RB, (r+1) RB) for the row pass: the 2 NP coefficients
//   k0 .. k0 + 2NP - 1 of every position, packed as NP complex sequences (z = C_k + i C_k+1), are
//   read from the coefficient store (pending positions only; the rest are zeros), FFT'd along x
//   (fft_seq), and kept in shared memory.  After a cluster barrier, CTA r takes the active columns
//   [r n_vx / CS, (r+1) n_vx / CS): it gathers each column's row transforms from all CTAs of the
//   cluster through distributed shared memory (X_k = (Z[v] + conj Z[-v]) / 2, X_k+1 = (Z[v] -
//   conj Z[-v]) / 2i, the real-pair split of rowfft_kernel), FFTs them along y, updates G (+)= X
//   for the column's active vy and writes the Wiener readout partial of its 2 NP coefficients,
//   opart[group][v] = sum_k G[v][k] K_v[k].  Exact like the two-kernel form (same
//   transforms, same order of the additions in G; the partial readouts are summed over groups).
// =====================================================================================
template <int LX, int LY, int CS, int NP>
__global__ void __launch_bounds__(256) fft2_kernel(const float* __restrict__ C, const int32_t* __restrict__ rows,
                                                   const uint32_t* __restrict__ masks, int n_rows, int mask_words,
                                                   const float2* __restrict__ twx, const float2* __restrict__ twy,
                                                   const int32_t* __restrict__ col_vx,
                                                   const int32_t* __restrict__ col_off,
                                                   const int32_t* __restrict__ act_vy, int n_vx,
                                                   float2* __restrict__ G, const float2* __restrict__ W,
                                                   float2* __restrict__ opart, int64_t n_act, int K, float sx_scale,
                                                   float sy_scale, int overwrite, int o_only, int late_trigger) {
  constexpr int SX = 1 << LX, SY = 1 << LY;
  constexpr int LCS = CS == 8 ? 3 : CS == 4 ? 2 : CS == 2 ? 1 : 0;
  constexpr int RB = SY / CS, LRB = LY - LCS;
  constexpr int LCNT = LRB + (NP == 2 ? 1 : 0), CNT = 1 << LCNT;    // row-pass sequences (row, pair)
  constexpr int CB = 8;                                               // columns per column-pass batch
  constexpr int LCNT2 = 3 + (NP == 2 ? 1 : 0) + 1, CNT2 = 1 << LCNT2; // (column, pair, k / k+1)
  static_assert(CNT2 == CB * NP * 2, "column batch");
  extern __shared__ __align__(16) float2 fsm[];
  float2* xr = fsm;                        // [SX][CNT]
  float2* xc = xr + SX * CNT;              // [SY][CNT2]
  float2* stx = xc + SY * CNT2;            // [SX]
  float2* sty = stx + SX;                  // [SY]
  __shared__ int sli[SY];                  // row -> index in the flush's row list, or -1
  __shared__ int2 scs[CB];                 // batch column: (slot of v, slot of -v)
  __shared__ int sgo[CB + 1];              // batch column: first accumulator row, then a prefix end
  cg::cluster_group cluster = cg::this_cluster();
  const int r = (int)cluster.block_rank();
  const int k0 = blockIdx.y * 2 * NP;
  const int tid = threadIdx.x;
  if (!late_trigger) pdl_trigger();
  for (int i = tid; i < SX; i += blockDim.x) stx[i] = __ldg(twx + i);
  for (int i = tid; i < SY; i += blockDim.x) { sty[i] = __ldg(twy + i); sli[i] = -1; }
  pdl_wait();   // C of the projections (and the uploaded row list / masks)
  __syncthreads();
  for (int i = tid; i < n_rows; i += blockDim.x) sli[__ldg(rows + i)] = i;
  __syncthreads();
  // ---- row pass: load this CTA's rows (sequence index fastest: conflict-free smem stores)
  for (int e = tid; e < RB * SX; e += blockDim.x) {
    const int i = e % RB, sx = e / RB, sy = r * RB + i;
    const int li = sli[sy];
    const bool ok = li >= 0 && ((__ldg(masks + (int64_t)li * mask_words + (sx >> 5)) >> (sx & 31)) & 1u);
    const float* src = C + ((int64_t)sy * SX + sx) * K + k0;
    if constexpr (NP == 2) {
      const float4 v = ok ? __ldg(reinterpret_cast<const float4*>(src)) : make_float4(0.f, 0.f, 0.f, 0.f);
      xr[sx * CNT + 2 * i] = make_float2(v.x, v.y);
      xr[sx * CNT + 2 * i + 1] = make_float2(v.z, v.w);
    } else {
      const float2 v = ok ? __ldg(reinterpret_cast<const float2*>(src)) : make_float2(0.f, 0.f);
      xr[sx * CNT + i] = v;
    }
  }
  __syncthreads();
  if (late_trigger) pdl_trigger();   // every read of C by this CTA is complete
  fft::fft_seq<LX>(xr, stx, LCNT);
  cluster.sync();                    // every CTA's row transforms are complete
  // ---- column pass over this CTA's share of the active columns
  const int jlo = (int)((int64_t)r * n_vx / CS), jhi = (int)((int64_t)(r + 1) * n_vx / CS);
  const float hs = 0.5f * sx_scale;
  for (int jb0 = jlo; jb0 < jhi; jb0 += CB) {
    const int nb = min(CB, jhi - jb0);
    if (tid < CB) {
      if (tid < nb) {
        const int v = __ldg(col_vx + jb0 + tid);
        scs[tid] = make_int2(fft::fslot<LX>(v), fft::fslot<LX>((SX - v) & (SX - 1)));
      }
    }
    if (tid == 0) {
      sgo[0] = 0;
      for (int b = 0; b < nb; ++b) sgo[b + 1] = sgo[b] + (__ldg(col_off + jb0 + b + 1) - __ldg(col_off + jb0 + b));
    }
    __syncthreads();
    // gather X_k, X_k+1 of the batch's columns for every scan row from the owning CTA (DSMEM)
    for (int e = tid; e < SY * CB * NP; e += blockDim.x) {
      const int q = e % (CB * NP), sy = e / (CB * NP);
      const int jb = q / NP, p = q - jb * NP;
      float2 x0 = make_float2(0.f, 0.f), x1 = x0;
      if (jb < nb) {
        const float2* src = cluster.map_shared_rank(xr, sy / RB);
        const int c = (sy % RB) * NP + p;
        const int2 sl = scs[jb];
        const float2 z = src[(sl.x << LCNT) + c], zm = src[(sl.y << LCNT) + c];
        x0 = make_float2((z.x + zm.x) * hs, (z.y - zm.y) * hs);
        x1 = make_float2((z.y + zm.y) * hs, (zm.x - z.x) * hs);
      }
      xc[sy * CNT2 + 2 * q] = x0;
      xc[sy * CNT2 + 2 * q + 1] = x1;
    }
    __syncthreads();
    fft::fft_seq<LY>(xc, sty, LCNT2);
    // output: thread = one active (vy, column) of the batch, all 2 NP coefficients: G (+)= X, and
    // the readout partial of these coefficients
    const int tot = sgo[nb];
    for (int f = tid; f < tot; f += blockDim.x) {
      int jb = 0;
      while (jb + 1 < nb && f >= sgo[jb + 1]) ++jb;
      const int64_t g = __ldg(col_off + jb0 + jb) + (f - sgo[jb]);
      const int slot = fft::fslot<LY>(__ldg(act_vy + g));
      const float2* xs = xc + slot * CNT2 + jb * 2 * NP;
      float2* Gr = G + g * K + k0;
      const float2* Wr = W + g * K + k0;
      float2 d = make_float2(0.f, 0.f);
#pragma unroll
      for (int e2 = 0; e2 < 2 * NP; ++e2) {
        const float2 w = __ldg(Wr + e2);
        const float2 o = (overwrite || o_only) ? make_float2(0.f, 0.f) : Gr[e2];
        const float2 z = xs[e2];
        const float2 gn = make_float2(fmaf(z.x, sy_scale, o.x), fmaf(z.y, sy_scale, o.y));
        if (!o_only) Gr[e2] = gn;
        d.x = fmaf(gn.x, w.x, fmaf(-gn.y, w.y, d.x));
        d.y = fmaf(gn.x, w.y, fmaf(gn.y, w.x, d.y));
      }
      opart[(int64_t)blockIdx.y * n_act + g] = d;
    }
    __syncthreads();                 // xc and the batch tables reused
  }
  cluster.sync();                    // no CTA leaves while others may still read its row transforms
}

// Fused 2-D flush geometry: square power-of-two scans from 32 to 256; two coefficient pairs per
// cluster up to 128, one at 256; cluster size from 64 KB of row transforms per CTA.  Opt-in
// (WDD_FUSED=1): measured slower than the two-kernel flush -- with 2-4 coefficients per cluster
// (what fits the cluster's shared memory) every position is an 8-16 byte read at a K * 4-byte
// stride (Medium flush 78 vs 38 us, Large 1.37 vs 0.32 ms; profiles/README.md).
bool fused_possible(const Plan& p) {
  static const bool on = [] { const char* e = std::getenv("WDD_FUSED"); return e && std::atoi(e) == 1; }();
  return on && p.Sx == p.Sy && is_pow2(p.Sx) && p.Sx >= 32 && p.Sx <= 256 && p.Kl % 4 == 0;
}

static int fused_np(const Plan& p) { return p.Sx <= 128 ? 2 : 1; }

int fused_tiles(const Plan& p) { return p.Kl / (2 * fused_np(p)); }

template <int LX, int CS, int NP>
static cudaError_t launch_fft2_t(const Plan& p, const int32_t* rows, const uint32_t* masks, int n_rows, bool overwrite,
                                 bool o_only, cudaStream_t st) {
  constexpr int SX = 1 << LX, RB = SX / CS;
  constexpr int CNT = RB * NP, CNT2 = 8 * NP * 2;
  constexpr size_t smem = (size_t)(SX * CNT + SX * CNT2 + 2 * SX) * sizeof(float2);
  auto kern = fft2_kernel<LX, LX, CS, NP>;
  cudaError_t e = func_attr_once((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const bool pdl = !project_is_lean(p);   // (as the row FFT: see launch_rowdft)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS, p.Kl / (2 * NP));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, (const float*)p.d_Call, rows, masks, n_rows, p.mask_words,
                            (const float2*)p.d_twx, (const float2*)p.d_twy, (const int32_t*)p.d_col_vx,
                            (const int32_t*)p.d_col_off, (const int32_t*)p.d_act_vy, p.n_vx, p.d_G,
                            (const float2*)p.d_W, p.d_opart, (int64_t)p.n_act, p.Kl,
                            (float)(1.0 / std::sqrt((double)p.Sx)), (float)(1.0 / std::sqrt((double)p.Sy)),
                            overwrite ? 1 : 0, o_only ? 1 : 0, pdl ? 1 : 0);
}

cudaError_t launch_fft2(const Plan& p, const int32_t* rows, const uint32_t* masks, int n_rows, bool overwrite,
                        bool o_only, cudaStream_t st) {
  switch (p.Sx) {
    case 32: return launch_fft2_t<5, 1, 2>(p, rows, masks, n_rows, overwrite, o_only, st);
    case 64: return launch_fft2_t<6, 1, 2>(p, rows, masks, n_rows, overwrite, o_only, st);
    case 128: return launch_fft2_t<7, 4, 2>(p, rows, masks, n_rows, overwrite, o_only, st);
    case 256: return launch_fft2_t<8, 8, 1>(p, rows, masks, n_rows, overwrite, o_only, st);
    default: return cudaErrorInvalidValue;
  }
}

// =====================================================================================
// Readout (a6): o_v = sum_k G[v][k] W[v][k], one warp per active v
// =====================================================================================
__global__ void __launch_bounds__(256) readout_kernel(const float2* __restrict__ G, const float2* __restrict__ W,
                                                      int64_t n_act, int K, float2* __restrict__ o) {
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= n_act) return;
  const float4* Gr = reinterpret_cast<const float4*>(G + g * K);
  const float4* Wr = reinterpret_cast<const float4*>(W + g * K);
  float re = 0.f, im = 0.f;
#pragma unroll 4
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
  if (lane == 0) o[g] = make_float2(re, im);
}

__global__ void fence_kernel() {}

cudaError_t launch_fence(cudaStream_t st) {
  fence_kernel<<<1, 32, 0, st>>>();
  return cudaGetLastError();
}

cudaError_t launch_readout(const Plan& p, const float2* G, float2* o, cudaStream_t st) {
  const int64_t threads = p.n_act * 32;
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  readout_kernel<<<blocks, 256, 0, st>>>(G, p.d_W, p.n_act, p.Kl, o);
  return cudaGetLastError();
}

// o_v = sum over the `tiles` partial sums (fixed order), scattered to the dense spectrum
__device__ __forceinline__ float2 sum_tiles(const float2* __restrict__ op, int tiles, int64_t n_act, int64_t g) {
  float2 acc = make_float2(0.f, 0.f);
  for (int t0 = 0; t0 < tiles; t0 += 16) {     // sixteen independent loads in flight, summed in order
    float2 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u)
      v[u] = t0 + u < tiles ? __ldg(op + (int64_t)(t0 + u) * n_act + g) : make_float2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      acc.x += v[u].x;
      acc.y += v[u].y;
    }
  }
  return acc;
}

// Spectrum-only accumulator: o[g] += sum over the flush's partial readouts (fixed order).
__global__ void oacc_kernel(const float2* __restrict__ op, int tiles, int64_t n_act, float2* __restrict__ o) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_act) return;
  const float2 d = sum_tiles(op, tiles, n_act, g);
  const float2 v = o[g];
  o[g] = make_float2(v.x + d.x, v.y + d.y);
}

cudaError_t launch_oacc(const Plan& p, int tiles, cudaStream_t st) {
  oacc_kernel<<<(unsigned)((p.n_act + 255) / 256), 256, 0, st>>>(p.d_opart, tiles, p.n_act, p.d_oacc);
  return cudaGetLastError();
}

// o[g] = sum over the partial readouts (fixed order): the rank's spectrum before the NCCL combine
__global__ void otiles_kernel(const float2* __restrict__ op, int tiles, int64_t n_act, float2* __restrict__ o) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  pdl_trigger();
  pdl_wait();   // partial readouts of the preceding flush / readout kernel
  if (g < n_act) o[g] = sum_tiles(op, tiles, n_act, g);
}

cudaError_t launch_otiles(const Plan& p, const float2* op, int tiles, float2* o, cudaStream_t st) {
  return launch_pdl(otiles_kernel, dim3((unsigned)((p.n_act + 255) / 256)), dim3(256), 0, st, true, op, tiles,
                    (int64_t)p.n_act, o);
}

__global__ void scatter_kernel(const float2* __restrict__ op, int tiles, const int32_t* __restrict__ vpos,
                               int64_t n_act, float2* __restrict__ spec) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  pdl_trigger();
  pdl_wait();   // partial readouts of the preceding flush / readout kernel
  if (g < n_act) spec[__ldg(vpos + g)] = sum_tiles(op, tiles, n_act, g);
}

// =====================================================================================
// Finalize (a8): out = conj(IDFT2(o)) / sqrt(S) [/ sqrt(o_0)]; cuFFT for scans that are not
// powers of two, else the two-pass shared-memory FFT below.
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

// a8 on power-of-two scans without cuFFT.  O = conj(IDFT2_unitary(o)) = DFT2(conj o) / sqrt(S),
// as two passes of the shared-memory FFT: rows (A[vy][x] = sum_vx conj o[vy][vx] W_Sx^{vx x})
// into a scratch image, then columns with the unitary scale and the optional 1/sqrt(o_0).
template <int LOGN>
__global__ void __launch_bounds__(256) img_rows_kernel(const float2* __restrict__ spec, const float2* __restrict__ tw,
                                                       float2* __restrict__ A, int logc) {
  constexpr int N = 1 << LOGN;
  extern __shared__ __align__(16) float2 fsm[];
  float2* x = fsm;                 // [N][cnt]: x[vx * cnt + c] = conj o[vy0 + c][vx]
  float2* stw = fsm + (N << logc);
  const int vy0 = blockIdx.x << logc;
  pdl_trigger();
  for (int i = threadIdx.x; i < N; i += blockDim.x) stw[i] = __ldg(tw + i);
  pdl_wait();   // the spectrum of the preceding scatter kernel
  for (int e = threadIdx.x; e < (N << logc); e += blockDim.x) {
    const int c = e >> LOGN, vx = e & (N - 1);
    const float2 v = __ldg(spec + (int64_t)(vy0 + c) * N + vx);
    x[(vx << logc) + c] = make_float2(v.x, -v.y);
  }
  __syncthreads();
  fft::fft_seq<LOGN>(x, stw, logc);
  for (int e = threadIdx.x; e < (N << logc); e += blockDim.x) {
    const int c = e >> LOGN, xx = e & (N - 1);
    A[(int64_t)(vy0 + c) * N + xx] = x[(fft::fslot<LOGN>(xx) << logc) + c];
  }
}

__device__ __forceinline__ float2 inv_principal_sqrt(float2 o0) {
  // 1 / sqrt(o_0), principal branch (eq:extract; R13); 1 if o_0 == 0
  const double a = o0.x, b = o0.y, r = hypot(a, b);
  if (!(r > 0)) return make_float2(1.f, 0.f);
  const double s = sqrt(0.5 * (r + fabs(a)));
  double wr, wi;
  if (a >= 0) { wr = s; wi = b / (2 * s); } else { wr = fabs(b) / (2 * s); wi = copysign(s, b); }
  const double d = wr * wr + wi * wi;
  return make_float2((float)(wr / d), (float)(-wi / d));
}

template <int LOGN>
__global__ void __launch_bounds__(256) img_cols_kernel(const float2* __restrict__ A, const float2* __restrict__ tw,
                                                       float2* __restrict__ out, int Sx, int logc, float scale,
                                                       const float2* __restrict__ spec, int normalize) {
  constexpr int N = 1 << LOGN;     // Sy
  extern __shared__ __align__(16) float2 fsm[];
  const int cnt = 1 << logc;
  float2* x = fsm;                 // [N][cnt]: x[vy * cnt + c] = A[vy][x0 + c]
  float2* stw = fsm + (N << logc);
  const int x0 = blockIdx.x << logc;
  pdl_trigger();
  for (int i = threadIdx.x; i < N; i += blockDim.x) stw[i] = __ldg(tw + i);
  pdl_wait();   // row pass of the preceding kernel
  for (int e = threadIdx.x; e < (N << logc); e += blockDim.x) {
    const int vy = e >> logc, c = e & (cnt - 1);
    x[e] = __ldg(A + (int64_t)vy * Sx + x0 + c);
  }
  __syncthreads();
  fft::fft_seq<LOGN>(x, stw, logc);
  float2 f = make_float2(scale, 0.f);
  if (normalize) {
    const float2 w = inv_principal_sqrt(__ldg(spec));   // o_0 (v = 0 is image position 0)
    f = make_float2(w.x * scale, w.y * scale);
  }
  for (int e = threadIdx.x; e < (N << logc); e += blockDim.x) {
    const int y = e >> logc, c = e & (cnt - 1);
    out[(int64_t)y * Sx + x0 + c] = cmul(x[(fft::fslot<LOGN>(y) << logc) + c], f);
  }
}

// a8 in one launch for images up to 256 x 256: a cluster of CS CTAs, CTA r owns RB = Sy/CS rows
// for the row pass and CB = Sx/CS columns for the column pass; the transposition between the two
// passes goes through distributed shared memory (no global round trip, one launch).  The spectrum
// rows are gathered straight from the partial readouts (o_v = their fixed-order tile sum, zero for
// inactive v through gidx), so no scatter pass runs before it.
template <int LX, int LY, int CS>
__global__ void __launch_bounds__(512) img_fused_kernel(const float2* __restrict__ op, int tiles, int64_t n_act,
                                                        const int32_t* __restrict__ gidx, int g_dc,
                                                        const float2* __restrict__ twx, const float2* __restrict__ twy,
                                                        float2* __restrict__ out, float scale, int normalize) {
  constexpr int SX = 1 << LX, SY = 1 << LY, RB = SY / CS, CB = SX / CS;
  constexpr int LRB = LY - (CS == 16 ? 4 : CS == 8 ? 3 : CS == 4 ? 2 : CS == 2 ? 1 : 0);
  constexpr int LCB = LX - (CS == 16 ? 4 : CS == 8 ? 3 : CS == 4 ? 2 : CS == 2 ? 1 : 0);
  extern __shared__ __align__(16) float2 fsm[];
  float2* xr = fsm;                         // [SX][RB]  row pass (frequency vx at slot fslot<LX>)
  float2* xc = xr + SX * RB;                // [SY][CB]  column pass
  float2* stx = xc + SY * CB;               // [SX]
  float2* sty = stx + SX;                   // [SY]
  cg::cluster_group cluster = cg::this_cluster();
  const int r = (int)cluster.block_rank();
  pdl_trigger();
  for (int i = threadIdx.x; i < SX; i += blockDim.x) stx[i] = __ldg(twx + i);
  for (int i = threadIdx.x; i < SY; i += blockDim.x) sty[i] = __ldg(twy + i);
  pdl_wait();   // the partial readouts of the preceding flush / readout kernel
  const int vy0 = r * RB;
  // up to 4 positions per thread per round: their accumulator rows load together, then their tile
  // sums (two dependent load rounds per 4 positions instead of per position)
  for (int e0 = threadIdx.x; e0 < SX * RB; e0 += 4 * blockDim.x) {
    int g[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * (int)blockDim.x;
      g[u] = e < SX * RB ? __ldg(gidx + (int64_t)(vy0 + (e >> LX)) * SX + (e & (SX - 1))) : -1;
    }
    float2 acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] = make_float2(0.f, 0.f);
    for (int t0 = 0; t0 < tiles; t0 += 8) {          // (the fixed tile order of sum_tiles)
      float2 v[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < 8; ++q)
          v[u][q] = g[u] >= 0 && t0 + q < tiles ? __ldg(op + (int64_t)(t0 + q) * n_act + g[u]) : make_float2(0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          acc[u].x += v[u][q].x;
          acc[u].y += v[u][q].y;
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * (int)blockDim.x;
      if (e < SX * RB)
        xr[((e & (SX - 1)) << LRB) + (e >> LX)] = make_float2(acc[u].x, -acc[u].y);   // conj(o): O = DFT2(conj o) / sqrt(S)
    }
  }
  __syncthreads();
  fft::fft_seq<LX>(xr, stx, LRB);
  cluster.sync();                           // every CTA's row pass is complete
  const int x0 = r * CB;
  for (int e = threadIdx.x; e < SY * CB; e += blockDim.x) {
    const int vy = e >> LCB, cc = e & (CB - 1);
    const float2* src = cluster.map_shared_rank(xr, vy / RB);
    xc[e] = src[(fft::fslot<LX>(x0 + cc) << LRB) + (vy % RB)];
  }
  cluster.sync();                           // remote reads done before any CTA exits
  fft::fft_seq<LY>(xc, sty, LCB);
  float2 f = make_float2(scale, 0.f);
  if (normalize) {
    const float2 w = inv_principal_sqrt(sum_tiles(op, tiles, n_act, g_dc));
    f = make_float2(w.x * scale, w.y * scale);
  }
  for (int e = threadIdx.x; e < SY * CB; e += blockDim.x) {
    const int y = e >> LCB, cc = e & (CB - 1);
    out[(int64_t)y * SX + x0 + cc] = cmul(xc[(fft::fslot<LY>(y) << LCB) + cc], f);
  }
}

template <int LX, int LY, int CSMAX>
static cudaError_t launch_img_fused(const Plan& p, const float2* op, int tiles, float2* out, cudaStream_t st) {
  constexpr int CS0 = (LX >= 4 && LY >= 4) ? 16 : 1 << (LX < LY ? LX : LY);
  constexpr int CS = CS0 < CSMAX ? CS0 : CSMAX;
  constexpr int SX = 1 << LX, SY = 1 << LY;
  constexpr size_t smem = (size_t)(SX * (SY / CS) + SY * (SX / CS) + SX + SY) * 8;
  {
    cudaError_t e = func_attr_once((const void*)img_fused_kernel<LX, LY, CS>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && CS > 8)
      e = func_attr_once((const void*)img_fused_kernel<LX, LY, CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  // 512 threads: Medium finalize 12.6 -> 10.6 us, +0.75% end to end against 256 (1024: no better)
  static const int nt = [] { const char* e = std::getenv("WDD_IMG_NT"); return e ? std::atoi(e) : 512; }();
  cfg.gridDim = dim3(CS);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, img_fused_kernel<LX, LY, CS>, op, tiles, (int64_t)p.n_act,
                            (const int32_t*)p.d_gidx, (int)p.g_dc, (const float2*)p.d_twx,
                            (const float2*)p.d_twy, out, (float)(1.0 / std::sqrt((double)p.S)), p.normalize);
}

static cudaError_t launch_img_fused_dispatch(const Plan& p, const float2* op, int tiles, float2* out,
                                             cudaStream_t st) {
  return with_log(ilog2(p.Sx), [&](auto LNX) {
    constexpr int LX = decltype(LNX)::value;
    return with_log(ilog2(p.Sy), [&](auto LNY) -> cudaError_t {
      constexpr int LY = decltype(LNY)::value;
      // cluster size: 16 CTAs (non-portable) by default; WDD_IMG_CS=8 for the portable maximum
      static const int cs = [] { const char* e = std::getenv("WDD_IMG_CS"); return e ? std::atoi(e) : 16; }();
      if constexpr (LX <= 8 && LY <= 8)
        return cs == 8 ? launch_img_fused<LX, LY, 8>(p, op, tiles, out, st)
                       : launch_img_fused<LX, LY, 16>(p, op, tiles, out, st);
      else return cudaErrorInvalidValue;
    });
  });
}

bool finalize_uses_fft(const Plan& p) {
  return is_pow2(p.Sx) && is_pow2(p.Sy) && p.Sx >= 2 && p.Sy >= 2 && p.Sx <= (1 << kFftMaxLog) &&
         p.Sy <= (1 << kFftMaxLog);
}

// Images up to 128 x 128 take the one-launch cluster kernel, which gathers o from the partial
// readouts itself.  Otherwise the partial readouts are first summed (fixed order) and scattered
// to image order (one coalesced pass over the tiles; inactive positions of d_spec stay zero from
// plan creation), then larger power-of-two images take the row and column passes (>= 128 CTAs
// each) and other sizes (or WDD_IMG=cufft) cuFFT.
cudaError_t launch_finalize(const Plan& p, const float2* op, int tiles, float2* out, cudaStream_t st) {
  static const int img_mode = [] {
    const char* e = std::getenv("WDD_IMG");
    return !e ? 0 : std::strcmp(e, "cufft") == 0 ? 1 : std::strcmp(e, "unfused") == 0 ? 2 : std::strcmp(e, "fused") == 0 ? 3 : 0;
  }();
  const bool own = finalize_uses_fft(p) && img_mode != 1;
  const int fused_max = img_mode == 3 ? 256 : img_mode == 2 ? 0 : 128;
  if (own && p.Sx <= fused_max && p.Sy <= fused_max) return launch_img_fused_dispatch(p, op, tiles, out, st);
  cudaError_t e = launch_spectrum(p, op, tiles, p.d_spec, st);
  if (e != cudaSuccess) return e;
  return launch_image(p, p.d_spec, out, st);
}

// spec[v] = sum of the partial readouts of active v (fixed order); inactive positions of spec are
// not written (the plan's own spectrum buffer keeps them zero from creation)
cudaError_t launch_spectrum(const Plan& p, const float2* op, int tiles, float2* spec, cudaStream_t st) {
  return launch_pdl(scatter_kernel, dim3((unsigned)((p.n_act + 255) / 256)), dim3(256), 0, st, true, op, tiles,
                    (const int32_t*)p.d_vpos, (int64_t)p.n_act, spec);
}

// O = conj(IDFT2_unitary(spec)) [/ sqrt(spec[0])] from a dense Sy x Sx spectrum (a8)
cudaError_t launch_image(const Plan& p, const float2* spec, float2* out, cudaStream_t st) {
  const int64_t S = p.S;
  static const int img_mode = [] {
    const char* e = std::getenv("WDD_IMG");
    return !e ? 0 : std::strcmp(e, "cufft") == 0 ? 1 : 0;
  }();
  const bool own = finalize_uses_fft(p) && img_mode != 1;
  if (own) {
    const int lx = ilog2(p.Sx), ly = ilog2(p.Sy);
    // 2^lr rows per CTA: enough sequences for the threads of the FFT passes, >= 128 CTAs if possible
    const int lr = std::max(0, std::min(ilog2(std::max(1, 4096 / p.Sx)), ly - 7));
    cudaError_t e = with_log(lx, [&](auto LN) {
      constexpr int L = decltype(LN)::value;
      const size_t smem = ((size_t)p.Sx << lr) * 8 + (size_t)p.Sx * 8 + 16;
      // threads: the larger FFT pass has N1 << lr independent register DFTs
      const int nt = std::max(32, std::min(256, fft::Split<L>::N1 << lr));
      return launch_pdl(img_rows_kernel<L>, dim3(p.Sy >> lr), dim3(nt), smem, st, true, spec,
                        (const float2*)p.d_twx, p.d_img_tmp, lr);
    });
    if (e != cudaSuccess) return e;
    const int lc = std::max(0, std::min(ilog2(std::max(1, 4096 / p.Sy)), lx - 7));
    return with_log(ly, [&](auto LN) {
      constexpr int L = decltype(LN)::value;
      const size_t smem = ((size_t)p.Sy << lc) * 8 + (size_t)p.Sy * 8 + 16;
      const int nt = std::max(32, std::min(256, fft::Split<L>::N1 << lc));
      return launch_pdl(img_cols_kernel<L>, dim3(p.Sx >> lc), dim3(nt), smem, st, true, (const float2*)p.d_img_tmp,
                        (const float2*)p.d_twy, out, p.Sx, lc, (float)(1.0 / std::sqrt((double)S)),
                        spec, p.normalize);
    });
  }
  if (cufftSetStream(p.fft, st) != CUFFT_SUCCESS) return cudaErrorUnknown;
  if (cufftExecC2C(p.fft, reinterpret_cast<cufftComplex*>(const_cast<float2*>(spec)),
                   reinterpret_cast<cufftComplex*>(out), CUFFT_INVERSE) != CUFFT_SUCCESS)
    return cudaErrorUnknown;
  conj_scale_kernel<<<(unsigned)((S + 255) / 256), 256, 0, st>>>(out, S, 1.0 / std::sqrt((double)S), spec,
                                                                 p.normalize);
  return cudaGetLastError();
}

#ifdef WDD_RG_DEBUG
}  // namespace wdd
extern "C" int wdd_rg_debug(unsigned* host /* 148 x 8 */) {
  cudaStream_t s;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return -1;
  void* d = nullptr;
  cudaGetSymbolAddress(&d, wdd::g_rgdbg);
  cudaMemcpyAsync(host, d, sizeof(unsigned) * 148 * 8, cudaMemcpyDeviceToHost, s);
  for (int i = 0; i < 2000; ++i) {
    if (cudaStreamQuery(s) == cudaSuccess) return 0;
    struct timespec ts = {0, 1000000};
    nanosleep(&ts, nullptr);
  }
  return -2;
}
namespace wdd {
#endif
}  // namespace wdd
