// internal.h -- plan state and kernel launchers shared by plan.cpp and kernels.cu.
#pragma once
#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/wdd.h"

namespace wdd {

struct FullWddWork;   // fullwdd.cu: scratch + cuFFT plans of wdd_full_wdd, kept across calls

enum ProfSlot { kSlotProject = 0, kSlotRowDft = 1, kSlotFlush = 2, kSlotReadout = 3, kSlotFinalize = 4, kNumSlots = 5 };

constexpr int kMaxShards = 8;        // coefficient shards (ranks) a projection can write to

// Destinations of the projection's coefficient rows: a = n_x row of H(I) (k = a*L + b) goes to
// shard o with alo[o] <= a < alo[o+1], at C[o] + position * K[o] + (a - alo[o]) * L.
struct ProjDst {
  int n = 1;
  float* C[kMaxShards] = {};
  int K[kMaxShards] = {};
  int alo[kMaxShards + 1] = {};
};

struct Plan {
  // geometry
  int Sy = 0, Sx = 0, Q = 0, L = 0, K = 0, dtype = 0, normalize = 0, device = 0, combine = 0;
  // coefficient sharding (opts.k_shards): this plan owns rows a in [a_split[shard],
  // a_split[shard+1]) of every frame's H(I), i.e. the Kl = (a1 - a0) * L coefficients from k0; its
  // coefficient store, R, G, bank and readout cover only those.  Unsharded: nshard = 1, Kl = K.
  int nshard = 1, shard = 0, Kl = 0, k0 = 0;
  std::vector<int> a_split;            // nshard + 1
  float* peer_base[kMaxShards] = {};   // each shard's store allocation (2 x S x Kl_o), this process's view
  bool peers_ipc[kMaxShards] = {};     // opened with cudaIpcOpenMemHandle (closed at destroy)
  bool peers_ready = false;
  int store_par = 0;                   // which of the two stores is current (flips at every swap)
  float* d_Cbase = nullptr;            // the allocation holding both coefficient stores
  int64_t S = 0, n_act = 0;
  int n_vx = 0;
  double step = 0, lambda = 0, alpha = 0, defocus = 0, eps = 0, dq = 0, qa = 0, R = 0, sigma = 0;
  double b_scale = 1.0;  // power-of-two prescale of the fp16 basis operand (2^s)
  double sc1 = 1.0, sc2 = 1.0;  // projection epilogue scales: 2^(eT-s), 2^(-s-eT)
  int sm_count = 148;
  mutable int last_proj_grid = 0;   // CTAs of the latest projection launch (launch_rowdft's PDL choice)
  int ingest_spread = 0;              // 1: every projection launch over all SMs (latency grid)
  int ingest_overlap = 0;             // 1: frames are complete before the previous library call on the stream
                                      // (projection reads them before its predecessor grid completes)
  unsigned* d_err = nullptr;          // device error flags (f32 frame range), sticky until wdd_check

  // host tables
  std::vector<double> basis;          // Q*L, Psi[m][n]
  std::vector<int32_t> active_v;      // n_act, accumulator order (vx-major, vy ascending)
  std::vector<int32_t> col_vx;        // n_vx
  std::vector<int32_t> col_off;       // n_vx + 1
  std::vector<int32_t> act_vy;        // n_act
  std::vector<int2> flush_tiles;      // (column j, first row i0) of 32-row tiles
  std::vector<uint64_t> seen;         // S bits
  std::vector<uint8_t> row_dirty;     // Sy: row has coefficients in d_Call not yet flushed into G
  std::vector<uint32_t> pending;      // Sy x mask_words bits: position ingested, not yet row-transformed
  std::vector<uint8_t> row_staged;    // Sy: R holds this row's DFT, not yet folded into G
  int mask_words = 1;                 // ceil(Sx / 32)
  int64_t frames_ingested = 0;
  int64_t frames_enqueued = 0;        // frames this plan projected since the reset (its own ingest calls)
  int64_t proj_rem_after = -1;        // scan positions still to come after the projection being launched (-1: unknown)

  // device buffers
  void* d_Bpack = nullptr;            // fp16 [Psi_hi | Psi_lo] B operand, smem image
  float* d_psi = nullptr;             // Q*L f32
  float2* d_Fx = nullptr;             // n_vx * Sx
  float2* d_Fy = nullptr;             // Sy * Sy
  float2* d_twx = nullptr;            // Sx FFT twiddles exp(-2 pi i m / Sx), m < Sx
  float2* d_twy = nullptr;            // Sy FFT twiddles exp(-2 pi i m / Sy), m < Sy
  int32_t* d_col_vx = nullptr;        // n_vx active vx, ascending
  // Hermitian half plane (the active set is symmetric under v -> -v, power-of-two Sx): the row
  // FFT writes only the n_vh primary columns (vx <= Sx/2) to R, the y-FFT writes each primary
  // column's mirror from the same transform (colfft_kernel); r_half is set per flush (FFT flushes)
  int n_vh = 0;                       // 0: not available
  int32_t* d_col_vx_half = nullptr;   // n_vh primary vx
  bool half_identity = false;         // d_col_vx_half[j] == j
  int2* d_half_map = nullptr;         // n_vh (accumulator column of vx, of -vx or -1)
  mutable bool r_half = false;
  float2* d_W = nullptr;              // n_act * K
  float2* d_G = nullptr;              // n_act * K
  float2* d_Gsum = nullptr;           // n_act * K (combine = 1 only)
  float2* d_R = nullptr;              // n_vx * Sy * K   R[j][sy][k]
  float* d_Call = nullptr;            // S * K: coefficients of ingested frames at their scan
                                      // positions (only the pending ones are ever read)
  float* d_Call_alt = nullptr;        // the other coefficient store: a reset after ingests swaps
                                      // them, so the next acquisition's projection may overlap
                                      // (PDL) the previous acquisition's readout, which still
                                      // reads the old store
  bool c_fresh = false;               // d_Call was swapped in by the last reset (not yet written) and
                                      // its first projection may be PDL-launched (see wdd_reset)
  bool c_read_since_swap = false;     // a row transform (reader of d_Call) was launched since the last swap
  bool barrier_since_swap = false;    // shard groups: a readout barrier collective since the last swap
  int32_t* d_act_vy = nullptr;
  int32_t* d_col_off = nullptr;
  int32_t* d_vpos = nullptr;          // n_act flattened v (scatter positions)
  int2* d_flush_tiles = nullptr;
  float2* d_o = nullptr;              // n_act (multi-rank combine of o)
  float2* d_opart = nullptr;          // opart_cap x n_act partial readouts (per colfft k-tile)
  int32_t* d_gidx = nullptr;          // S: accumulator row of v, or -1 (inactive)
  int32_t* d_iota = nullptr;          // Sy: 0, 1, ..., Sy-1 (row list of contiguous flushes)
  uint32_t* d_ones = nullptr;         // Sy x mask_words all-ones pending masks (complete rows)
  int64_t g_dc = 0;                   // accumulator row of v = 0
  int opart_cap = 1;                  // rows of d_opart
  int opart_tiles = 0;                // valid partial-readout rows for the current G (0: stale)
  bool G_zero = true;                 // G is logically zero (reset); its memory may be stale
  // spectrum-only accumulator (opts.accumulator = 1): each flush adds its increment
  // of o = sum_k G K_v to d_oacc; R keeps every row's DFT so G = F_y R is formed on demand
  bool o_only = false;
  float2* d_oacc = nullptr;           // n_act
  std::vector<uint32_t> ingested;     // spectrum-only plans: Sy x mask_words positions ingested since the reset
  float2* d_spec = nullptr;           // Sy*Sx
  // pipelined GEMM flush (rgemm_kernel): (column j, first vy) of 128-row tiles, G / W tensor maps
  std::vector<int2> rg_items;
  int2* d_rg_items = nullptr;
  alignas(64) unsigned char rg_tmap[6 * 128] = {};   // RgMaps (kernels.cu): W, G, R tensor maps
  bool rg_ready = false;
  FullWddWork* fw = nullptr;          // conventional-WDD workspace (first wdd_full_wdd call)
  float2* d_img_tmp = nullptr;        // Sy*Sx scratch of the image transform (row pass)
  void* d_meta = nullptr;             // per-chunk row tables
  void* h_meta = nullptr;             // pinned host mirror of d_meta (2 slots)
  cudaEvent_t meta_ev[2] = {nullptr, nullptr};
  int meta_slot = 0;
  size_t meta_slot_bytes = 0;
  int64_t chunk_cap = 0;
  void* d_stage[2] = {nullptr, nullptr};  // host-ingest staging
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};   // staging slot consumed by the projection
  cudaEvent_t copy_ev[2] = {nullptr, nullptr};    // staging slot filled by the H2D copy
  int stage_slot = 0;
  cudaStream_t copy_stream = nullptr;
  cufftHandle fft = 0;
  bool fft_ok = false;
  cudaStream_t stream = nullptr;      // plan stream (last ingest)
  // pipelined readouts (opts.readout_async): readout-family calls run on ro_stream, forked from
  // the plan stream (ro_fork); ro_done[par] = the latest readout that read coefficient store par,
  // ro_last = the latest readout; *_valid: recorded in the current context (eagerly, or inside the
  // capture in progress -- a capture's records are joined at capture end and then forgotten)
  int readout_async = 0;
  cudaStream_t ro_stream = nullptr;
  cudaEvent_t ro_fork = nullptr, ro_fork_sync = nullptr, ro_last = nullptr, ro_done[2] = {nullptr, nullptr};
  bool ro_last_valid = false, ro_done_valid[2] = {false, false};

  // multi-rank
  void* nccl = nullptr;
  int nranks = 1, rank = 0;

  // graph capture
  bool capturing = false;
  void* cap_host = nullptr;           // pinned arena for captured metadata copies
  void* cap_dev = nullptr;            // device arena (same offsets)
  size_t cap_bytes = 0, cap_used = 0;
  std::vector<cudaGraphExec_t> graphs;

  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::pair<int, size_t>> prof_marks;  // (slot, index of start event)
  int64_t launches = 0;
};

// ---- kernel launchers (kernels.cu); return cudaError_t of the launch
// projection of n frames; C row of frame f = idx ? idx[f] : f (idx: device array or null)
// projection of n frames; scan position of frame f = idx ? idx[f] : pos0 + f (idx: device array or
// null); coefficient rows go to `dst`.  wait_start: the kernel waits for the preceding grid before
// reading frames (the frames may be produced by a caller kernel right before the ingest); else
// frames are read at once (ingest_overlap)
cudaError_t launch_project(const Plan& p, const void* frames, int64_t n, const ProjDst& dst, const int32_t* idx,
                           int64_t pos0, cudaStream_t st, bool wait_start);
// cudaFuncSetAttribute once per (device, kernel, attribute, value); thread-safe
cudaError_t func_attr_once(const void* fn, cudaFuncAttribute attr, int value);
// row DFT (a4) of the listed scan rows from the pending positions of d_Call (masks: n_rows x
// mask_words bits) into R; FFT for power-of-two Sx, DFT matrix otherwise
// kbase / KR: only coefficients kbase .. kbase + KR - 1, R as a [n_vx][Sy][KR] chunk (KR <= 0: all)
cudaError_t launch_rowdft(const Plan& p, const int32_t* rows, const uint32_t* masks, int n_rows, cudaStream_t st,
                          int kbase = 0, int KR = 0);
// rank update (a5) of the listed staged rows of R into G; FFT along y or DFT matrix
// (overwrite: G is logically zero, write instead of accumulate).  The FFT form also writes the
// per-k-tile partial Wiener readout d_opart[colfft_tiles][n_act].
// o_only: spectrum-only plans -- no G update, the partial readouts are of this flush's increment
// kind: flush_kind() result to use (-1: choose); row0 >= 0: the rows are row0 .. row0 + n_rows - 1
cudaError_t launch_flush(const Plan& p, const int32_t* rows, int n_rows, bool overwrite, cudaStream_t st,
                         bool o_only = false, int kind = -1, int row0 = -1, int kbase = 0, int KR = 0);
int flush_chunk(const Plan& p);   // coefficients per L2-resident R chunk of an FFT flush (Kl: none)
// o_acc += sum of `tiles` partial readouts (spectrum-only plans)
cudaError_t launch_oacc(const Plan& p, int tiles, cudaStream_t st);
bool flush_uses_fft(const Plan& p, int n_rows);
bool rowfft_applies(const Plan& p);   // the row transform is rowfft_kernel (power-of-two Sx <= 1024)
// a4 + a5 + a6 in one cluster kernel (scans up to 256 x 256): row FFT, y-FFT, G update and the
// partial readouts (fused_tiles of them), R never materialised; rows / masks as launch_rowdft
bool fused_possible(const Plan& p);
int fused_tiles(const Plan& p);
cudaError_t launch_fft2(const Plan& p, const int32_t* rows, const uint32_t* masks, int n_rows, bool overwrite,
                        bool o_only, cudaStream_t st);
int flush_kind(const Plan& p, int n_rows, bool allow_rg = true);   // 3 pipelined GEMM, 2 GEMM, 1 FFT, 0 DFT matrix
int flush_tiles(const Plan& p, int n_rows, int kind = -1);   // partial-readout tiles a flush writes (0: none)
bool rgemm_possible(const Plan& p, int n_rows);
cudaError_t rgemm_prepare(Plan& p);   // tensor maps + item table of the pipelined GEMM flush
int colfft_tiles(const Plan& p);
int colfft_tiles_max(const Plan& p);   // >= colfft_tiles(p) whatever r_half
bool finalize_uses_fft(const Plan& p);
// o[g] = sum_k G[g][k] W[g][k] (one warp per active v)
cudaError_t launch_readout(const Plan& p, const float2* G, float2* o, cudaStream_t st);
// an ordinary (non-PDL) launch of an empty kernel that triggers nothing early: every later kernel
// starts after all earlier work on the stream has completed (around the shard barrier collective)
cudaError_t launch_fence(cudaStream_t st);
// image from the partial readouts op[tiles][n_act] (summed over tiles in order)
cudaError_t launch_finalize(const Plan& p, const float2* op, int tiles, float2* out, cudaStream_t st);
// o[g] = fixed-order sum of `tiles` partial readouts (n_act entries, accumulator order)
cudaError_t launch_otiles(const Plan& p, const float2* op, int tiles, float2* o, cudaStream_t st);
// dense image-order spectrum from partial readouts (writes the active positions only)
cudaError_t launch_spectrum(const Plan& p, const float2* op, int tiles, float2* spec, cudaStream_t st);
// a8 from a dense Sy x Sx spectrum
cudaError_t launch_image(const Plan& p, const float2* spec, float2* out, cudaStream_t st);
// host helper: pack the fp16 B operand image of the projection kernel
void pack_basis_fp16(const Plan& p, std::vector<uint16_t>& out, double& scale);
size_t project_smem_bytes(int Q, int L);
bool project_is_lean(const Plan& p);   // projection runs two CTAs per SM for this plan
int project_occupancy(const Plan& p);  // resident projection CTAs per SM (runtime occupancy query)
// plan-time Wiener bank (Algorithm 1) on the GPU in float64 (bank.cu): q_host = detector grid
// (Q), apx_host = aperture pixel interval of each detector row (x > y: empty), [ax_lo,
// ax_lo + n_axc) the aperture's column range; writes n_act x K complex64 (or complex128 if f64)
// in accumulator order to W_dev; needs the plan's column tables on the device; synchronous
cudaError_t build_bank(const Plan& p, const double* q_host, const int2* apx_host, int ax_lo, int n_axc, void* W_dev,
                       bool f64);
constexpr double kPi = 3.14159265358979323846;
// conventional (full) WDD of a whole scan (fullwdd.cu): frames_dev S x Q x Q in
// scan order, out_dev Sy x Sx complex64; stream-ordered on p.stream; err receives a message
wdd_status full_wdd(Plan& p, const void* frames_dev, void* out_dev, char* err, size_t errn);
void full_wdd_release(Plan& p);

}  // namespace wdd
