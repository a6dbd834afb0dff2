// plan.cpp -- host side of libwdd: plan-time float64 math (basis, twiddles, exact active set,
// Wiener bank; Algorithm 1), buffer management, ingest
// bookkeeping (range / duplicate checks, row grouping, staging policy), readout orchestration
// and the NCCL combine.  No step of the per-frame path runs here: it only launches kernels.
//
// Compiled with -ffp-contract=off so the aperture tests round exactly like the float64 oracle
// reading R10.
#include <cuda_runtime.h>
#include <cufft.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

using namespace wdd;

namespace {

thread_local std::string g_err = "no error";

wdd_status fail(wdd_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CUDA_TRY(expr)                                                                          \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      return fail(e_ == cudaErrorMemoryAllocation ? WDD_E_NOMEM : WDD_E_CUDA, "%s: %s (%s:%d)", \
                  #expr, cudaGetErrorString(e_), __FILE__, __LINE__);                           \
  } while (0)

#define NCCL_TRY(expr)                                                                     \
  do {                                                                                     \
    ncclResult_t r_ = (expr);                                                              \
    if (r_ != ncclSuccess) return fail(WDD_E_NCCL, "%s: %s", #expr, ncclGetErrorString(r_)); \
  } while (0)


// ------------------------------------------------------------------ plan math (float64)
// Normalised Hermite functions by the three-term recurrence (R3).
void hermite_basis(int Q, int L, double sigma, std::vector<double>& Psi) {
  Psi.assign((size_t)Q * L, 0.0);
  const int c = Q / 2;
  const double norm = 1.0 / std::sqrt(sigma), p0 = std::pow(kPi, -0.25);
  for (int m = 0; m < Q; ++m) {
    const double u = (m - c) / sigma;
    double pm2 = 0, pm1 = p0 * std::exp(-0.5 * u * u);
    Psi[(size_t)m * L] = pm1 * norm;
    if (L > 1) {
      double p1 = std::sqrt(2.0) * u * pm1;
      Psi[(size_t)m * L + 1] = p1 * norm;
      pm2 = pm1;
      pm1 = p1;
    }
    for (int n = 2; n < L; ++n) {
      const double pn = std::sqrt(2.0 / n) * u * pm1 - std::sqrt((n - 1.0) / n) * pm2;
      Psi[(size_t)m * L + n] = pn * norm;
      pm2 = pm1;
      pm1 = pn;
    }
  }
}

int64_t signed_freq(int64_t v, int64_t S) { return v < (S + 1) / 2 ? v : v - S; }  // fftfreq (R15)

struct ApertureRows {
  std::vector<int> row_begin;  // Q + 1
  std::vector<int> mx;         // pixels inside the aperture, row-major
};

ApertureRows aperture(const Plan& p, const std::vector<double>& q) {
  ApertureRows a;
  a.row_begin.assign(p.Q + 1, 0);
  const double qa2 = p.qa * p.qa;
  for (int my = 0; my < p.Q; ++my) {
    a.row_begin[my] = (int)a.mx.size();
    for (int mx = 0; mx < p.Q; ++mx)
      if (q[my] * q[my] + q[mx] * q[mx] <= qa2) a.mx.push_back(mx);
  }
  a.row_begin[p.Q] = (int)a.mx.size();
  return a;
}

// Exact discrete active set (R9, R10): v active iff some aperture pixel q also has
// |q + q_hat_v|^2 <= q_alpha^2.  Candidates need |q_hat_v| <= 2 q_alpha (triangle inequality).
void active_set(const Plan& p, const std::vector<double>& q, const ApertureRows& ap, std::vector<int32_t>& act) {
  const double qa2 = p.qa * p.qa, lim = 2.0 * p.qa * (1.0 + 1e-9);
  std::vector<double> fy(p.Sy), fx(p.Sx);
  for (int v = 0; v < p.Sy; ++v) fy[v] = (double)signed_freq(v, p.Sy) / ((double)p.Sy * p.step);
  for (int v = 0; v < p.Sx; ++v) fx[v] = (double)signed_freq(v, p.Sx) / ((double)p.Sx * p.step);
  std::vector<std::pair<int, int>> cand;
  for (int vy = 0; vy < p.Sy; ++vy) {
    if (std::fabs(fy[vy]) > lim) continue;
    for (int vx = 0; vx < p.Sx; ++vx)
      if (fy[vy] * fy[vy] + fx[vx] * fx[vx] <= lim * lim) cand.emplace_back(vy, vx);
  }
  std::vector<uint8_t> on(cand.size(), 0);
  const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::atomic<size_t> next(0);
  auto work = [&]() {
    for (;;) {
      const size_t i0 = next.fetch_add(256);
      if (i0 >= cand.size()) break;
      for (size_t i = i0; i < std::min(cand.size(), i0 + 256); ++i) {
        const double sy = fy[cand[i].first], sx = fx[cand[i].second];
        bool hit = false;
        for (int my = 0; my < p.Q && !hit; ++my) {
          const double a = q[my] + sy;
          for (int e = ap.row_begin[my]; e < ap.row_begin[my + 1]; ++e) {
            const double b = q[ap.mx[e]] + sx;
            if (a * a + b * b <= qa2) { hit = true; break; }
          }
        }
        on[i] = hit;
      }
    }
  };
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t) th.emplace_back(work);
  for (auto& t : th) t.join();
  act.clear();
  for (size_t i = 0; i < cand.size(); ++i)
    if (on[i]) act.push_back(cand[i].first * p.Sx + cand[i].second);
}

// Aperture pixel interval of every detector row (the disc's rows are contiguous) and the
// aperture's column range, the tables the GPU bank build (bank.cu) works from.
struct ApertureIntervals {
  std::vector<int2> rows;
  int ax_lo = 0, n_axc = 0;
};

bool aperture_intervals(const Plan& p, const ApertureRows& ap, ApertureIntervals& out) {
  out.rows.assign(p.Q, make_int2(1, 0));
  int lo = p.Q, hi = -1;
  for (int my = 0; my < p.Q; ++my) {
    const int b = ap.row_begin[my], e = ap.row_begin[my + 1];
    if (b == e) continue;
    if (ap.mx[e - 1] - ap.mx[b] != e - 1 - b) return false;
    out.rows[my] = make_int2(ap.mx[b], ap.mx[e - 1]);
    lo = std::min(lo, ap.mx[b]);
    hi = std::max(hi, ap.mx[e - 1]);
  }
  out.ax_lo = hi >= lo ? lo : 0;
  out.n_axc = hi >= lo ? hi - lo + 1 : 0;
  return true;
}


void twiddles(int n_out, const int32_t* freqs, int S, std::vector<float2>& F) {
  // F[j][s] = exp(-2 pi i ((f_j * s) mod S) / S) / sqrt(S)  (integer angle reduction)
  F.resize((size_t)n_out * S);
  const double inv = 1.0 / std::sqrt((double)S);
  for (int j = 0; j < n_out; ++j)
    for (int s = 0; s < S; ++s) {
      const int64_t r = ((int64_t)freqs[j] * s) % S;
      const double ang = -2.0 * kPi * (double)r / (double)S;
      F[(size_t)j * S + s] = make_float2((float)(std::cos(ang) * inv), (float)(std::sin(ang) * inv));
    }
}

// FFT twiddles tw[m] = exp(-2 pi i m / N), m < N (unscaled; the kernels apply 1/sqrt(N))
void fft_twiddles(int N, std::vector<float2>& tw) {
  tw.resize(std::max(1, N));
  for (int m = 0; m < (int)tw.size(); ++m) {
    const double ang = -2.0 * kPi * (double)m / (double)N;
    tw[m] = make_float2((float)std::cos(ang), (float)std::sin(ang));
  }
}

// ------------------------------------------------------------------ launch helpers
struct Prof {
  Plan& p;
  cudaStream_t st;
  int slot;
  size_t i0 = 0;
  Prof(Plan& pp, int s, cudaStream_t stream) : p(pp), st(stream), slot(s) {
    p.launches++;
    if (!p.prof || p.capturing) return;
    if (p.ev_used + 2 > p.ev_pool.size()) {
      for (int k = 0; k < 64; ++k) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        p.ev_pool.push_back(e);
      }
    }
    i0 = p.ev_used;
    p.ev_used += 2;
    cudaEventRecord(p.ev_pool[i0], st);
  }
  ~Prof() {
    if (!p.prof || p.capturing) return;
    cudaEventRecord(p.ev_pool[i0 + 1], st);
    p.prof_marks.emplace_back(slot, i0);
  }
};

constexpr int64_t kMaxLaunchFrames = 1 << 20;   // frames of one projection launch (contiguous calls)

// Two coefficient stores (WDD_C_DOUBLE=0: one; the first projection of every acquisition then waits
// for the previous readout).
bool double_c_store() {
  static const bool on = [] { const char* e = std::getenv("WDD_C_DOUBLE"); return !(e && std::atoi(e) == 0); }();
  return on;
}

wdd_status check_plan(wdd_plan_t plan) {
  if (!plan) return fail(WDD_E_ARG, "plan is NULL");
  return WDD_OK;
}

Plan* P(wdd_plan_t h) { return reinterpret_cast<Plan*>(h); }

void use_stream(Plan& p, cudaStream_t st) {
  if (st == p.stream || p.capturing) return;
  // keep the plan's own work ordered across a stream switch
  cudaEvent_t e;
  if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) {
    cudaEventRecord(e, p.stream);
    cudaStreamWaitEvent(st, e, 0);
    cudaEventDestroy(e);
  }
  p.stream = st;
}

// Readout-family calls of a plan with opts.readout_async: the scope forks the readout stream off
// the plan stream (everything enqueued so far, i.e. every projection the readout reads, comes
// first), points p.stream at it for the calls inside, and records the completion events the
// plan stream's later hazards wait for (wdd_reset, wdd_graph_launch, wdd_readout_wait).
struct RoScope {
  Plan& p;
  cudaStream_t saved = nullptr;
  bool on = false;
  wdd_status status = WDD_OK;
  explicit RoScope(Plan& q) : p(q) {
    if (!p.readout_async) return;
    if (cudaEventRecord(p.ro_fork, p.stream) != cudaSuccess || cudaStreamWaitEvent(p.ro_stream, p.ro_fork, 0) != cudaSuccess) {
      status = fail(WDD_E_CUDA, "readout stream fork: %s", cudaGetErrorString(cudaGetLastError()));
      return;
    }
    saved = p.stream;
    p.stream = p.ro_stream;
    on = true;
  }
  ~RoScope() {
    if (!on) return;
    const int par = p.d_Call_alt ? p.store_par : 0;
    if (cudaEventRecord(p.ro_done[par], p.ro_stream) == cudaSuccess) p.ro_done_valid[par] = true;
    if (cudaEventRecord(p.ro_last, p.ro_stream) == cudaSuccess) p.ro_last_valid = true;
    p.stream = saved;
  }
};

// stream waits for an event if it was recorded in the current context
cudaError_t wait_if(cudaStream_t st, cudaEvent_t e, bool valid) { return valid ? cudaStreamWaitEvent(st, e, 0) : cudaSuccess; }

wdd_status upload_meta(Plan& p, const void* host, size_t bytes, void** dev_out) {
  if (bytes > p.meta_slot_bytes) return fail(WDD_E_ARG, "metadata too large");
  if (p.capturing) {
    // captured copies read a host block that outlives every replay: bump-allocate from the
    // pinned / device capture arenas reserved by wdd_capture_begin (owned until destroy)
    const size_t off = (p.cap_used + 255) / 256 * 256;
    if (off + bytes > p.cap_bytes) return fail(WDD_E_NOMEM, "capture metadata arena exhausted");
    uint8_t* h = static_cast<uint8_t*>(p.cap_host) + off;
    uint8_t* d = static_cast<uint8_t*>(p.cap_dev) + off;
    std::memcpy(h, host, bytes);
    CUDA_TRY(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, p.stream));
    p.cap_used = off + bytes;
    *dev_out = d;
    return WDD_OK;
  }
  const int s = p.meta_slot;
  p.meta_slot ^= 1;
  CUDA_TRY(cudaEventSynchronize(p.meta_ev[s]));
  uint8_t* h = static_cast<uint8_t*>(p.h_meta) + s * p.meta_slot_bytes;
  uint8_t* d = static_cast<uint8_t*>(p.d_meta) + s * p.meta_slot_bytes;
  std::memcpy(h, host, bytes);
  CUDA_TRY(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, p.stream));
  CUDA_TRY(cudaEventRecord(p.meta_ev[s], p.stream));
  *dev_out = d;
  return WDD_OK;
}

// Validate a whole call (range, duplicates within the call and against the seen set) before
// anything is enqueued.  On success the indices are marked seen.
// idx[0 .. n) is the run idx[0], idx[0] + 1, ...  (frames arriving in scan order: the common case)
static bool is_run(const int32_t* idx, int64_t n) {
  for (int64_t i = 1; i < n; ++i)
    if (idx[i] != idx[0] + i) return false;
  return true;
}

// run: 1 / 0 if the caller already knows whether idx is a contiguous run, -1 to check here
wdd_status validate_and_mark(Plan& p, const int32_t* idx, int64_t n, int run = -1) {
  if (n > 0 && (run >= 0 ? run == 1 : is_run(idx, n))) {
    // contiguous run: range by its ends, duplicates word by word over the seen bitmap, then marked
    // (same outcome as the per-index loop below: nothing is marked unless the whole call is valid)
    const int64_t a = idx[0], b = a + n;   // [a, b)
    if (a < 0 || b > p.S) {
      const int64_t i = (a < 0 || a >= p.S) ? 0 : p.S - a;   // first position outside the range
      return fail(WDD_E_RANGE, "scan index %lld at position %lld outside [0, %lld)", (long long)(a + i),
                  (long long)i, (long long)p.S);
    }
    for (int64_t w = a >> 6; w <= (b - 1) >> 6; ++w) {
      const int64_t lo = std::max<int64_t>(a, w << 6), hi = std::min<int64_t>(b, (w + 1) << 6);   // [lo, hi)
      const uint64_t m = (hi - lo == 64 ? ~0ull : ((1ull << (hi - lo)) - 1)) << (lo & 63);
      if (const uint64_t d = p.seen[(size_t)w] & m) {
        const int64_t s = (w << 6) + __builtin_ctzll(d);
        return fail(WDD_E_DUP, "scan index %lld (position %lld) already ingested or repeated", (long long)s,
                    (long long)(s - a));
      }
    }
    for (int64_t w = a >> 6; w <= (b - 1) >> 6; ++w) {
      const int64_t lo = std::max<int64_t>(a, w << 6), hi = std::min<int64_t>(b, (w + 1) << 6);
      p.seen[(size_t)w] |= (hi - lo == 64 ? ~0ull : ((1ull << (hi - lo)) - 1)) << (lo & 63);
    }
    return WDD_OK;
  }
  for (int64_t i = 0; i < n; ++i)
    if (idx[i] < 0 || (int64_t)idx[i] >= p.S)
      return fail(WDD_E_RANGE, "scan index %d at position %lld outside [0, %lld)", idx[i], (long long)i,
                  (long long)p.S);
  std::vector<int32_t> marked;
  marked.reserve((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    const int32_t s = idx[i];
    uint64_t& w = p.seen[(size_t)s >> 6];
    const uint64_t bit = 1ull << (s & 63);
    if (w & bit) {
      for (int32_t m : marked) p.seen[(size_t)m >> 6] &= ~(1ull << (m & 63));
      return fail(WDD_E_DUP, "scan index %d (position %lld) already ingested or repeated", s, (long long)i);
    }
    w |= bit;
    marked.push_back(s);
  }
  return WDD_OK;
}

// Positions whose coefficients are (or, for a peer rank's frames, will be) in the current store:
// their rows are row-transformed at the next flush.
void mark_pending(Plan& p, const int32_t* idx, int64_t n, int run = -1) {
  if (n > 0 && (run >= 0 ? run == 1 : is_run(idx, n))) {
    // contiguous run: whole mask words per scan row
    const int64_t a = idx[0], b = a + n;
    for (int64_t sy = a / p.Sx; sy <= (b - 1) / p.Sx; ++sy) {
      p.row_dirty[sy] = 1;
      const int64_t x0 = std::max<int64_t>(a - sy * p.Sx, 0), x1 = std::min<int64_t>(b - sy * p.Sx, p.Sx);   // [x0, x1)
      for (int64_t w = x0 >> 5; w <= (x1 - 1) >> 5; ++w) {
        const int64_t lo = std::max<int64_t>(x0, w << 5), hi = std::min<int64_t>(x1, (w + 1) << 5);
        const uint32_t m = (hi - lo == 32 ? ~0u : ((1u << (hi - lo)) - 1)) << (lo & 31);
        p.pending[(size_t)sy * p.mask_words + w] |= m;
        if (p.o_only) p.ingested[(size_t)sy * p.mask_words + w] |= m;
      }
    }
    return;
  }
  for (int64_t i = 0; i < n; ++i) {
    const int sy = idx[i] / p.Sx, sx = idx[i] % p.Sx;
    p.row_dirty[sy] = 1;
    p.pending[(size_t)sy * p.mask_words + (sx >> 5)] |= 1u << (sx & 31);
    if (p.o_only) p.ingested[(size_t)sy * p.mask_words + (sx >> 5)] |= 1u << (sx & 31);
  }
}

// The current store of shard o (this plan's or a peer's, as mapped into this process)
float* shard_store(const Plan& p, int o) {
  const int Ko = (p.a_split[o + 1] - p.a_split[o]) * p.L;
  return p.peer_base[o] + (size_t)p.store_par * p.S * Ko;
}

ProjDst proj_dst(const Plan& p) {
  ProjDst d;
  d.n = p.nshard;
  for (int o = 0; o < p.nshard; ++o) {
    d.C[o] = p.nshard == 1 ? p.d_Call : shard_store(p, o);
    d.K[o] = (p.a_split[o + 1] - p.a_split[o]) * p.L;
    d.alo[o] = p.a_split[o];
  }
  d.alo[p.nshard] = p.L;
  return d;
}

// Enqueue the projection of one chunk of already-validated frames; its coefficients land in
// the coefficient store(s) at their scan positions (the row DFT happens at flush time).
wdd_status enqueue_chunk(Plan& p, const void* frames_dev, const int32_t* idx, int64_t nc, bool first, int run = -1) {
  cudaStream_t st = p.stream;
  const bool contiguous = run >= 0 ? run == 1 : is_run(idx, nc);
  const ProjDst dst = proj_dst(p);
  const int32_t* d_idx = nullptr;
  if (!contiguous) {
    void* d = nullptr;
    wdd_status s = upload_meta(p, idx, (size_t)nc * sizeof(int32_t), &d);
    if (s != WDD_OK) return s;
    d_idx = static_cast<const int32_t*>(d);
  }
  {
    Prof pr(p, kSlotProject, st);
    // (frames of the first chunk of a call may come from a caller kernel enqueued right before it:
    // unless the plan was created with ingest_overlap, that launch reads them only after its
    // predecessor grid has completed; later chunks are ordered behind it)
    // (a single-rank plan knows how much of the scan is still to come: the launches that end a scan
    // spread their frames thinner, so the chain's last CTAs finish together -- see launch_project_t)
    p.proj_rem_after = (p.nranks == 1 && p.nshard == 1) ? std::max<int64_t>(0, p.S - (p.frames_enqueued + nc)) : -1;
    const cudaError_t e = launch_project(p, frames_dev, nc, dst, d_idx, contiguous ? idx[0] : 0, st,
                                         first && !p.ingest_overlap);
    p.proj_rem_after = -1;
    CUDA_TRY(e);
  }
  p.frames_enqueued += nc;
  p.c_fresh = false;
  // The row DFT of completed rows is deferred to the next flush (readout): launched per batch it
  // would sit between the PDL-chained projection launches and stall them (measured: 246 us vs
  // 162 us per Medium acquisition).
  mark_pending(p, idx, nc, contiguous ? 1 : 0);
  return WDD_OK;
}

size_t frame_bytes(const Plan& p) { return (size_t)p.Q * p.Q * (p.dtype == 0 ? 2 : 4); }

// Row DFT (a4) of the pending positions of the listed rows into the row staging R; the rows
// become *staged* (R holds their DFT until the next rank update folds it into G).  The metadata
// block is the row list followed by one pending bitmask per row; positions outside the mask are
// read as zeros, so the coefficient store never needs clearing (each scan position is ingested at
// most once per reset).  A contiguous range of complete rows (offline scans, live scans in scan
// order) needs no upload: the rows are a slice of the plan's device iota and the masks all-ones.
// Row list + per-row pending masks of a row transform (device pointers *dr / *dm; the bookkeeping:
// the rows' pending positions are consumed).  A contiguous range of complete rows needs no upload.
wdd_status row_blob(Plan& p, const std::vector<int32_t>& rows_in, const int32_t** dr_out, const uint32_t** dm_out) {
  const int n_rows = (int)rows_in.size();
  std::vector<int32_t> blob(rows_in);
  const size_t mask_off = ((size_t)n_rows + 3) / 4 * 4;
  blob.resize(mask_off + (size_t)n_rows * p.mask_words, 0);
  bool simple = blob[n_rows - 1] - blob[0] == n_rows - 1;
  for (int r = 0; r < n_rows; ++r) {
    const int sy = blob[r];
    for (int w = 0; w < p.mask_words; ++w) {
      uint32_t& m = p.pending[(size_t)sy * p.mask_words + w];
      const int bits = std::min(32, p.Sx - 32 * w);
      const uint32_t full = bits == 32 ? 0xFFFFFFFFu : ((1u << bits) - 1u);
      simple = simple && m == full;
      blob[mask_off + (size_t)r * p.mask_words + w] = (int32_t)m;
      m = 0;
    }
    p.row_dirty[sy] = 0;
  }
  if (simple) {
    *dr_out = p.d_iota + blob[0];
    *dm_out = p.d_ones;
    return WDD_OK;
  }
  void* d = nullptr;
  wdd_status s = upload_meta(p, blob.data(), blob.size() * sizeof(int32_t), &d);
  if (s != WDD_OK) return s;
  *dr_out = static_cast<const int32_t*>(d);
  *dm_out = reinterpret_cast<const uint32_t*>(*dr_out + mask_off);
  return WDD_OK;
}

wdd_status stage_rows(Plan& p, const std::vector<int32_t>& rows_in) {
  const int n_rows = (int)rows_in.size();
  if (n_rows == 0) return WDD_OK;
  const int32_t* dr = nullptr;
  const uint32_t* dm = nullptr;
  wdd_status s = row_blob(p, rows_in, &dr, &dm);
  if (s != WDD_OK) return s;
  for (int32_t sy : rows_in) p.row_staged[sy] = 1;
  Prof pr(p, kSlotRowDft, p.stream);
  CUDA_TRY(launch_rowdft(p, dr, dm, n_rows, p.stream));
  p.c_read_since_swap = true;
  return WDD_OK;
}

// Flush: row DFT of the rows that still have pending positions (partial rows), then the
// phase-weighted rank update (a5, with the fused partial readout a6) of G over every staged row.
wdd_status flush(Plan& p) {
  std::vector<int32_t> rows;
  for (int sy = 0; sy < p.Sy; ++sy)
    if (p.row_dirty[sy]) rows.push_back(sy);
  p.r_half = false;
  if (!rows.empty() && flush_kind(p, (int)rows.size()) == 1 && fused_possible(p)) {
    // the whole flush (row FFT, y-FFT, G update, partial readouts) in one cluster kernel
    const int32_t* dr = nullptr;
    const uint32_t* dm = nullptr;
    wdd_status s = row_blob(p, rows, &dr, &dm);
    if (s != WDD_OK) return s;
    {
      Prof pr(p, kSlotFlush, p.stream);
      CUDA_TRY(launch_fft2(p, dr, dm, (int)rows.size(), p.G_zero, p.o_only, p.stream));
    }
    p.c_read_since_swap = true;
    if (p.o_only) {
      Prof pr(p, kSlotReadout, p.stream);
      CUDA_TRY(launch_oacc(p, fused_tiles(p), p.stream));
      return WDD_OK;
    }
    p.G_zero = false;
    p.opart_tiles = fused_tiles(p);
    return WDD_OK;
  }
  if (!rows.empty() && flush_kind(p, (int)rows.size()) == 1 && flush_chunk(p) < p.Kl) {
    // FFT flush in coefficient chunks whose R staging stays in L2: per chunk, the row FFT of the
    // pending rows and the y-FFT + G update + partial readouts of the same coefficients
    const int32_t* dr = nullptr;
    const uint32_t* dm = nullptr;
    wdd_status s = row_blob(p, rows, &dr, &dm);
    if (s != WDD_OK) return s;
    const int n_rows = (int)rows.size(), KR = flush_chunk(p);
    const bool contig = rows.back() - rows.front() == n_rows - 1;
    p.r_half = p.n_vh > 0;
    for (int kb = 0; kb < p.Kl; kb += KR) {
      {
        Prof pr(p, kSlotRowDft, p.stream);
        CUDA_TRY(launch_rowdft(p, dr, dm, n_rows, p.stream, kb, KR));
      }
      Prof pr(p, kSlotFlush, p.stream);
      CUDA_TRY(launch_flush(p, dr, n_rows, p.G_zero, p.stream, p.o_only, 1, contig ? rows.front() : -1, kb, KR));
    }
    p.c_read_since_swap = true;
    if (p.o_only) {
      Prof pr(p, kSlotReadout, p.stream);
      CUDA_TRY(launch_oacc(p, flush_tiles(p, n_rows, 1), p.stream));
      return WDD_OK;
    }
    p.G_zero = false;
    p.opart_tiles = flush_tiles(p, n_rows, 1);
    return WDD_OK;
  }
  // (the flush form is chosen before the rows are staged: an FFT flush stages the half plane)
  int n_stage = 0;
  for (int sy = 0; sy < p.Sy; ++sy) n_stage += (p.row_staged[sy] || p.row_dirty[sy]) ? 1 : 0;
  if (n_stage == 0) return WDD_OK;
  const int kind = flush_kind(p, n_stage);
  p.r_half = kind == 1 && p.n_vh > 0;   // (rows are staged and consumed within one flush call)
  wdd_status s = stage_rows(p, rows);
  if (s != WDD_OK) return s;
  rows.clear();
  for (int sy = 0; sy < p.Sy; ++sy)
    if (p.row_staged[sy]) rows.push_back(sy);
  const int n_rows = (int)rows.size();
  if (n_rows == 0) return WDD_OK;
  const int32_t* dr = nullptr;
  const bool contig = rows.back() - rows.front() == n_rows - 1;
  if (contig) {
    dr = p.d_iota + rows.front();
  } else {
    void* d = nullptr;
    if ((s = upload_meta(p, rows.data(), rows.size() * sizeof(int32_t), &d)) != WDD_OK) return s;
    dr = static_cast<const int32_t*>(d);
  }
  {
    Prof pr(p, kSlotFlush, p.stream);
    CUDA_TRY(launch_flush(p, dr, n_rows, p.G_zero, p.stream, p.o_only, kind, contig ? rows.front() : -1));
  }
  for (int32_t sy : rows) p.row_staged[sy] = 0;
  if (p.o_only) {                     // o += this flush's increment; G is not touched
    Prof pr(p, kSlotReadout, p.stream);
    CUDA_TRY(launch_oacc(p, flush_tiles(p, n_rows, kind), p.stream));
    return WDD_OK;
  }
  p.G_zero = false;
  p.opart_tiles = flush_tiles(p, n_rows, kind);
  return WDD_OK;
}

// Spectrum-only plans keep no G: form it on request from the coefficient store, which holds every
// position ingested since the reset (never cleared, each position ingested at most once) -- row
// DFT of every ingested position into R (scratch here: flush() has emptied it), then one rank
// update into G with overwrite.
wdd_status form_G(Plan& p) {
  std::vector<int32_t> rows;
  for (int sy = 0; sy < p.Sy; ++sy)
    for (int w = 0; w < p.mask_words; ++w)
      if (p.ingested[(size_t)sy * p.mask_words + w]) {
        rows.push_back(sy);
        break;
      }
  if (rows.empty()) {
    CUDA_TRY(cudaMemsetAsync(p.d_G, 0, (size_t)p.n_act * p.Kl * sizeof(float2), p.stream));
    return WDD_OK;
  }
  const int n_rows = (int)rows.size();
  std::vector<int32_t> blob(rows);
  const size_t mask_off = ((size_t)n_rows + 3) / 4 * 4;
  blob.resize(mask_off + (size_t)n_rows * p.mask_words, 0);
  for (int r = 0; r < n_rows; ++r)
    for (int w = 0; w < p.mask_words; ++w)
      blob[mask_off + (size_t)r * p.mask_words + w] = (int32_t)p.ingested[(size_t)rows[r] * p.mask_words + w];
  void* d = nullptr;
  wdd_status s = upload_meta(p, blob.data(), blob.size() * sizeof(int32_t), &d);
  if (s != WDD_OK) return s;
  const int32_t* dr = static_cast<const int32_t*>(d);
  const int kind = flush_kind(p, n_rows);
  p.r_half = kind == 1 && p.n_vh > 0;
  CUDA_TRY(launch_rowdft(p, dr, reinterpret_cast<const uint32_t*>(dr + mask_off), n_rows, p.stream));
  p.c_read_since_swap = true;
  CUDA_TRY(launch_flush(p, dr, n_rows, /*overwrite*/ true, p.stream, false, kind));
  p.r_half = false;
  return WDD_OK;
}

// Make the memory of G hold its logical value (after a reset nothing has been written yet).
wdd_status materialize_G(Plan& p) {
  if (p.o_only) return form_G(p);
  if (p.G_zero) {
    CUDA_TRY(cudaMemsetAsync(p.d_G, 0, (size_t)p.n_act * p.Kl * sizeof(float2), p.stream));
    p.G_zero = false;
    p.opart_tiles = 0;
  }
  return WDD_OK;
}

// Shard groups: the coefficient rows of this plan's shard arrive from every rank's projections
// (peer stores).  Before the flush reads them, every rank's earlier work must be complete: an
// ordinary launch of an empty kernel (starts once all earlier work on this stream is done), a
// one-element allreduce (completes once every rank has reached it), and another empty kernel
// (later kernels start only after the collective has completed, however NCCL launches).
wdd_status shard_barrier(Plan& p) {
  if (p.nshard == 1 || !p.nccl) return WDD_OK;
  CUDA_TRY(launch_fence(p.stream));
  NCCL_TRY(ncclAllReduce(p.d_o, p.d_o, 1, ncclFloat, ncclSum, reinterpret_cast<ncclComm_t>(p.nccl), p.stream));
  CUDA_TRY(launch_fence(p.stream));
  p.barrier_since_swap = true;
  return WDD_OK;
}

// Flush, Wiener readout and (combine && a communicator is attached) the NCCL combine; *op / *tiles
// receive the partial readouts the image transform sums (tiles rows of n_act, accumulator order).
//  - G accumulator: the fused partial readouts of the flush (a6 in the rank-update epilogue), or one
//    readout pass over G when the last flush left none (DFT-matrix flush, nothing flushed);
//  - spectrum-only accumulator: the running o.
// Multi-rank ("merge ... sums up the contributions"): combine = 0 sums the partial
// readouts into o (n_act) and allreduces o -- exact by linearity, K x fewer bytes than G;
// combine = 1 (north star) allreduces the partial G and runs the readout on the sum.
wdd_status readout_spectrum(Plan& p, bool combine, const float2** op_out, int* tiles_out) {
  wdd_status s = WDD_OK;
  if (combine && (s = shard_barrier(p)) != WDD_OK) return s;
  if ((s = flush(p)) != WDD_OK) return s;
  const float2* op = p.d_opart;
  int tiles = p.opart_tiles;
  if (p.o_only) {
    op = p.d_oacc;
    tiles = 1;
  } else if (tiles == 0 && !(combine && p.nccl && p.combine == 1)) {
    if ((s = materialize_G(p)) != WDD_OK) return s;
    Prof pr(p, kSlotReadout, p.stream);
    CUDA_TRY(launch_readout(p, p.d_G, p.d_opart, p.stream));
    p.opart_tiles = tiles = 1;
  }
  if (combine && p.nccl) {
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(p.nccl);
    if (!p.o_only && p.combine == 1) {
      if ((s = materialize_G(p)) != WDD_OK) return s;
      NCCL_TRY(ncclAllReduce(p.d_G, p.d_Gsum, (size_t)p.n_act * p.Kl * 2, ncclFloat, ncclSum, comm, p.stream));
      Prof pr(p, kSlotReadout, p.stream);
      CUDA_TRY(launch_readout(p, p.d_Gsum, p.d_o, p.stream));
    } else {
      Prof pr(p, kSlotReadout, p.stream);
      CUDA_TRY(launch_otiles(p, op, tiles, p.d_o, p.stream));
    }
    if (p.o_only || p.combine == 0)
      NCCL_TRY(ncclAllReduce(p.d_o, p.d_o, (size_t)p.n_act * 2, ncclFloat, ncclSum, comm, p.stream));
    op = p.d_o;
    tiles = 1;
  }
  *op_out = op;
  *tiles_out = tiles;
  return WDD_OK;
}

void free_plan(Plan* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  if (p->stream) cudaStreamSynchronize(p->stream);
  if (p->ro_stream) cudaStreamSynchronize(p->ro_stream);
  cudaDeviceSynchronize();
  if (p->nccl) ncclCommDestroy(reinterpret_cast<ncclComm_t>(p->nccl));
  for (int o = 0; o < kMaxShards; ++o)
    if (p->peers_ipc[o] && p->peer_base[o]) cudaIpcCloseMemHandle(p->peer_base[o]);
  full_wdd_release(*p);
  void* bufs[] = {p->d_rg_items, p->d_oacc, p->d_iota, p->d_ones, p->d_opart, p->d_gidx, p->d_Bpack, p->d_psi, p->d_Fx, p->d_Fy, p->d_twx, p->d_twy, p->d_col_vx, p->d_col_vx_half, p->d_half_map, p->d_W, p->d_G, p->d_Gsum, p->d_R, p->d_Cbase,
                  p->d_act_vy, p->d_col_off, p->d_vpos, p->d_flush_tiles, p->d_o, p->d_spec, p->d_img_tmp,
                  p->d_meta, p->d_stage[0], p->d_stage[1], p->d_err};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (p->h_meta) cudaFreeHost(p->h_meta);
  for (auto g : p->graphs) cudaGraphExecDestroy(g);
  if (p->cap_host) cudaFreeHost(p->cap_host);
  if (p->cap_dev) cudaFree(p->cap_dev);
  for (auto& e : p->meta_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : p->stage_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : p->copy_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : p->ev_pool) cudaEventDestroy(e);
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  for (cudaEvent_t e : {p->ro_fork, p->ro_last, p->ro_done[0], p->ro_done[1], p->ro_fork_sync})
    if (e) cudaEventDestroy(e);
  if (p->ro_stream) cudaStreamDestroy(p->ro_stream);
  if (p->fft_ok) cufftDestroy(p->fft);
  delete p;
}

}  // namespace

// =====================================================================================
// C ABI
// =====================================================================================
extern "C" {

const char* wdd_last_error(void) { return g_err.c_str(); }

wdd_status wdd_plan_create(const int32_t scan_shape[2], double step_A, const int32_t det_shape[2], int32_t K,
                           const wdd_probe* probe, double wiener_eps, const wdd_plan_opts* opts, wdd_plan_t* out) {
  if (!out) return fail(WDD_E_ARG, "out is NULL");
  *out = nullptr;
  if (!scan_shape || !det_shape || !probe) return fail(WDD_E_ARG, "NULL shape or probe");
  wdd_plan_opts o{};
  if (opts) o = *opts;
  for (int r : o.reserved)
    if (r) return fail(WDD_E_ARG, "opts.reserved must be zero");
  if (o.ingest_overlap != 0 && o.ingest_overlap != 1) return fail(WDD_E_ARG, "ingest_overlap must be 0 or 1");
  if (o.ingest_spread != 0 && o.ingest_spread != 1) return fail(WDD_E_ARG, "ingest_spread must be 0 or 1");
  if (o.readout_async != 0 && o.readout_async != 1) return fail(WDD_E_ARG, "readout_async must be 0 or 1");
  if (o.readout_async && o.k_shards > 1) return fail(WDD_E_STATE, "readout_async is not available in a shard group");
  const int Sy = scan_shape[0], Sx = scan_shape[1], Q = det_shape[0];
  if (Sy < 2 || Sx < 2 || (int64_t)Sy * Sx > (1ll << 30)) return fail(WDD_E_ARG, "scan shape %d x %d unsupported", Sy, Sx);
  if (det_shape[1] != Q || !(Q == 32 || Q == 64 || Q == 128 || Q == 256))
    return fail(WDD_E_ARG, "detector must be square with Q in {32,64,128,256}, got %d x %d", det_shape[0], det_shape[1]);
  const int L = (int)std::lround(std::sqrt((double)K));
  if (K <= 0 || L * L != K) return fail(WDD_E_ARG, "K = %d is not a perfect square", K);
  if (L % 8 != 0 || L < 8 || L > 32 || L > Q) return fail(WDD_E_ARG, "L = %d must be a multiple of 8 in [8, 32] and <= Q", L);
  if (!(wiener_eps > 0)) return fail(WDD_E_ARG, "wiener_eps must be > 0");
  if (!(step_A > 0) || !(probe->wavelength_A > 0) || !(probe->semiangle_rad > 0))
    return fail(WDD_E_ARG, "step, wavelength and semi-angle must be > 0");
  if (o.dtype != 0 && o.dtype != 1) return fail(WDD_E_ARG, "dtype must be 0 (u16) or 1 (f32)");
  if (o.combine != 0 && o.combine != 1) return fail(WDD_E_ARG, "combine must be 0 or 1");
  if (o.accumulator != 0 && o.accumulator != 1) return fail(WDD_E_ARG, "accumulator must be 0 (G) or 1 (spectrum)");
  if (o.accumulator == 1 && (Sy < 2 || Sy > 1024 || (Sy & (Sy - 1)) != 0))
    return fail(WDD_E_ARG, "the spectrum-only accumulator needs a power-of-two Sy in [2, 1024] (got %d)", Sy);
  const int nshard = o.k_shards <= 1 ? 1 : o.k_shards;
  if (o.k_shards < 0 || nshard > kMaxShards || nshard > L || o.k_rank < 0 || o.k_rank >= nshard)
    return fail(WDD_E_ARG, "k_shards = %d / k_rank = %d: need 0 <= k_rank < k_shards <= min(%d, L)", o.k_shards,
                o.k_rank, kMaxShards);

  Plan* p = new Plan();
  p->Sy = Sy; p->Sx = Sx; p->Q = Q; p->L = L; p->K = K; p->S = (int64_t)Sy * Sx;
  p->dtype = o.dtype; p->normalize = o.normalize ? 1 : 0; p->device = o.device; p->combine = o.combine;
  p->step = step_A; p->lambda = probe->wavelength_A; p->alpha = probe->semiangle_rad; p->defocus = probe->defocus_A;
  p->eps = wiener_eps;
  p->o_only = o.accumulator == 1;
  p->ingest_overlap = o.ingest_overlap;
  p->ingest_spread = o.ingest_spread;
  p->readout_async = o.readout_async;
  p->nshard = nshard;
  p->shard = nshard > 1 ? o.k_rank : 0;
  if (nshard > 1) p->combine = 0;   // (the shards' G are disjoint: the combine sums o)
  for (int i = 0; i <= nshard; ++i) p->a_split.push_back(i * L / nshard);   // as even as possible
  p->k0 = p->a_split[p->shard] * L;
  p->Kl = (p->a_split[p->shard + 1] - p->a_split[p->shard]) * L;
  p->dq = o.det_px_rad > 0 ? o.det_px_rad / p->lambda : 1.0 / (Q * step_A);  // R17
  p->qa = p->alpha / p->lambda;                                               // R7
  p->R = p->qa / p->dq;
  p->sigma = o.sigma_px > 0 ? o.sigma_px : std::sqrt(Q / (2.0 * kPi));        // R1

  auto bail = [&](wdd_status s) { free_plan(p); return s; };
  if (cudaSetDevice(p->device) != cudaSuccess) return bail(fail(WDD_E_CUDA, "cudaSetDevice(%d) failed", p->device));
  {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device) == cudaSuccess && sms > 0) p->sm_count = sms;
  }

  // basis + Gram check
  hermite_basis(Q, L, p->sigma, p->basis);
  double gram = 0;
  for (int a = 0; a < L; ++a)
    for (int b = 0; b < L; ++b) {
      double s = 0;
      for (int m = 0; m < Q; ++m) s += p->basis[(size_t)m * L + a] * p->basis[(size_t)m * L + b];
      gram = std::max(gram, std::fabs(s - (a == b ? 1.0 : 0.0)));
    }
  if (gram > 1e-10) return bail(fail(WDD_E_ARG, "basis Gram error %.3g > 1e-10 (sigma %.4g px)", gram, p->sigma));

  // detector grid, aperture, active set in accumulator order
  std::vector<double> q(Q);
  for (int m = 0; m < Q; ++m) q[m] = (double)(m - Q / 2) * p->dq;
  ApertureRows ap = aperture(*p, q);
  std::vector<int32_t> act;
  active_set(*p, q, ap, act);
  std::sort(act.begin(), act.end(), [&](int32_t a, int32_t b) {
    const int ax = a % Sx, bx = b % Sx;
    return ax != bx ? ax < bx : a < b;
  });
  p->active_v = act;
  p->n_act = (int64_t)act.size();
  if (p->n_act == 0) return bail(fail(WDD_E_ARG, "empty active set"));
  p->act_vy.resize(act.size());
  for (size_t g = 0; g < act.size(); ++g) {
    const int vx = act[g] % Sx;
    p->act_vy[g] = act[g] / Sx;
    if (p->col_vx.empty() || p->col_vx.back() != vx) {
      p->col_vx.push_back(vx);
      p->col_off.push_back((int32_t)g);
    }
  }
  p->col_off.push_back((int32_t)act.size());
  p->n_vx = (int)p->col_vx.size();
  for (int j = 0; j < p->n_vx; ++j)
    for (int i0 = 0; i0 < p->col_off[j + 1] - p->col_off[j]; i0 += 32) p->flush_tiles.push_back(make_int2(j, i0));
  // Hermitian half plane: G[-v][k] = conj G[v][k] (real coefficients), so when the active set is
  // closed under v -> -v the FFT flush transforms only the columns vx <= Sx/2 (WDD_HALF=0: off)
  std::vector<int32_t> half_vx;
  std::vector<int2> half_map;
  {
    static const bool half_env = [] { const char* e = std::getenv("WDD_HALF"); return !(e && std::atoi(e) == 0); }();
    bool sym = half_env && rowfft_applies(*p);
    if (sym) {
      std::vector<bool> on((size_t)p->S, false);
      for (int32_t v : act) on[(size_t)v] = true;
      for (int32_t v : act) {
        const int vy = v / Sx, vx = v % Sx;
        if (!on[(size_t)((Sy - vy) % Sy) * Sx + (Sx - vx) % Sx]) { sym = false; break; }
      }
    }
    for (int j = 0; sym && j < p->n_vx; ++j) {
      const int vx = p->col_vx[j];
      if (2 * vx > Sx) continue;
      const int mvx = (Sx - vx) % Sx;
      int jm = -1;
      if (mvx != vx)
        jm = (int)(std::lower_bound(p->col_vx.begin(), p->col_vx.end(), mvx) - p->col_vx.begin());
      half_vx.push_back(vx);
      half_map.push_back(make_int2(j, jm));
    }
    if (sym) {
      p->n_vh = (int)half_vx.size();
      p->half_identity = true;       // primary columns vx = 0 .. n_vh - 1 (the row FFT needs no column table)
      for (int j = 0; j < p->n_vh; ++j) p->half_identity = p->half_identity && half_vx[j] == j;
    }
  }

  // twiddles
  std::vector<float2> Fx, Fy;
  twiddles(p->n_vx, p->col_vx.data(), Sx, Fx);
  std::vector<int32_t> ally(Sy);
  for (int v = 0; v < Sy; ++v) ally[v] = v;
  twiddles(Sy, ally.data(), Sy, Fy);
  std::vector<float2> twx, twy;
  fft_twiddles(Sx, twx);
  fft_twiddles(Sy, twy);

  // bank: built on the device once the column tables are there (below)
  ApertureIntervals apiv;
  if (!aperture_intervals(*p, ap, apiv)) return bail(fail(WDD_E_ARG, "aperture rows are not pixel intervals"));
  const size_t nW = (size_t)p->n_act * p->Kl;   // G and bank: this plan's coefficients only

  // device buffers
  std::vector<uint16_t> bpack;
  pack_basis_fp16(*p, bpack, p->b_scale);
  {
    // |T| <= max|I| * max_a sum_qx |Psi[qx][a]|; choose eT so T * 2^eT stays below 2^15 in fp16
    double colsum = 0;
    for (int a = 0; a < L; ++a) {
      double s = 0;
      for (int m = 0; m < Q; ++m) s += std::fabs(p->basis[(size_t)m * L + a]);
      colsum = std::max(colsum, s);
    }
    const double bound = (p->dtype == 0 ? 65535.0 : 65504.0) * colsum;
    const int eT = (int)std::floor(std::log2(32768.0 / bound));
    const int es = (int)std::lround(std::log2(p->b_scale));
    p->sc1 = std::ldexp(1.0, eT - es);
    p->sc2 = std::ldexp(1.0, -es - eT);
  }
  std::vector<float> psi32(p->basis.begin(), p->basis.end());
  std::vector<int32_t> vpos(act.begin(), act.end());
  std::vector<int32_t> iota(Sy);
  for (int i = 0; i < Sy; ++i) iota[i] = i;
  std::vector<int32_t> gidx((size_t)p->S, -1);
  for (size_t g = 0; g < act.size(); ++g) gidx[(size_t)act[g]] = (int32_t)g;
  if (gidx[0] < 0) return bail(fail(WDD_E_ARG, "v = 0 is not active (empty aperture?)"));
  p->g_dc = gidx[0];
  p->chunk_cap = 8192;
  p->mask_words = (Sx + 31) / 32;
  p->meta_slot_bytes = std::max((size_t)p->chunk_cap, (size_t)Sy * (1 + p->mask_words) + 4) * sizeof(int32_t);
  p->seen.assign((size_t)(p->S + 63) / 64, 0);
  p->row_dirty.assign(Sy, 0);
  p->row_staged.assign(Sy, 0);
  p->ingested.assign(p->o_only ? (size_t)Sy * p->mask_words : 0, 0u);
  p->pending.assign((size_t)Sy * p->mask_words, 0);

#define ALLOC(ptr, bytes)                                                                           \
  if (cudaMalloc((void**)&(ptr), (bytes)) != cudaSuccess)                                           \
    return bail(fail(WDD_E_NOMEM, "cudaMalloc(%s, %zu bytes) failed", #ptr, (size_t)(bytes)));
  ALLOC(p->d_Bpack, bpack.size() * 2);
  ALLOC(p->d_psi, psi32.size() * 4);
  ALLOC(p->d_Fx, Fx.size() * sizeof(float2));
  ALLOC(p->d_Fy, Fy.size() * sizeof(float2));
  ALLOC(p->d_twx, twx.size() * sizeof(float2));
  ALLOC(p->d_twy, twy.size() * sizeof(float2));
  ALLOC(p->d_col_vx, p->col_vx.size() * sizeof(int32_t));
  if (p->n_vh) {
    ALLOC(p->d_col_vx_half, half_vx.size() * sizeof(int32_t));
    ALLOC(p->d_half_map, half_map.size() * sizeof(int2));
  }
  ALLOC(p->d_W, nW * sizeof(float2));
  ALLOC(p->d_G, nW * sizeof(float2));
  if (p->combine == 1) ALLOC(p->d_Gsum, nW * sizeof(float2));
  ALLOC(p->d_R, (size_t)p->n_vx * Sy * p->Kl * sizeof(float2));
  // the two coefficient stores in one allocation (one IPC handle for peers of a shard group)
  const size_t c_store = (size_t)p->S * p->Kl;
  const int n_stores = (double_c_store() || nshard > 1) ? 2 : 1;
  ALLOC(p->d_Cbase, n_stores * c_store * sizeof(float));
  p->d_Call = p->d_Cbase;
  p->d_Call_alt = n_stores == 2 ? p->d_Cbase + c_store : nullptr;
  p->peer_base[p->shard] = p->d_Cbase;
  p->peers_ready = nshard == 1;
  ALLOC(p->d_act_vy, act.size() * 4);
  ALLOC(p->d_col_off, p->col_off.size() * 4);
  ALLOC(p->d_vpos, act.size() * 4);
  ALLOC(p->d_flush_tiles, p->flush_tiles.size() * sizeof(int2));
  ALLOC(p->d_o, act.size() * sizeof(float2));
  if (rgemm_prepare(*p) != cudaSuccess) return bail(fail(WDD_E_CUDA, "GEMM flush setup failed"));
  p->opart_cap = std::max({1, colfft_tiles_max(*p), flush_tiles(*p, 1 << 20), p->rg_ready ? flush_tiles(*p, 64, 3) : 1,
                           fused_possible(*p) ? fused_tiles(*p) : 1});
  ALLOC(p->d_opart, (size_t)p->opart_cap * act.size() * sizeof(float2));
  ALLOC(p->d_gidx, (size_t)p->S * sizeof(int32_t));
  ALLOC(p->d_oacc, act.size() * sizeof(float2));
  ALLOC(p->d_iota, (size_t)Sy * sizeof(int32_t));
  ALLOC(p->d_ones, (size_t)Sy * p->mask_words * sizeof(uint32_t));
  ALLOC(p->d_spec, (size_t)p->S * sizeof(float2));
  ALLOC(p->d_img_tmp, (size_t)p->S * sizeof(float2));
  ALLOC(p->d_err, sizeof(unsigned));
  ALLOC(p->d_meta, 2 * p->meta_slot_bytes);
#undef ALLOC
  if (cudaMallocHost(&p->h_meta, 2 * p->meta_slot_bytes) != cudaSuccess)
    return bail(fail(WDD_E_NOMEM, "pinned metadata buffer"));
  for (auto& e : p->meta_ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return bail(fail(WDD_E_CUDA, "event"));
  for (auto& e : p->stage_ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return bail(fail(WDD_E_CUDA, "event"));
  for (auto& e : p->copy_ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return bail(fail(WDD_E_CUDA, "event"));
  for (cudaEvent_t* e : {&p->ro_fork, &p->ro_last, &p->ro_done[0], &p->ro_done[1], &p->ro_fork_sync})
    if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return bail(fail(WDD_E_CUDA, "event"));
  if (p->readout_async && cudaStreamCreateWithFlags(&p->ro_stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(WDD_E_CUDA, "readout stream"));
  auto up = [&](void* d, const void* h, size_t b) { return cudaMemcpy(d, h, b, cudaMemcpyHostToDevice) == cudaSuccess; };
  bool ok = up(p->d_Bpack, bpack.data(), bpack.size() * 2) && up(p->d_psi, psi32.data(), psi32.size() * 4) &&
            up(p->d_Fx, Fx.data(), Fx.size() * sizeof(float2)) && up(p->d_Fy, Fy.data(), Fy.size() * sizeof(float2)) &&
            up(p->d_twx, twx.data(), twx.size() * sizeof(float2)) && up(p->d_twy, twy.data(), twy.size() * sizeof(float2)) &&
            up(p->d_col_vx, p->col_vx.data(), p->col_vx.size() * sizeof(int32_t)) &&
            (!p->n_vh || (up(p->d_col_vx_half, half_vx.data(), half_vx.size() * 4) &&
                          up(p->d_half_map, half_map.data(), half_map.size() * sizeof(int2)))) &&
            up(p->d_act_vy, p->act_vy.data(), act.size() * 4) &&
            up(p->d_col_off, p->col_off.data(), p->col_off.size() * 4) && up(p->d_vpos, vpos.data(), act.size() * 4) &&
            up(p->d_gidx, gidx.data(), gidx.size() * 4) && up(p->d_iota, iota.data(), iota.size() * 4) &&
            up(p->d_flush_tiles, p->flush_tiles.data(), p->flush_tiles.size() * sizeof(int2));
  ok = ok && cudaMemset(p->d_oacc, 0, act.size() * sizeof(float2)) == cudaSuccess &&
       cudaMemset(p->d_ones, 0xFF, (size_t)Sy * p->mask_words * sizeof(uint32_t)) == cudaSuccess &&
       cudaMemset(p->d_G, 0, nW * sizeof(float2)) == cudaSuccess &&
       cudaMemset(p->d_Cbase, 0, n_stores * c_store * sizeof(float)) == cudaSuccess &&
       cudaMemset(p->d_spec, 0, (size_t)p->S * sizeof(float2)) == cudaSuccess &&
       cudaMemset(p->d_err, 0, sizeof(unsigned)) == cudaSuccess;
  if (!ok) return bail(fail(WDD_E_CUDA, "upload failed: %s", cudaGetErrorString(cudaGetLastError())));
  if (nshard == 1) {
    const cudaError_t e = build_bank(*p, q.data(), apiv.rows.data(), apiv.ax_lo, apiv.n_axc, p->d_W, false);
    if (e != cudaSuccess) return bail(fail(WDD_E_CUDA, "bank build: %s", cudaGetErrorString(e)));
  } else {
    // the whole bank into scratch, then this shard's coefficient columns [k0, k0 + Kl)
    void* tmp = nullptr;
    cudaError_t e = cudaMalloc(&tmp, (size_t)p->n_act * K * sizeof(float2));
    if (e == cudaSuccess) e = build_bank(*p, q.data(), apiv.rows.data(), apiv.ax_lo, apiv.n_axc, tmp, false);
    if (e == cudaSuccess)
      e = cudaMemcpy2D(p->d_W, (size_t)p->Kl * sizeof(float2), static_cast<float2*>(tmp) + p->k0, (size_t)K * sizeof(float2),
                       (size_t)p->Kl * sizeof(float2), (size_t)p->n_act, cudaMemcpyDeviceToDevice);
    if (tmp) cudaFree(tmp);
    if (e != cudaSuccess) return bail(fail(WDD_E_CUDA, "bank build: %s", cudaGetErrorString(e)));
  }
  if (cufftPlan2d(&p->fft, Sy, Sx, CUFFT_C2C) != CUFFT_SUCCESS) return bail(fail(WDD_E_CUDA, "cufftPlan2d failed"));
  p->fft_ok = true;
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(WDD_E_CUDA, "plan upload sync failed"));
  *out = reinterpret_cast<wdd_plan_t>(p);
  return WDD_OK;
}

wdd_status wdd_destroy(wdd_plan_t plan) {
  free_plan(P(plan));
  return WDD_OK;
}

wdd_status wdd_ingest(wdd_plan_t plan, const void* frames_dev, const int32_t* scan_idx_host, int64_t n, void* stream) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (n < 0) return fail(WDD_E_ARG, "n < 0");
  if (n == 0) return WDD_OK;
  if (!frames_dev || !scan_idx_host) return fail(WDD_E_ARG, "NULL frames or indices");
  if (!p.peers_ready) return fail(WDD_E_STATE, "shard plan: wdd_set_shard_peers / wdd_link_shards first");
  CUDA_TRY(cudaSetDevice(p.device));
  // a call over a contiguous run of scan positions is one projection launch (no index upload):
  // each CTA then streams many frames, and its pipeline fill / drain is paid once per call
  // (Large: 0.70 -> see DESIGN.md); scattered indices go in chunks of the metadata slot size.
  // The host bookkeeping of a run is word-wise (validate_and_mark, mark_pending).
  const bool contiguous = is_run(scan_idx_host, n);
  wdd_status s = validate_and_mark(p, scan_idx_host, n, contiguous ? 1 : 0);
  if (s != WDD_OK) return s;
  use_stream(p, reinterpret_cast<cudaStream_t>(stream));
  const size_t fb = frame_bytes(p);
  const int64_t cap = contiguous ? std::max<int64_t>(p.chunk_cap, kMaxLaunchFrames) : p.chunk_cap;
  for (int64_t c0 = 0; c0 < n; c0 += cap) {
    const int64_t nc = std::min<int64_t>(cap, n - c0);
    s = enqueue_chunk(p, static_cast<const uint8_t*>(frames_dev) + (size_t)c0 * fb, scan_idx_host + c0, nc, c0 == 0,
                      contiguous ? 1 : -1);
    if (s != WDD_OK) return s;
  }
  p.frames_ingested += n;
  return WDD_OK;
}

wdd_status wdd_ingest_host(wdd_plan_t plan, const void* frames_host, const int32_t* scan_idx_host, int64_t n,
                           void* stream) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (n < 0) return fail(WDD_E_ARG, "n < 0");
  if (n == 0) return WDD_OK;
  if (!frames_host || !scan_idx_host) return fail(WDD_E_ARG, "NULL frames or indices");
  if (p.capturing) return fail(WDD_E_STATE, "wdd_ingest_host cannot be captured");
  if (!p.peers_ready) return fail(WDD_E_STATE, "shard plan: wdd_set_shard_peers / wdd_link_shards first");
  CUDA_TRY(cudaSetDevice(p.device));
  wdd_status s = validate_and_mark(p, scan_idx_host, n);
  if (s != WDD_OK) return s;
  use_stream(p, reinterpret_cast<cudaStream_t>(stream));
  const size_t fb = frame_bytes(p);
  const int64_t stage_frames = std::max<int64_t>(1, std::min<int64_t>(p.chunk_cap, (64ll << 20) / (int64_t)fb));
  if (!p.d_stage[0]) {
    CUDA_TRY(cudaMalloc(&p.d_stage[0], stage_frames * fb));
    CUDA_TRY(cudaMalloc(&p.d_stage[1], stage_frames * fb));
    CUDA_TRY(cudaStreamCreateWithFlags(&p.copy_stream, cudaStreamNonBlocking));
  }
  for (int64_t c0 = 0; c0 < n; c0 += stage_frames) {
    const int slot = p.stage_slot;
    p.stage_slot ^= 1;
    const int64_t nc = std::min<int64_t>(stage_frames, n - c0);
    CUDA_TRY(cudaStreamWaitEvent(p.copy_stream, p.stage_ev[slot], 0));  // previous user of the slot done
    CUDA_TRY(cudaMemcpyAsync(p.d_stage[slot], static_cast<const uint8_t*>(frames_host) + (size_t)c0 * fb, nc * fb,
                             cudaMemcpyHostToDevice, p.copy_stream));
    CUDA_TRY(cudaEventRecord(p.copy_ev[slot], p.copy_stream));
    CUDA_TRY(cudaStreamWaitEvent(p.stream, p.copy_ev[slot], 0));
    s = enqueue_chunk(p, p.d_stage[slot], scan_idx_host + c0, nc, true);   // (after a copy: no PDL overlap anyway)
    if (s != WDD_OK) return s;
    CUDA_TRY(cudaEventRecord(p.stage_ev[slot], p.stream));
  }
  // the H2D copies stay asynchronous: the plan stream waits for them, and the caller keeps the
  // host buffer valid until that stream has passed this call (as for device frames)
  p.frames_ingested += n;
  return WDD_OK;
}

wdd_status wdd_readout(wdd_plan_t plan, void* complex_out_dev) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (!complex_out_dev) return fail(WDD_E_ARG, "NULL output");
  CUDA_TRY(cudaSetDevice(p.device));
  RoScope ro(p);
  if (ro.status != WDD_OK) return ro.status;
  const float2* op = nullptr;
  int tiles = 0;
  wdd_status s = readout_spectrum(p, /*combine*/ true, &op, &tiles);
  if (s != WDD_OK) return s;
  Prof pr(p, kSlotFinalize, p.stream);
  CUDA_TRY(launch_finalize(p, op, tiles, static_cast<float2*>(complex_out_dev), p.stream));
  return WDD_OK;
}

wdd_status wdd_readout_spectrum(wdd_plan_t plan, void* spectrum_out_dev, int32_t combine) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (!spectrum_out_dev) return fail(WDD_E_ARG, "NULL output");
  CUDA_TRY(cudaSetDevice(p.device));
  RoScope ro(p);
  if (ro.status != WDD_OK) return ro.status;
  const float2* op = nullptr;
  int tiles = 0;
  wdd_status s = readout_spectrum(p, combine != 0, &op, &tiles);
  if (s != WDD_OK) return s;
  CUDA_TRY(cudaMemsetAsync(spectrum_out_dev, 0, (size_t)p.S * sizeof(float2), p.stream));
  CUDA_TRY(launch_spectrum(p, op, tiles, static_cast<float2*>(spectrum_out_dev), p.stream));
  return WDD_OK;
}

wdd_status wdd_image_from_spectrum(wdd_plan_t plan, const void* spectrum_dev, void* complex_out_dev) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (!spectrum_dev || !complex_out_dev) return fail(WDD_E_ARG, "NULL buffer");
  if (spectrum_dev == complex_out_dev) return fail(WDD_E_ARG, "spectrum and image must not alias");
  CUDA_TRY(cudaSetDevice(p.device));
  RoScope ro(p);
  if (ro.status != WDD_OK) return ro.status;
  Prof pr(p, kSlotFinalize, p.stream);
  CUDA_TRY(launch_image(p, static_cast<const float2*>(spectrum_dev), static_cast<float2*>(complex_out_dev), p.stream));
  return WDD_OK;
}

wdd_status wdd_ingest_remote(wdd_plan_t plan, const int32_t* scan_idx_host, int64_t n) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (n < 0) return fail(WDD_E_ARG, "n < 0");
  if (n == 0) return WDD_OK;
  if (!scan_idx_host) return fail(WDD_E_ARG, "NULL indices");
  if (p.nshard == 1) return fail(WDD_E_STATE, "wdd_ingest_remote needs a shard plan (opts.k_shards > 1)");
  wdd_status s = validate_and_mark(p, scan_idx_host, n);
  if (s != WDD_OK) return s;
  mark_pending(p, scan_idx_host, n);
  p.frames_ingested += n;
  return WDD_OK;
}

wdd_status wdd_shard_store_handle(wdd_plan_t plan, uint8_t handle[64]) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (!handle) return fail(WDD_E_ARG, "NULL handle");
  if (p.nshard == 1) return fail(WDD_E_STATE, "not a shard plan");
  CUDA_TRY(cudaSetDevice(p.device));
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
  CUDA_TRY(cudaIpcGetMemHandle(&h, p.d_Cbase));
  std::memcpy(handle, &h, 64);
  return WDD_OK;
}

wdd_status wdd_set_shard_peers(wdd_plan_t plan, int32_t nshard, int32_t rank, const uint8_t* handles) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (!handles) return fail(WDD_E_ARG, "NULL handles");
  if (p.nshard == 1 || nshard != p.nshard || rank != p.shard)
    return fail(WDD_E_ARG, "shard group (%d, %d) does not match the plan's (%d, %d)", nshard, rank, p.nshard, p.shard);
  CUDA_TRY(cudaSetDevice(p.device));
  for (int o = 0; o < nshard; ++o) {
    if (o == p.shard) continue;
    if (p.peers_ipc[o] && p.peer_base[o]) cudaIpcCloseMemHandle(p.peer_base[o]);
    p.peers_ipc[o] = false;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + 64 * (size_t)o, 64);
    void* d = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&d, h, cudaIpcMemLazyEnablePeerAccess));
    p.peer_base[o] = static_cast<float*>(d);
    p.peers_ipc[o] = true;
  }
  p.peers_ready = true;
  return WDD_OK;
}

wdd_status wdd_link_shards(int32_t nshard, const wdd_plan_t* plans) {
  if (!plans || nshard < 2 || nshard > kMaxShards) return fail(WDD_E_ARG, "need 2..%d plans", kMaxShards);
  for (int r = 0; r < nshard; ++r) {
    const Plan* q = P(plans[r]);
    const Plan* q0 = P(plans[0]);
    if (!q || q->nshard != nshard || q->shard != r || q->S != q0->S || q->L != q0->L || q->Q != q0->Q)
      return fail(WDD_E_ARG, "plan %d is not shard %d of %d of the same geometry", r, r, nshard);
  }
  for (int r = 0; r < nshard; ++r) {
    Plan& q = *P(plans[r]);
    CUDA_TRY(cudaSetDevice(q.device));
    for (int o = 0; o < nshard; ++o) {
      const Plan& po = *P(plans[o]);
      if (po.device != q.device) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(po.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          return fail(WDD_E_CUDA, "peer access %d -> %d: %s", q.device, po.device, cudaGetErrorString(e));
        cudaGetLastError();
      }
      q.peer_base[o] = po.d_Cbase;
      q.peers_ipc[o] = false;
    }
    q.peers_ready = true;
  }
  return WDD_OK;
}

wdd_status wdd_readout_host(wdd_plan_t plan, void* complex_out_host) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (!complex_out_host) return fail(WDD_E_ARG, "NULL output");
  if (p.capturing) return fail(WDD_E_STATE, "wdd_readout_host cannot be captured");
  CUDA_TRY(cudaSetDevice(p.device));
  void* d = nullptr;
  CUDA_TRY(cudaMallocAsync(&d, (size_t)p.S * sizeof(float2), p.stream));
  wdd_status s = wdd_readout(plan, d);
  if (s == WDD_OK) {
    CUDA_TRY(wait_if(p.stream, p.ro_last, p.readout_async && p.ro_last_valid));
    CUDA_TRY(cudaMemcpyAsync(complex_out_host, d, (size_t)p.S * sizeof(float2), cudaMemcpyDeviceToHost, p.stream));
  }
  cudaFreeAsync(d, p.stream);
  CUDA_TRY(cudaStreamSynchronize(p.stream));
  if (s == WDD_OK && p.dtype == 1) s = wdd_check(plan);   // (host readout synchronises anyway)
  return s;
}

wdd_status wdd_get_accumulator(wdd_plan_t plan, void* G_out_dev, int32_t* active_v_host, int64_t* n_act) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  CUDA_TRY(cudaSetDevice(p.device));
  if (n_act) *n_act = p.n_act;
  if (active_v_host) std::memcpy(active_v_host, p.active_v.data(), p.active_v.size() * 4);
  if (G_out_dev) {
    RoScope ro(p);
    if (ro.status != WDD_OK) return ro.status;
    wdd_status s = shard_barrier(p);
    if (s == WDD_OK) s = flush(p);
    if (s == WDD_OK) s = materialize_G(p);
    if (s != WDD_OK) return s;
    CUDA_TRY(cudaMemcpyAsync(G_out_dev, p.d_G, (size_t)p.n_act * p.Kl * sizeof(float2), cudaMemcpyDeviceToDevice, p.stream));
  }
  return WDD_OK;
}

wdd_status wdd_reset(wdd_plan_t plan) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  CUDA_TRY(cudaSetDevice(p.device));
  p.G_zero = true;          // the next flush writes G instead of accumulating (no clearing pass)
  // (pipelined readouts: the running spectrum below, and a single coefficient store, are still
  // read by the last readout)
  if (p.readout_async && (p.o_only || !p.d_Call_alt)) CUDA_TRY(wait_if(p.stream, p.ro_last, p.ro_last_valid));
  if (p.o_only) CUDA_TRY(cudaMemsetAsync(p.d_oacc, 0, (size_t)p.n_act * sizeof(float2), p.stream));
  std::fill(p.ingested.begin(), p.ingested.end(), 0u);
  p.opart_tiles = 0;
  // coefficients of frames ingested but never flushed are simply forgotten: only pending
  // positions are ever read from the coefficient store
  std::fill(p.seen.begin(), p.seen.end(), 0);
  std::fill(p.row_dirty.begin(), p.row_dirty.end(), 0);
  std::fill(p.row_staged.begin(), p.row_staged.end(), 0);
  std::fill(p.pending.begin(), p.pending.end(), 0u);
  if (p.d_Call_alt && p.frames_ingested > 0) {
    // shard groups: the store this acquisition is about to write (on every rank) was read by the
    // row transforms of the acquisition before the previous one; without a readout barrier in the
    // previous acquisition, one here orders those reads before any rank's next projection
    if (p.nshard > 1 && !p.barrier_since_swap) {
      wdd_status s = shard_barrier(p);
      if (s != WDD_OK) return s;
    }
    p.barrier_since_swap = false;
    // the previous acquisition's flush / readout may still read the current store: the next
    // acquisition writes the other one, so its first projection need not wait for them.  That
    // store was last read by the row transform of the acquisition before the previous one; the
    // first projection may overlap (PDL) the previous readout only if a row transform of the
    // previous acquisition lies in between: that launch is ordered after every earlier read of C
    // (a PDL-launched row FFT triggers its dependents only after its own C loads, an ordinary
    // launch starts after all earlier work), and the projection is downstream of it
    std::swap(p.d_Call, p.d_Call_alt);
    p.store_par ^= 1;
    // pipelined readouts: the store swapped in is free once the last readout that read it is done
    if (p.readout_async) CUDA_TRY(wait_if(p.stream, p.ro_done[p.store_par], p.ro_done_valid[p.store_par]));
    p.c_fresh = p.c_read_since_swap;
    p.c_read_since_swap = false;
  }
  p.frames_ingested = 0;
  p.frames_enqueued = 0;
  return WDD_OK;
}

wdd_status wdd_nccl_get_unique_id(uint8_t id[128]) {
  if (!id) return fail(WDD_E_ARG, "NULL id");
  ncclUniqueId u;
  NCCL_TRY(ncclGetUniqueId(&u));
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
  return WDD_OK;
}

wdd_status wdd_set_comm(wdd_plan_t plan, int32_t nranks, int32_t rank, const uint8_t id[128]) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (nranks < 1 || rank < 0 || rank >= nranks || !id) return fail(WDD_E_ARG, "bad nranks/rank/id");
  CUDA_TRY(cudaSetDevice(p.device));
  if (p.nccl) {
    ncclCommDestroy(reinterpret_cast<ncclComm_t>(p.nccl));
    p.nccl = nullptr;
  }
  p.nranks = nranks;
  p.rank = rank;
  // (a one-rank communicator too: the combine path then runs exactly as on N ranks)
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t c;
  NCCL_TRY(ncclCommInitRank(&c, nranks, u, rank));
  p.nccl = c;
  return WDD_OK;
}

wdd_status wdd_get_info(wdd_plan_t plan, wdd_plan_info* info) {
  if (check_plan(plan)) return WDD_E_ARG;
  if (!info) return fail(WDD_E_ARG, "NULL info");
  const Plan& p = *P(plan);
  wdd_plan_info i{};
  i.Sy = p.Sy; i.Sx = p.Sx; i.Q = p.Q; i.L = p.L; i.K = p.K; i.n_vx = p.n_vx; i.dtype = p.dtype;
  i.normalize = p.normalize; i.n_act = p.n_act; i.dq = p.dq; i.q_alpha = p.qa; i.R_px = p.R;
  i.sigma_px = p.sigma; i.wavelength_A = p.lambda; i.step_A = p.step; i.eps = p.eps;
  i.bytes_G = p.n_act * p.Kl * 8; i.bytes_bank = i.bytes_G; i.bytes_R = (int64_t)p.n_vx * p.Sy * p.Kl * 8;
  i.bytes_C = p.S * p.Kl * 4; i.frames_ingested = p.frames_ingested; i.nranks = p.nranks; i.rank = p.rank;
  i.proj_ctas_per_sm = project_occupancy(p);
  i.k_shards = p.nshard; i.k_rank = p.shard; i.k_lo = p.k0; i.k_count = p.Kl;
  i.n_vh = p.n_vh;
  *info = i;
  return WDD_OK;
}

wdd_status wdd_get_tables(wdd_plan_t plan, double* basis, double* bank, int32_t* active_v) {
  if (check_plan(plan)) return WDD_E_ARG;
  const Plan& p = *P(plan);
  if (basis) std::memcpy(basis, p.basis.data(), p.basis.size() * sizeof(double));
  if (active_v) std::memcpy(active_v, p.active_v.data(), p.active_v.size() * 4);
  if (bank) {   // the same device build as the plan's bank, in complex128
    std::vector<double> q(p.Q);
    for (int m = 0; m < p.Q; ++m) q[m] = (double)(m - p.Q / 2) * p.dq;
    ApertureIntervals apiv;
    if (!aperture_intervals(p, aperture(p, q), apiv)) return fail(WDD_E_ARG, "aperture rows are not pixel intervals");
    CUDA_TRY(cudaSetDevice(p.device));
    void* d = nullptr;
    const size_t bytes = (size_t)p.n_act * p.K * 2 * sizeof(double);
    CUDA_TRY(cudaMalloc(&d, bytes));
    cudaError_t e = build_bank(p, q.data(), apiv.rows.data(), apiv.ax_lo, apiv.n_axc, d, true);
    if (e == cudaSuccess) e = cudaMemcpy(bank, d, bytes, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return fail(WDD_E_CUDA, "bank build: %s", cudaGetErrorString(e));
  }
  return WDD_OK;
}

wdd_status wdd_full_wdd(wdd_plan_t plan, const void* frames_dev, void* complex_out_dev, void* stream) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (!frames_dev || !complex_out_dev) return fail(WDD_E_ARG, "NULL buffer");
  if (p.capturing) return fail(WDD_E_STATE, "wdd_full_wdd cannot be captured");
  CUDA_TRY(cudaSetDevice(p.device));
  use_stream(p, reinterpret_cast<cudaStream_t>(stream));
  char msg[256] = {0};
  const wdd_status s = full_wdd(p, frames_dev, complex_out_dev, msg, sizeof msg);
  if (s != WDD_OK) return fail(s, "%s", msg);
  return WDD_OK;
}

wdd_status wdd_project(wdd_plan_t plan, const void* frames_dev, int64_t n, void* C_out_dev, void* stream) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (n < 0 || (n > 0 && (!frames_dev || !C_out_dev))) return fail(WDD_E_ARG, "bad arguments");
  CUDA_TRY(cudaSetDevice(p.device));
  Prof pr(p, kSlotProject, reinterpret_cast<cudaStream_t>(stream));
  ProjDst d;
  d.C[0] = static_cast<float*>(C_out_dev);
  d.K[0] = p.K;
  d.alo[1] = p.L;
  CUDA_TRY(launch_project(p, frames_dev, n, d, nullptr, 0, reinterpret_cast<cudaStream_t>(stream),
                          /*wait_start*/ true));
  return WDD_OK;
}

wdd_status wdd_profile_enable(wdd_plan_t plan, int32_t enable) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  p.prof = enable != 0;
  p.prof_marks.clear();
  p.ev_used = 0;
  return WDD_OK;
}

wdd_status wdd_profile_read(wdd_plan_t plan, int32_t slot, double* ms_total, int64_t* count) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (slot < 0 || slot >= kNumSlots) return fail(WDD_E_ARG, "bad slot");
  double ms = 0;
  int64_t c = 0;
  for (auto& m : p.prof_marks) {
    if (m.first != slot) continue;
    CUDA_TRY(cudaEventSynchronize(p.ev_pool[m.second + 1]));
    float t = 0;
    CUDA_TRY(cudaEventElapsedTime(&t, p.ev_pool[m.second], p.ev_pool[m.second + 1]));
    ms += t;
    ++c;
  }
  if (ms_total) *ms_total = ms;
  if (count) *count = c;
  return WDD_OK;
}

wdd_status wdd_launch_count(wdd_plan_t plan, int64_t* count, int32_t reset) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (count) *count = p.launches;
  if (reset) p.launches = 0;
  return WDD_OK;
}

wdd_status wdd_capture_begin(wdd_plan_t plan, void* stream) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (p.capturing) return fail(WDD_E_STATE, "already capturing");
  if (stream == nullptr || reinterpret_cast<cudaStream_t>(stream) == cudaStreamLegacy ||
      reinterpret_cast<cudaStream_t>(stream) == cudaStreamPerThread)
    return fail(WDD_E_ARG, "capture needs a created (non-default) stream");
  CUDA_TRY(cudaSetDevice(p.device));
  if (!p.cap_host) {
    p.cap_bytes = 16u << 20;
    CUDA_TRY(cudaMallocHost(&p.cap_host, p.cap_bytes));
    CUDA_TRY(cudaMalloc(&p.cap_dev, p.cap_bytes));
  }
  use_stream(p, reinterpret_cast<cudaStream_t>(stream));
  CUDA_TRY(cudaStreamSynchronize(p.stream));
  if (p.ro_stream) CUDA_TRY(cudaStreamSynchronize(p.ro_stream));
  p.ro_last_valid = p.ro_done_valid[0] = p.ro_done_valid[1] = false;   // (eager readouts all done)
  CUDA_TRY(cudaStreamBeginCapture(p.stream, cudaStreamCaptureModeThreadLocal));
  p.capturing = true;
  return WDD_OK;
}

wdd_status wdd_capture_end(wdd_plan_t plan, int64_t* graph_handle) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (!p.capturing) return fail(WDD_E_STATE, "not capturing");
  p.capturing = false;
  // join the readout stream's captured work (a capture must end with every forked stream joined;
  // a replay of the graph therefore completes only after its last readout)
  const cudaError_t je = wait_if(p.stream, p.ro_last, p.readout_async && p.ro_last_valid);
  p.ro_last_valid = p.ro_done_valid[0] = p.ro_done_valid[1] = false;
  cudaGraph_t g = nullptr;
  const cudaError_t ee = cudaStreamEndCapture(p.stream, &g);
  CUDA_TRY(je);
  CUDA_TRY(ee);
  cudaGraphExec_t ex = nullptr;
  cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  CUDA_TRY(e);
  p.graphs.push_back(ex);
  if (graph_handle) *graph_handle = (int64_t)p.graphs.size() - 1;
  return WDD_OK;
}

wdd_status wdd_graph_launch(wdd_plan_t plan, int64_t graph_handle, void* stream) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (p.capturing) return fail(WDD_E_STATE, "graph launch while capturing");
  if (graph_handle < 0 || graph_handle >= (int64_t)p.graphs.size()) return fail(WDD_E_ARG, "bad graph handle");
  CUDA_TRY(cudaSetDevice(p.device));
  use_stream(p, reinterpret_cast<cudaStream_t>(stream));
  // (a replayed acquisition may swap in the store an eager readout still reads)
  CUDA_TRY(wait_if(p.stream, p.ro_last, p.readout_async && p.ro_last_valid));
  CUDA_TRY(cudaGraphLaunch(p.graphs[(size_t)graph_handle], p.stream));
  return WDD_OK;
}

wdd_status wdd_check(wdd_plan_t plan) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (p.capturing) return fail(WDD_E_STATE, "wdd_check cannot be captured");
  CUDA_TRY(cudaSetDevice(p.device));
  CUDA_TRY(cudaStreamSynchronize(p.stream));
  if (p.ro_stream) CUDA_TRY(cudaStreamSynchronize(p.ro_stream));
  unsigned f = 0;
  CUDA_TRY(cudaMemcpy(&f, p.d_err, sizeof f, cudaMemcpyDeviceToHost));
  if (f) {
    CUDA_TRY(cudaMemset(p.d_err, 0, sizeof f));
    return fail(WDD_E_RANGE, "float32 frames with values the fp16 hi/lo split cannot hold (|x| > 65504 or not "
                "finite) were ingested since the last check; their coefficients are not valid");
  }
  return WDD_OK;
}

wdd_status wdd_sync(wdd_plan_t plan) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  CUDA_TRY(cudaSetDevice(p.device));
  CUDA_TRY(cudaStreamSynchronize(p.stream));
  if (p.copy_stream) CUDA_TRY(cudaStreamSynchronize(p.copy_stream));
  if (p.ro_stream) CUDA_TRY(cudaStreamSynchronize(p.ro_stream));
  return WDD_OK;
}

wdd_status wdd_readout_wait(wdd_plan_t plan, void* stream) {
  if (check_plan(plan)) return WDD_E_ARG;
  Plan& p = *P(plan);
  if (p.capturing) return fail(WDD_E_STATE, "wdd_readout_wait cannot be captured");
  CUDA_TRY(cudaSetDevice(p.device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (p.readout_async && p.ro_last_valid) {
    CUDA_TRY(cudaStreamWaitEvent(st, p.ro_last, 0));
  } else if (st != p.stream) {
    // synchronous readouts (or a replayed graph, whose readouts joined the plan stream): order
    // `stream` after the plan stream
    CUDA_TRY(cudaEventRecord(p.ro_fork_sync, p.stream));
    CUDA_TRY(cudaStreamWaitEvent(st, p.ro_fork_sync, 0));
  }
  return WDD_OK;
}

}  // extern "C"
