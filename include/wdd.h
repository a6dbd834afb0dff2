/*
 * wdd.h -- C ABI of libwdd, the B200 (sm_100a) hot path of Live Wigner Distribution
 * Deconvolution (Bangun et al., arXiv 2212.01309; /root/reference/PAPER.md cited as P:line).
 *
 * The library implements the data-parallel hot path of the paper's Algorithm 2
 * (`Algo:ModifiedWDD`) with the Wiener step deferred to readout (exact by
 * linearity):
 *   ingest : per frame, the Hermite-Gauss projection H(I_s) = psi_x^T I_s^T psi_y
 *            (P:359-364), then the scan-frequency accumulation G[v,k] += f_s[v] * vec(H(I_s))[k]
 *            of eq:outer_prod, in the separable form F_2D = F_y (x) F_x:
 *            a 1-D DFT along each scan row, staged, and a phase-weighted rank update along y.
 *   readout: o_v = sum_k G[v,k] * K_v[k]  with the pre-computed Wiener bank
 *            K_v = conj(H(Y_v)) / (|H(Y_v)|^2 + eps) (Algorithm 1),
 *            then O = conj(F^{-1} o), optionally / sqrt(o_0) (eq:extract).
 *
 * Conventions (DESIGN.md §3 lists every reading of the paper these rest on):
 *   scan index  s = sy*Sx + sx, row-major, y outer.  Scan step Delta (Angstrom), square grid.
 *   frames      n x Q x Q row-major, DC at pixel (Q/2, Q/2), uint16 counts or float32.
 *   basis       Psi[m,n] = psi_n((m - Q/2)/sigma)/sqrt(sigma), normalised Hermite functions,
 *               sigma = sqrt(Q/(2 pi)) px unless overridden; coefficient k = a*L + b with
 *               a = n_x (detector column order) and b = n_y.
 *   scan freq   v = vy*Sx + vx in FFT order, q_hat_v = (v~y/(Sy*Delta), v~x/(Sx*Delta)).
 *   DFTs        unitary (1/sqrt(Sy*Sx) overall), forward e^{-i 2 pi ...}.
 *   active set  v with Y_v not identically 0 (exact discrete overlap test); G and
 *               the bank store only active v, in "accumulator order": sorted by (vx, vy).
 *
 * Threading / streams: a plan is externally synchronised (one host thread at a time).  All
 * device work of a plan is ordered on the stream passed to the most recent wdd_ingest (or the
 * legacy default stream before the first ingest); readout and accessors run on that stream.
 * Nothing here throws; every call returns wdd_status and sets a thread-local message.
 */
#ifndef WDD_H_
#define WDD_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  WDD_OK = 0,
  WDD_E_ARG = 1,     /* invalid argument / unsupported shape; nothing was enqueued           */
  WDD_E_RANGE = 2,   /* a scan index outside [0, Sy*Sx); the whole call was rejected          */
  WDD_E_DUP = 3,     /* a scan index ingested before or repeated in the call; call rejected   */
  WDD_E_NOMEM = 4,   /* device or pinned-host allocation failed                               */
  WDD_E_CUDA = 5,    /* a CUDA runtime / cuFFT error (message in wdd_last_error())            */
  WDD_E_NCCL = 6,    /* an NCCL error                                                         */
  WDD_E_STATE = 7    /* call not valid in the plan's current state                            */
} wdd_status;

typedef struct wdd_plan* wdd_plan_t;

/* Probe of the north-star ABI: p_hat(q) = 1[|q| <= alpha/lambda] exp(-i pi lambda df |q|^2). */
typedef struct {
  double wavelength_A;   /* electron wavelength lambda, Angstrom (> 0)                        */
  double semiangle_rad;  /* aperture semi-angle alpha, rad (> 0)                              */
  double defocus_A;      /* defocus df, Angstrom                                              */
} wdd_probe;

typedef struct {
  double det_px_rad;     /* detector pixel in rad; 0 => dq = 1/(Q*Delta) (real pixel = step)  */
  double sigma_px;       /* Hermite-Gauss width in px; 0 => sqrt(Q/(2 pi))                    */
  int32_t dtype;         /* frame dtype: 0 = uint16 counts, 1 = float32 (|x| <= 65504)        */
  int32_t normalize;     /* 0 = literal Algorithm 2 output, 1 = divide by sqrt(o_0)*/
  int32_t device;        /* CUDA device ordinal; the plan's buffers live there                */
  int32_t combine;       /* multi-rank readout: 0 = allreduce o (default), 1 = allreduce G    */
  int32_t accumulator;   /* 0 = G(q,k) materialised and updated at every flush (north star);
                            1 = spectrum only: each flush adds its increment of the
                            Wiener readout o_v = sum_k G[v,k] K_v[k] (linear in G) to a running o
                            and never reads or writes G; wdd_get_accumulator forms G on demand
                            from the coefficient store (one full row DFT + rank update).  Needs a
                            power-of-two Sy in [2, 1024]; multi-rank readout always sums o
                            (combine is ignored).                                               */
  int32_t ingest_overlap;/* 0 (default) = wdd_ingest may follow a caller kernel that writes the frames:
                            the first projection of each call reads them only after the preceding
                            grid on the stream has completed.  1 = the caller guarantees the frames
                            are complete before the previous LIBRARY call on the stream was enqueued
                            (or arrive by a copy / event): every projection launch then streams its
                            frames while the previous one drains (PDL), which is what keeps a chain
                            of small batches at HBM speed.                                        */
  int32_t k_shards;      /* coefficient sharding over a rank group: 0 or 1 = none;
                            n > 1 = this plan owns the coefficient rows a (k = a*L + b) of shard
                            k_rank of n (contiguous, as even as possible, n <= L) -- its coefficient
                            store, R staging, G and bank hold only those k; see wdd_set_shard_peers */
  int32_t k_rank;        /* this plan's shard, 0 <= k_rank < k_shards                              */
  int32_t ingest_spread; /* 0 (default) = throughput grid: ~0.5-1 MiB of frames per projection CTA,
                            so consecutive (PDL-chained) batches stream side by side on the SMs;
                            1 = latency grid: every launch spread over all SMs (a lone batch on an
                            idle GPU finishes sooner; chained small batches lose overlap)          */
  int32_t readout_async; /* 0 (default) = readouts run on the plan stream.  1 = pipelined acquisitions:
                            wdd_readout / wdd_readout_spectrum / wdd_get_accumulator /
                            wdd_image_from_spectrum run on the plan's own readout stream, which first
                            waits for everything enqueued on the plan stream so far; the plan stream
                            goes on with the next ingests (the next acquisition, in the other
                            coefficient store) while the readout runs.  The output is valid once
                            wdd_readout_wait has ordered a stream after it (or after wdd_sync).  The
                            library orders its own hazards: a reset waits for the last readout of the
                            store it swaps in (spectrum-only plans: for the last readout), and
                            consecutive readouts share the readout stream (with a communicator, so do
                            all of the plan's collectives).  Not in a shard group (its reset barrier
                            is a collective on the plan stream): WDD_E_STATE at create.            */
  int32_t reserved[1];   /* must be zero                                                      */
} wdd_plan_opts;

/* Plan creation (host, blocking): derives dq, R, sigma; computes in float64 the basis Psi,
 * the twiddles F_y / F_x, the exact active set and the Wiener bank (Algorithm 1);
 * allocates and uploads every device buffer (basis, twiddles, bank, G, row staging, cuFFT plan).
 *   scan_shape = {Sy, Sx} (>= 2 each); det_shape = {Q, Q} with Q in {32, 64, 128, 256};
 *   K = L*L with L a multiple of 8, 8 <= L <= 32, L <= Q; wiener_eps > 0; step_A > 0.
 *   opts may be NULL (all defaults).  On success *out owns all plan memory.
 * Errors: WDD_E_ARG (shapes, K not a supported square, eps <= 0, basis Gram error > 1e-10),
 *         WDD_E_NOMEM, WDD_E_CUDA. */
wdd_status wdd_plan_create(const int32_t scan_shape[2], double step_A, const int32_t det_shape[2],
                           int32_t K, const wdd_probe* probe, double wiener_eps,
                           const wdd_plan_opts* opts, wdd_plan_t* out);

/* Ingest n frames (stream-ordered, asynchronous; Algorithm 2 loop body P:514-518 + eq:outer_prod).
 *   frames_dev     caller-owned DEVICE buffer, n x Q x Q in the plan dtype, contiguous; it must
 *                  stay valid until `stream` has passed this call.
 *   scan_idx_host  HOST array of n scan indices, read synchronously (may be freed on return).
 *   stream         cudaStream_t (0 = legacy default stream).
 * The whole call is validated before anything is enqueued: WDD_E_RANGE / WDD_E_DUP reject it
 * with no effect (so live ingestion in any partition/order equals offline).
 * n == 0 is a no-op. */
wdd_status wdd_ingest(wdd_plan_t plan, const void* frames_dev, const int32_t* scan_idx_host,
                      int64_t n, void* stream);

/* Same as wdd_ingest for frames in HOST memory (pinned for asynchronous copies): the library
 * copies them through double-buffered device staging on its own copy stream, so the H2D copy of
 * one chunk overlaps the projection of the previous one.  Stream-ordered like wdd_ingest: the
 * host buffer must stay valid (and unmodified) until `stream` has passed this call. */
wdd_status wdd_ingest_host(wdd_plan_t plan, const void* frames_host, const int32_t* scan_idx_host,
                           int64_t n, void* stream);

/* Readout (non-mutating w.r.t. the ingested set; valid at any time):
 * flush staged rows into G, o_v = sum_k G[v,k] K_v[k] for active v (0 elsewhere), multi-rank
 * combine, O = conj(IDFT2_unitary(o)) [/ sqrt(o_0)].
 *   complex_out_dev  DEVICE buffer of Sy*Sx interleaved float2 (complex64), row-major [sy][sx].
 * Enqueued on the plan stream (opts.readout_async: on the readout stream, see wdd_readout_wait);
 * the caller synchronises that stream before reading.
 * Multi-rank (after wdd_set_comm) this is collective: every rank must call it, and every rank
 * receives the same image.  Two readouts with no ingest in between give identical bytes. */
wdd_status wdd_readout(wdd_plan_t plan, void* complex_out_dev);

/* Order `stream` (cudaStream_t, 0 = legacy default stream) after the plan's latest readout-family
 * call, so work enqueued there may read its output.  With opts.readout_async = 0 the readouts are
 * already on the plan stream and this only orders `stream` after the plan stream.  Never blocks
 * the host. */
wdd_status wdd_readout_wait(wdd_plan_t plan, void* stream);

/* The readout's spectrum instead of the image: o_v = sum_k G[v,k] K_v[k] at the active v, 0
 * elsewhere (Sy*Sx complex64, image order v = vy*Sx + vx, FFT order per axis), DEVICE buffer.
 * combine != 0: after the multi-rank NCCL combine (collective, as wdd_readout); combine == 0: this
 * rank's own partial spectrum (no communication) -- partial spectra of disjoint ingests (or of
 * coefficient shards) sum to the full one (linearity).  Stream-ordered. */
wdd_status wdd_readout_spectrum(wdd_plan_t plan, void* spectrum_out_dev, int32_t combine);

/* The final transform of a given spectrum: O = conj(IDFT2_unitary(o)) [/ sqrt(o_0)];
 * spectrum_dev and complex_out_dev are DEVICE buffers of Sy*Sx complex64 (must not alias). */
wdd_status wdd_image_from_spectrum(wdd_plan_t plan, const void* spectrum_dev, void* complex_out_dev);

/* Synchronise the plan stream and report deferred device-side errors: WDD_E_RANGE if float32
 * frames with values the projection's fp16 hi/lo split cannot represent (|x| > 65504, inf, NaN)
 * were ingested since the last check (the flag is then cleared).  wdd_readout_host checks too. */
wdd_status wdd_check(wdd_plan_t plan);

/* Readout into a HOST buffer (Sy*Sx complex64); blocks until the bytes are on the host. */
wdd_status wdd_readout_host(wdd_plan_t plan, void* complex_out_host);

/* Release every resource of the plan (synchronises its stream first).  NULL is a no-op. */
wdd_status wdd_destroy(wdd_plan_t plan);

/* Flush staged rows and copy this rank's accumulator G (n_act x K complex64, accumulator order;
 * shard plans: n_act x k_count, their coefficients only) into G_out_dev (DEVICE, may be NULL) and
 * the active list (flattened v = vy*Sx + vx, int32, in the same order) into active_v_host (HOST,
 * may be NULL).  *n_act receives n_act.  Collective in a shard group with a communicator. */
wdd_status wdd_get_accumulator(wdd_plan_t plan, void* G_out_dev, int32_t* active_v_host,
                               int64_t* n_act);

/* Forget every ingested frame: G = 0, staging cleared, seen-bitmap cleared (stream-ordered).
 * After ingests it also swaps the plan's two coefficient stores (2 x S x K float32, allocated at
 * create; WDD_C_DOUBLE=0 allocates one), so the next acquisition's first projection may overlap
 * the previous acquisition's readout, which still reads the old store.  Device work: none
 * (spectrum-only plans: one memset of the running spectrum). */
wdd_status wdd_reset(wdd_plan_t plan);

/* Multi-rank combine over NCCL (NVLink / NVSwitch).  Rank 0 creates the id, the caller
 * broadcasts it (e.g. via torch.distributed), every rank calls wdd_set_comm with it.
 * Each rank ingests a disjoint index set; wdd_readout allreduces (opts.combine) and every
 * rank receives the full image ("merge ... sums up the contributions").
 * nranks == 1 creates a one-rank communicator: the readout then runs the combine path (partial
 * readouts summed into o, allreduce) exactly as on N ranks.  Calling it again replaces the comm. */
wdd_status wdd_nccl_get_unique_id(uint8_t id[128]);
wdd_status wdd_set_comm(wdd_plan_t plan, int32_t nranks, int32_t rank, const uint8_t id[128]);

/* ----------------------- coefficient-sharded rank groups -----------------------
 * A plan created with opts.k_shards = n > 1, opts.k_rank = r owns the coefficient rows a in
 * [floor(r L / n), floor((r+1) L / n)) of H(I) (k = a*L + b): its coefficient store, row staging R,
 * accumulator G and Wiener bank hold only those k_count = (a1 - a0) L coefficients.  Every rank
 * ingests its own frames (any partition of the scan: contiguous rows, round-robin batches) and the
 * projection kernel stores each frame's coefficient rows of shard o straight into rank o's store
 * (peer memory over NVLink / NVSwitch: the exchange is fused into the projection's epilogue, about
 * 4K (n-1)/n bytes per frame against the frame's 2 Q^2).  At readout every rank flushes and reads
 * out its own coefficients over the whole scan, o_v = sum_{k in shard} G[v,k] K_v[k], and the NCCL
 * allreduce of o sums the shards (P:522-523 is a sum over k; P:536, P:542 merge by summation), so
 * the per-rank readout cost is 1/n of the single-GPU one.
 * Protocol: every rank creates the plan with the same geometry and its own k_rank, calls
 * wdd_set_comm (all ranks), exchanges store handles (wdd_shard_store_handle -> all-gather ->
 * wdd_set_shard_peers) and then, for each acquisition: wdd_reset (collective in a shard group),
 * wdd_ingest of its own frames, wdd_ingest_remote of every other rank's scan positions (host
 * bookkeeping only: those coefficients arrive from the peers), wdd_readout (collective; a barrier
 * collective orders every rank's projections before the flush reads the store).
 * In one process (tests, or several devices of one process) wdd_link_shards replaces the handle
 * exchange; without a communicator the caller orders ingests before readouts (e.g. one stream or a
 * device synchronisation) and combines wdd_readout_spectrum(..., combine = 0) itself. */

/* Positions ingested by other ranks of the plan's shard group (validated like wdd_ingest: range,
 * duplicates; the whole call is rejected on error).  Host bookkeeping only. */
wdd_status wdd_ingest_remote(wdd_plan_t plan, const int32_t* scan_idx_host, int64_t n);
/* IPC handle (64 bytes, cudaIpcGetMemHandle) of the plan's coefficient-store allocation. */
wdd_status wdd_shard_store_handle(wdd_plan_t plan, uint8_t handle[64]);
/* handles: nshard x 64 bytes, rank order (this rank's own entry is ignored); opens the peers'
 * stores in this process (cudaIpcOpenMemHandle).  nshard / rank must match the plan's options. */
wdd_status wdd_set_shard_peers(wdd_plan_t plan, int32_t nshard, int32_t rank, const uint8_t* handles);
/* Single process: plans[r] is shard r of nshard (same geometry); links their stores directly
 * (enables peer access between distinct devices). */
wdd_status wdd_link_shards(int32_t nshard, const wdd_plan_t* plans);

/* Thread-local description of the last error (never NULL). */
const char* wdd_last_error(void);

/* ------------------------------- introspection / test hooks ------------------------------ */
typedef struct {
  int32_t Sy, Sx, Q, L, K, n_vx, dtype, normalize;
  int64_t n_act;
  double dq, q_alpha, R_px, sigma_px, wavelength_A, step_A, eps;
  int64_t bytes_G, bytes_bank, bytes_R, bytes_C;
  int64_t frames_ingested;
  int32_t nranks, rank;
  int32_t proj_ctas_per_sm;   /* resident projection CTAs per SM (occupancy query; 2 = lean variant) */
  int32_t k_shards, k_rank;   /* coefficient shard group (1, 0 when unsharded)                         */
  int32_t k_lo, k_count;      /* this plan's coefficients k_lo .. k_lo + k_count - 1 (G, bank, store)  */
  int32_t n_vh;               /* primary scan-frequency columns of the Hermitian half-plane FFT flush
                                 (vx <= Sx/2; 0 = the active set is not symmetric, full plane)         */
} wdd_plan_info;
wdd_status wdd_get_info(wdd_plan_t plan, wdd_plan_info* info);

/* Conventional (full) WDD of a whole scan with the plan's geometry, probe and eps -- the paper's
 * comparison method (eq:deconv_mat P:90-95 and eq:extract P:97-106), no
 * dimensionality reduction: the unitary scan DFT of the 4-D data, per scan frequency v the
 * inverse detector DFT chi_v and the probe's W_P^v = F^-1(Y_v), the Wiener quotient
 * chi_v conj(W_P) / (|W_P|^2 + eps) summed over r (R12), and O = conj(F^-1_unitary(x)) (R13;
 * / sqrt(x_0) if the plan normalises).  frames_dev: DEVICE, S = Sy*Sx frames of Q x Q in the
 * plan's dtype, in scan order (s = sy*Sx + sx); complex_out_dev: DEVICE, Sy*Sx complex64.
 * Stream-ordered on `stream`; the first call allocates about (S + n_act)*Q*Q*8 bytes of device
 * scratch (the frames as float32 and the half-plane scan DFT, pixel-major; the active scan
 * frequencies' rows) and the
 * cuFFT plans, kept by the plan until wdd_destroy (WDD_E_NOMEM if the scratch is not available);
 * Q must be even.  Independent of the plan's ingest state. */
wdd_status wdd_full_wdd(wdd_plan_t plan, const void* frames_dev, void* complex_out_dev, void* stream);

/* Plan tables as the library computed them (host outputs, any may be NULL):
 *   basis  Q x L float64 (Psi[m][n]);  bank  n_act x K complex128 (accumulator order, before
 *   rounding to complex64);  active_v  n_act int32 (accumulator order). */
wdd_status wdd_get_tables(wdd_plan_t plan, double* basis, double* bank, int32_t* active_v);

/* Run only the projection kernel on n device frames: C_out_dev receives n x K float32,
 * C[f][a*L+b].  Enqueued on `stream`; does not touch the plan's accumulation state. */
wdd_status wdd_project(wdd_plan_t plan, const void* frames_dev, int64_t n, void* C_out_dev,
                       void* stream);

/* Per-kernel device timing (CUDA events around each launch) and launch counting.
 * wdd_profile_enable(plan, 1) starts recording; wdd_profile_read synchronises and returns,
 * for kernel slot i (0 = ingest, 1 = rowdft, 2 = flush, 3 = readout, 4 = finalize), the total
 * milliseconds and launch count since the last enable.  wdd_launch_count returns the number of
 * library kernels launched by this plan since creation (or the last counter reset). */
wdd_status wdd_profile_enable(wdd_plan_t plan, int32_t enable);
wdd_status wdd_profile_read(wdd_plan_t plan, int32_t slot, double* ms_total, int64_t* count);
wdd_status wdd_launch_count(wdd_plan_t plan, int64_t* count, int32_t reset);

/* CUDA-graph capture of a fixed call sequence (launch-bound live loops, e.g. 512-frame batches).
 * wdd_capture_begin starts stream capture on `stream`; every following wdd_reset / wdd_ingest /
 * wdd_readout / wdd_get_accumulator of this plan is recorded instead of executed (host-side
 * validation and bookkeeping still happen at capture time, once).  wdd_capture_end instantiates
 * the graph and returns a handle; wdd_graph_launch replays the recorded DEVICE work on `stream`.
 * Replays do not repeat host bookkeeping, so a captured sequence should begin with wdd_reset
 * (then each replay is a complete, self-contained acquisition).  wdd_ingest_host and
 * wdd_readout_host are not capturable (WDD_E_STATE).  Graphs are freed with the plan. */
wdd_status wdd_capture_begin(wdd_plan_t plan, void* stream);
wdd_status wdd_capture_end(wdd_plan_t plan, int64_t* graph_handle);
wdd_status wdd_graph_launch(wdd_plan_t plan, int64_t graph_handle, void* stream);

/* Block until all work enqueued by the plan has completed. */
wdd_status wdd_sync(wdd_plan_t plan);

#ifdef __cplusplus
}
#endif
#endif /* WDD_H_ */
