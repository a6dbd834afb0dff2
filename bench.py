#!/usr/bin/env python
"""Benchmark: diffraction frames/s ingested (projection + accumulation) + readout, Live WDD hot path.

Workload (default): BASELINE.json configs[4], "Box" -- the config the metric's "1/2/4/8 GPU" is
quoted on: 1024 x 1024 scan, 256 x 256 uint16 frames, K = 24 x 24, scan rows split across the
ranks.  One STEP = one whole acquisition (1 048 576 frames over all ranks) through the public C
ABI: wdd_reset, one wdd_ingest per batch (a1-a3, and the pending marks of a4), wdd_readout (a4-a5
flush, a6 Wiener readout, a7 NCCL combine, a8 inverse DFT + conj).

Frames: a device-resident pool of >= 1 GiB (>= 8 x the 126 MB L2: no step re-reads frames from L2)
of forward-model frames (synth/gpu.py: the paper's eq:forward, with Poisson noise at the
config's dose), cycled over the rank's scan positions, one wdd_ingest per pool-sized
batch (Box: 8 192 frames = 1 GiB per call).  Plans are created with ingest_overlap = 1 (the pool is
complete before the first library call), so consecutive projection launches stream back to back.
The acquisitions are captured as CUDA graphs (wdd_capture_begin; host validation of every index
set happens once, at capture) and replayed; consecutive acquisitions alternate the plan's two
coefficient stores, so each acquisition's first projection overlaps the previous readout.

Other configs: --config medium|large|live|tiny (Live: 1024-frame batches in scan order, a readout
every 64 scan rows; with N ranks the batches go round-robin, batch b -> rank b mod N).

Multi-GPU (torchrun, one process per GPU, NCCL): rows (Live: batches) are split across the ranks --
one acquisition, "strong" scaling.  --combine kshard (default for N > 1): every rank owns K/N of the
coefficients; the projection's epilogue stores each frame's coefficients of
another rank's shard straight into that rank's coefficient store over NVLink (peer memory), so the
per-rank readout shrinks as 1/N and only the n_act-entry spectrum is allreduced.  --combine
partial: every rank keeps a partial accumulator over all K and the spectrum (or G) is allreduced.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config box]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import CONFIGS, Acquisition  # noqa: E402

METRIC = "diffraction frames/s ingested (projection+accumulation), % of roofline, 1/2/4/8 GPU"
UNIT = "frames/s"
# the paper's own Live-WDD throughput on an exactly matching workload exists only for
# Medium, (128, 128, 128, 128) at L = 16: 12 412 frames/s (tab:fps_inc_scan; 32-core AMD
# EPYC 7543P).  Its nearest row to Box (1024^2 scan, but 128^2 detector and L = 16): 343 frames/s
# -- context only, another workload on another machine.
PAPER_FPS = {"medium": 12412.0}
PAPER_CONTEXT = {
    "medium": "paper P:815: 12 412 frames/s for (128,128,128,128), L=16, 32-core EPYC 7543P (context, not the target)",
    "box": "paper P:818: 343 frames/s for a 1024^2 scan with 128^2 frames, L=16, 32-core EPYC 7543P "
           "(nearest row; not this workload; context only)",
}
POOL_BYTES = 1 << 30


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def _traffic(workload):
    """DRAM bytes (read + write) per projection launch from the committed ncu --set full capture
    (profiles/ncu_traffic.json, written by tools/ncu_traffic.py), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f).get(workload, {})
    return d.get("project_kernel_bytes_per_launch")


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples = []
        self.period = period_s
        self.stop_ev = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                util = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                self.samples.append((mhz, rs, util))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        nv = self.nv
        names = {
            "gpu_idle": nv.nvmlClocksEventReasonGpuIdle,
            "applications_clocks_setting": nv.nvmlClocksEventReasonApplicationsClocksSetting,
            "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
            "hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
            "sync_boost": nv.nvmlClocksEventReasonSyncBoost,
            "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
            "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
            "hw_power_brake_slowdown": nv.nvmlClocksEventReasonHwPowerBrakeSlowdown,
        }
        loaded = [s for s in self.samples if s[2] > 0] or self.samples
        reasons = sorted({n for _, r, _ in loaded for n, bit in names.items() if r & bit and n != "gpu_idle"})
        return {"sm_mhz": statistics.median(s[0] for s in loaded), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(loaded)}


def host_info():
    """CPU model and the BLAS thread count the oracle ran with (SURVEY §8(d) CPU timing)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), None)
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = max((d.get("num_threads", 0) for d in threadpool_info() if d.get("user_api") == "blas"),
                   default=None)
    except Exception:
        pass
    return {"cpu_model": model, "blas_threads": blas}


# ----------------------------------------------------------------------------------------- oracle
class OracleSample:
    """The float64 oracle (as it stands) timed on a bounded sample of one acquisition, scaled to the
    whole acquisition.  Per acquisition the oracle does: the projection of every frame (cost linear
    in frames), one unitary 2-D FFT of the zero-filled coefficient stack over the scan per
    coefficient (linear in K), the readout sum over the active v (linear in K) and one inverse DFT.
    Timed here: the projection of the first `rows` scan rows (scaled by S / frames), the FFT and the
    readout on `n_coef` of the K coefficients (scaled by K / n_coef), the image transform once.  The
    bank is plan-time (the library's plan builds it too) and not timed; the timed readout uses a
    bank of the right shape.  Frames come from the host generator (not timed)."""

    def __init__(self, cfg, rows: int, n_coef: int):
        import oracle as O
        self.O, self.cfg = O, cfg
        self.rows, self.n_coef = min(rows, cfg.Sy), min(n_coef, cfg.K)
        g = O.geometry(cfg)
        self.idx = np.arange(self.rows * cfg.Sx)
        self.fr = Acquisition(cfg).frames_parallel(self.idx)
        self.Psi = O.hg_basis(cfg.Q, cfg.L, g.sigma)
        self.act = O.active_set(g, cfg.Sy, cfg.Sx)
        if self.n_coef == cfg.K and cfg.S * cfg.K <= (1 << 26):
            self.W = O.wiener_bank(g, self.Psi, self.act, cfg.Sy, cfg.Sx, cfg.eps)
            self.bank = "the oracle's Wiener bank"
        else:
            self.W = np.full((len(self.act), self.n_coef), 1.0 + 0.5j)
            self.bank = "a bank of the right shape (values do not change the cost)"

    def describe(self):
        c = self.cfg
        exact = self.rows == c.Sy and self.n_coef == c.K
        return (f"{c.name}: projection of the first {self.rows} scan rows ({len(self.idx)} frames) scaled to "
                f"{c.S} frames; 2-D scan FFT + Wiener readout on {self.n_coef} of {c.K} coefficients scaled to "
                f"{c.K}; one image IDFT; {self.bank}; float64 NumPy" + (" (the whole acquisition)" if exact else ""))

    def seconds(self) -> float:
        """Seconds the oracle needs for one whole acquisition (extrapolated from the sample)."""
        O, c = self.O, self.cfg
        t0 = time.perf_counter()
        C = O.vec(O.project(self.fr.astype(np.float64), self.Psi))
        t1 = time.perf_counter()
        G = O.accumulate_fft(C[:, :self.n_coef], self.idx, c.Sy, c.Sx)
        o = O.readout_spectrum(G[self.act], self.W, self.act, c.Sy, c.Sx)
        t2 = time.perf_counter()
        O.image_from_spectrum(o)
        t3 = time.perf_counter()
        return (t1 - t0) * c.S / len(self.idx) + (t2 - t1) * c.K / self.n_coef + (t3 - t2)


def run_reference(args):
    """--impl reference: the float64 oracle on the box's host cores, the same workload and metric;
    each step is one bounded sample of the acquisition (OracleSample), frames/s = S / extrapolated
    seconds.  Under torchrun rank 0 alone runs it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    small = cfg.S * cfg.K <= (1 << 23)
    smp = OracleSample(cfg, rows=cfg.Sy if small else 1, n_coef=cfg.K if small else 8)
    for _ in range(args.warmup):
        smp.seconds()
    t0 = time.perf_counter()
    secs = [smp.seconds() for _ in range(args.steps)]
    wall = time.perf_counter() - t0
    v = cfg.S / statistics.median(secs)
    cores = len(os.sched_getaffinity(0))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * cfg.S / v,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded forward model + Poisson, synth/)",
        "config": {"workload": cfg.name, "scan": [cfg.Sy, cfg.Sx], "detector": [cfg.Q, cfg.Q], "K": cfg.K,
                   "global_batch": cfg.S},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": smp.describe() + f"; median of {args.steps}", **host_info()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------- GPU arm
def _schedule(cfg, world, rank, batch, partition):
    """The acquisition as a list of steps for this rank: ("ingest", global batch, idx) for its own
    batches, ("remote", ..., idx) for the other ranks' batches (k-sharded plans mark them), and
    ("readout",) at the readout points (Live cadence: every cfg.readout_rows scan rows; else at
    the end).  partition "rows": contiguous row blocks per rank, batches within the rank's rows;
    "rr": global batches in scan order, batch b on rank b mod world."""
    steps = []
    if partition == "rows":
        blocks = np.array_split(np.arange(cfg.Sy), world)
        for r, rows in enumerate(blocks):
            idx = (rows[:, None] * cfg.Sx + np.arange(cfg.Sx)[None, :]).reshape(-1).astype(np.int32)
            for a in range(0, len(idx), batch):
                steps.append(("ingest" if r == rank else "remote", a, idx[a:a + batch]))
        steps.append(("readout",))
        return steps
    rows_done = 0
    for b, a in enumerate(range(0, cfg.S, batch)):
        idx = np.arange(a, min(cfg.S, a + batch), dtype=np.int32)
        steps.append(("ingest" if b % world == rank else "remote", a, idx))
        rows = (idx[-1] + 1) // cfg.Sx
        if cfg.readout_rows and rows - rows_done >= cfg.readout_rows:
            rows_done = rows
            steps.append(("readout",))
    if steps[-1][0] != "readout":
        steps.append(("readout",))
    return steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="wdd", choices=["wdd", "reference"])
    ap.add_argument("--config", default="box")
    ap.add_argument("--batch", type=int, default=0, help="frames per wdd_ingest (default: the config's, else pool-sized)")
    ap.add_argument("--pool-bytes", type=int, default=POOL_BYTES)
    ap.add_argument("--combine", default="auto", choices=["auto", "kshard", "partial"])
    ap.add_argument("--accumulator", default="G", choices=["G", "spectrum"])
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--readout-async", type=int, default=-1, choices=[-1, 0, 1],
                    help="pipelined acquisitions: readouts on the plan's readout stream (opts.readout_async); "
                         "-1 = on for large / live, where the readout overlapping the next projections gains "
                         "(Large +4%%, Live +2%%; Box even, Medium -2%%: tools/experiments/exp_roasync*.sh)")
    ap.add_argument("--acq-per-graph", type=int, default=0,
                    help="acquisitions per captured graph (0: 4 for small scans, 1 beyond)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=1)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.readout_async < 0:
        args.readout_async = int(args.config in ("large", "live"))

    import torch
    import torch.distributed as dist
    import paper_2212_01309_b200 as wdd
    from synth.gpu import GpuAcquisition

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    cfg = CONFIGS[args.config]
    fb = cfg.Q * cfg.Q * (2 if cfg.dtype == "u16" else 4)
    partition = "rr" if cfg.readout_rows else "rows"
    s_rank = cfg.S // world
    pool_cap = max(1, -(-args.pool_bytes // fb))
    batch = args.batch or cfg.batch or (s_rank if s_rank * fb <= 4 * args.pool_bytes else pool_cap)
    batch = min(batch, cfg.S)
    pool_n = max(batch, min(s_rank, pool_cap))
    pool_n = -(-pool_n // batch) * batch                      # whole batches: no batch wraps the pool
    combine = args.combine if args.combine != "auto" else ("kshard" if world > 1 else "partial")
    kshard = combine == "kshard" and world > 1
    schedule = _schedule(cfg, world, rank, batch, partition)
    own = [s for s in schedule if s[0] == "ingest"]
    n_own = sum(len(s[2]) for s in own)

    # device frame pool: forward-model frames of the rank's first positions (content does not
    # change the cost; the pool is cycled over the scan positions)
    pidx = np.concatenate([s[2] for s in own])[:pool_n]
    if len(pidx) < pool_n:
        pidx = np.resize(pidx, pool_n)
    sim = GpuAcquisition(cfg, device=f"cuda:{local}")
    pool = torch.cat([sim.frames(pidx[a:a + 4096]) for a in range(0, pool_n, 4096)])
    torch.cuda.synchronize()

    def frames_of(a, n):
        p0 = a % pool_n
        return pool[p0:p0 + n]

    def make_plan(sharded):
        pl = wdd.Plan.from_config(cfg, device=local, ingest_overlap=True, accumulator=args.accumulator,
                                  k_shards=world if sharded else 0, k_rank=rank if sharded else 0,
                                  readout_async=bool(args.readout_async) and not sharded)
        if world > 1:
            obj = [wdd.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            pl.set_comm(world, rank, obj[0])
        return pl

    plan = make_plan(kshard)
    combine_note = None
    if kshard:
        # map the peers' coefficient stores (CUDA IPC); if any rank cannot, every rank falls back to
        # the partial-accumulator combine (recorded in the JSON line)
        hs = [None] * world
        dist.all_gather_object(hs, plan.shard_store_handle())
        err = None
        try:
            plan.set_shard_peers(world, rank, hs)
        except wdd.WddError as e:
            err = str(e)
        errs = [None] * world
        dist.all_gather_object(errs, err)
        if any(errs):
            combine_note = "kshard peer mapping failed, partial combine used: " + next(e for e in errs if e)
            print(combine_note, file=sys.stderr, flush=True)
            plan.close()
            kshard, combine = False, "partial"
            schedule = _schedule(cfg, world, rank, batch, partition)
            plan = make_plan(False)
    out = torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device=f"cuda:{local}")
    stream = torch.cuda.Stream(device=local)      # graphs cannot capture the legacy default stream
    torch.cuda.synchronize()
    torch.cuda.set_stream(stream)

    def step_eager(events=None):
        plan.reset()
        for s in schedule:
            if s[0] == "ingest":
                if events is not None:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                plan.ingest(frames_of(s[1], len(s[2])), s[2], stream)
                if events is not None:
                    e1.record(stream)
                    events["ingest"].append((e0, e1))
            elif s[0] == "remote":
                if kshard:
                    plan.ingest_remote(s[2])
            else:
                if events is not None:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                plan.readout(out, wait=events is not None)
                if events is not None:
                    e1.record(stream)
                    events["readout"].append((e0, e1))

    # launches per step (library kernels only; cuFFT / NCCL kernels not counted)
    plan.launch_count(reset=True)
    step_eager()
    launches_per_step = plan.launch_count(reset=True)
    torch.cuda.synchronize()

    A = args.acq_per_graph or (4 if cfg.S <= 65536 else 1)
    graphs = {}

    def graph_for(n):
        if n not in graphs:
            plan.capture_begin(stream)
            for _ in range(n):
                step_eager()
            graphs[n] = plan.capture_end()
        return graphs[n]

    def run(n):
        if args.no_graph:
            for _ in range(n):
                step_eager()
        else:
            for _ in range(n // A):
                plan.graph_launch(graph_for(A), stream)
            if n % A:
                plan.graph_launch(graph_for(n % A), stream)
        plan.readout_wait(stream)     # (pipelined readouts: the last one completes inside the timed region)

    warmup = max(3, args.warmup)
    if not args.no_graph:
        graph_for(A)
        if args.steps % A:
            graph_for(args.steps % A)
    run(warmup)
    torch.cuda.synchronize()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        run(args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1)

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = max_over_ranks(ms)
    ms_step = ms / args.steps
    value = cfg.S * args.steps / (ms / 1e3)

    # ---- projection stage alone: a graph with the same reset + ingests and no readout, replayed
    # and timed with events on the plan stream (consecutive launches overlap: the stage time per
    # launch, not an isolated launch, is what the kernel costs inside the step)
    plan.capture_begin(stream)
    plan.reset()
    for s in own:
        plan.ingest(frames_of(s[1], len(s[2])), s[2], stream)
    h_ing = plan.capture_end()
    for _ in range(2):
        plan.graph_launch(h_ing, stream)
    torch.cuda.synchronize()
    reps = max(3, min(args.steps, 10 if cfg.S >= 1 << 18 else 100))   # (same on every rank)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(reps):
        plan.graph_launch(h_ing, stream)
    p1.record(stream)
    torch.cuda.synchronize()
    proj_ms_step = p0.elapsed_time(p1) / reps
    plan.reset()

    # ---- latencies: one eager acquisition with events around every call (events between
    # PDL-chained launches serialise them, so this pass is not used for throughput), and lone
    # batches on an idle GPU
    if world > 1:
        dist.barrier()
    evs = {"ingest": [], "readout": []}
    step_eager(evs)
    torch.cuda.synchronize()
    lat_ing = np.array([a.elapsed_time(b) for a, b in evs["ingest"]]) * 1e3
    lat_rd = np.array([a.elapsed_time(b) for a, b in evs["readout"]]) * 1e3
    def isolated(pl, hide_host=False):
        # a lone batch on an idle GPU (the second batch of an acquisition: not the wide first launch).
        # hide_host: a ~0.2 ms sleep kernel on the plan stream ahead of the first event, so the host's
        # submission of the call (Python, the C ABI, the launch) overlaps it and the events time the
        # device work of the batch alone; otherwise the interval includes the host submission.
        t = []
        for k in range(5):
            pl.reset()
            s0, s = own[0], own[min(1, len(own) - 1)]
            if s is not s0:
                pl.ingest(frames_of(s0[1], len(s0[2])), s0[2], stream)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if hide_host:
                with torch.cuda.stream(stream):
                    torch.cuda._sleep(400_000)
            e0.record(stream)
            pl.ingest(frames_of(s[1], len(s[2])), s[2], stream)
            e1.record(stream)
            torch.cuda.synchronize()
            t.append(e0.elapsed_time(e1) * 1e3)
        pl.reset()
        return t
    iso = isolated(plan) if not kshard else None          # (resets are collective in a shard group)
    iso_dev = isolated(plan, hide_host=True) if not kshard else None
    iso_spread = iso_spread_dev = None
    if world == 1:
        # the same on a plan with the latency grid (opts.ingest_spread = 1)
        lp = wdd.Plan.from_config(cfg, device=local, ingest_overlap=True, accumulator=args.accumulator,
                                  ingest_spread=True)
        iso_spread = isolated(lp)
        iso_spread_dev = isolated(lp, hide_host=True)
        lp.close()

    # ---- per-kernel device times (eager, event pairs around every launch: isolated-launch costs)
    plan.profile_enable(True)
    step_eager()
    torch.cuda.synchronize()
    kern = {}
    for name in ("project", "rowdft", "flush", "readout", "finalize"):
        tot, cnt = plan.profile_read(name)
        kern[name] = {"ms_total": tot, "launches": cnt, "ms_per_launch": tot / cnt if cnt else None}
    plan.profile_enable(False)
    plan.reset()

    peaks, peak_src = _peaks()
    info = plan.info()
    # wdd_ingest launches one projection per call over contiguous scan positions (all of bench.py's
    # batches are contiguous runs)
    n_launch = len(own)
    bytes_per_launch = n_own / n_launch * (fb + cfg.K * 4)     # frames read + C written (per launch)
    proj_ms_launch = proj_ms_step / n_launch
    achieved = bytes_per_launch / (proj_ms_launch * 1e-3) / 1e9
    # a lone batch's frame + C bytes at the copy peak (the floor of the isolated-batch latency)
    batch_bytes_floor_us = len(own[min(1, len(own) - 1)][2]) * (fb + cfg.K * 4) / (peaks["hbm_gbs"] * 1e9) * 1e6
    share = proj_ms_step / ms_step
    # whole-step algorithmic roofline (SURVEY §8(d) bytes per frame; every stage is HBM-bound):
    # frame + C write/read (8K) + R staging write/read (16 n_r K / Sx, n_r = the staged columns: the
    # n_vh primary columns of the Hermitian half plane for FFT flushes, all n_vx for the Live
    # cadence's GEMM flushes) + per readout the bank read (8 n_act K) and the G traffic (first
    # flush: write; later flushes: read + write; spectrum-only accumulator: none)
    n_read = sum(1 for s in schedule if s[0] == "readout")
    n_act, n_vx = info["n_act"], info["n_vx"]
    n_r = n_vx if (cfg.readout_rows or not info["n_vh"]) else info["n_vh"]
    g_passes = n_read + (2 * n_read - 1 if args.accumulator == "G" else 0)
    b_frame = fb + 8 * cfg.K + 16 * n_r * cfg.K / cfg.Sx + 8 * n_act * cfg.K * g_passes / cfg.S
    roof_fps = world * peaks["hbm_gbs"] * 1e9 / b_frame

    # ---- end to end through the public API: frames from pinned host memory (H2D inside the timed
    # region, wdd_ingest_host), the image back to the host (wdd_readout_host)
    pinned = pool.cpu().pin_memory()
    out_host = np.empty((cfg.Sy, cfg.Sx), dtype=np.complex64)

    def frames_host(a, n):
        p0 = a % pool_n
        return pinned[p0:p0 + n]

    def step_e2e():
        plan.reset()
        for s in schedule:
            if s[0] == "ingest":
                plan.ingest_host(frames_host(s[1], len(s[2])), s[2], stream)
            elif s[0] == "remote":
                if kshard:
                    plan.ingest_remote(s[2])
            else:
                plan.readout_host(out_host)

    e2e_steps = max(1, args.e2e_steps)
    step_e2e()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        step_e2e()
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = max_over_ranks(e0.elapsed_time(e1))
    e2e_value = cfg.S * e2e_steps / (e_ms / 1e3)

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            small = cfg.S * cfg.K <= (1 << 23)
            smp = OracleSample(cfg, rows=cfg.Sy if small else 4, n_coef=cfg.K if small else 32)
            secs = [smp.seconds() for _ in range(3)]
            cpu = {"value": cfg.S / statistics.median(secs), "unit": UNIT, "cores": len(os.sched_getaffinity(0)),
                   "kind": "oracle", "sample": smp.describe() + f"; median of 3 ({statistics.median(secs):.1f} s "
                   f"extrapolated per acquisition)", **host_info()}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": (value / PAPER_FPS[cfg.name]) if cfg.name in PAPER_FPS else None,
            "vs_baseline_ref": PAPER_CONTEXT.get(cfg.name),
            "dtype": "fp16x2+f32",
            "data": "synthetic (seeded forward model + Poisson on the GPU, synth/gpu.py); device frame pool",
            "config": {"workload": cfg.name, "scan": [cfg.Sy, cfg.Sx], "detector": [cfg.Q, cfg.Q],
                       "K": cfg.K, "batch": batch, "global_batch": cfg.S,
                       "parallelism": f"{'batches round-robin' if partition == 'rr' else 'rows'}/{world}"
                                      + (f", coefficient shards/{world} (P2P)" if kshard else ""),
                       "combine": combine, "combine_note": combine_note, "accumulator": args.accumulator,
                       "readouts_per_step": n_read,
                       "l2": f"inputs larger than L2: frame pool {pool_n * fb / 2**30:.2f} GiB cycled",
                       "graph": not args.no_graph, "acquisitions_per_graph": None if args.no_graph else A,
                       "readout_async": plan.readout_async},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": _traffic(cfg.name),
                         "kernel": "project_kernel", "peak_source": peak_src,
                         "bytes_per_launch": bytes_per_launch, "ms_per_launch": proj_ms_launch,
                         "launches_per_step": n_launch, "share_of_step": share},
            "step_roofline": {"bytes_per_frame": b_frame, "frames_per_s_at_hbm": roof_fps, "frac": value / roof_fps,
                              "frame_bytes_only_frames_per_s": world * peaks["hbm_gbs"] * 1e9 / fb},
            "latency": {
                "ingest_batch_us": {"p50": float(np.percentile(lat_ing, 50)), "p99": float(np.percentile(lat_ing, 99)),
                                    "max": float(lat_ing.max()), "n": int(len(lat_ing)), "frames": batch},
                "isolated_batch_us": {"median": float(np.median(iso)) if iso else None, "n": len(iso or []),
                                      "frames": len(own[min(1, len(own) - 1)][2]),
                                      "latency_grid_median": float(np.median(iso_spread)) if iso_spread else None,
                                      "device_median": float(np.median(iso_dev)) if iso_dev else None,
                                      "device_latency_grid_median":
                                          float(np.median(iso_spread_dev)) if iso_spread_dev else None,
                                      "floor_at_hbm": batch_bytes_floor_us},
                "readout_us": {"p50": float(np.percentile(lat_rd, 50)), "max": float(lat_rd.max()),
                               "n": int(len(lat_rd))},
                "how": "CUDA events around each call of one eager acquisition (ingest_batch, readout); "
                       "isolated_batch: one batch on an idle GPU after a sync (default throughput grid, "
                       "and on a plan with the latency grid, opts.ingest_spread = 1), from the call to "
                       "completion; device_*: the same with the host submission hidden behind a sleep "
                       "kernel (device work of the batch alone); floor_at_hbm: the batch's frame + C "
                       "bytes at the measured copy peak"},
            "kernels_isolated": kern,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(cfg.S * fb),
                    "d2h_bytes_per_step": int(cfg.S * 8 * n_read)},
            "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
