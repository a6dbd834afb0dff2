#!/usr/bin/env python
"""Benchmark: diffraction frames/s ingested (projection + accumulation) + readout, Live WDD hot path.

Workload (BASELINE.json configs[1], "Medium"): 128 x 128 scan, 128 x 128 uint16 frames, K = 16 x 16,
ingest in batches of 512 frames.  One STEP = one complete acquisition through the public C ABI:
wdd_reset, 32 x wdd_ingest (512 frames each, all of §8(a) a1-a5), wdd_readout (a5 flush, a6
Wiener readout, a7 combine, a8 inverse DFT + conj).  Frames are seeded synthetic data from
synth/ (the paper's forward model + Poisson dose), resident in HBM (537 MB > 126 MB L2, so no
step re-reads frames from L2).  The step is captured once as a CUDA graph (wdd_capture_begin) and
replayed; host validation of each index set happens at capture.

Multi-GPU (torchrun, one process per GPU): the scan rows are split across ranks ("strong"
scaling of one acquisition); each rank keeps a partial accumulator and wdd_readout allreduces
the Wiener-filtered spectrum over NCCL (exact by linearity).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
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
# the paper's own Live-WDD throughput on this exact workload, (128, 128, 128, 128) at
# L = 16: 12 412 frames/s (tab:fps_inc_scan; 32-core AMD EPYC 7543P, another machine)
PAPER_FPS = {"medium": 12412.0}


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
        return json.load(f).get(workload, {}).get("project_kernel_bytes_per_launch")


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


# ----------------------------------------------------------------------------------------- oracle
def oracle_prepare(cfg, n_frames: int):
    """Frames of the first n_frames scan positions and the plan-time tables (bank precomputed, as
    the library's plan is); not timed."""
    import oracle as O
    g = O.geometry(cfg)
    idx = np.arange(n_frames)
    fr = Acquisition(cfg).frames_parallel(idx)
    Psi = O.hg_basis(cfg.Q, cfg.L, g.sigma)
    act = O.active_set(g, cfg.Sy, cfg.Sx)
    W = O.wiener_bank(g, Psi, act, cfg.Sy, cfg.Sx, cfg.eps)
    return idx, fr, Psi, act, W


def oracle_pass(cfg, prep) -> float:
    """One timed pass of the float64 oracle (as it stands): projection + FFT accumulation + Wiener
    readout + inverse DFT of the prepared frames; returns seconds."""
    import oracle as O
    idx, fr, Psi, act, W = prep
    t0 = time.perf_counter()
    C = O.vec(O.project(fr.astype(np.float64), Psi))
    G = O.accumulate_fft(C, idx, cfg.Sy, cfg.Sx)
    o = O.readout_spectrum(G[act], W, act, cfg.Sy, cfg.Sx)
    O.image_from_spectrum(o)
    return time.perf_counter() - t0


def oracle_baseline(cfg, n_frames: int, repeats: int = 1):
    """Frames/s of the oracle on the first n_frames scan positions, median of `repeats` passes."""
    prep = oracle_prepare(cfg, n_frames)
    t = statistics.median(oracle_pass(cfg, prep) for _ in range(repeats))
    cores = len(os.sched_getaffinity(0))
    return n_frames / t, cores, t


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


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    # one step = one oracle pass over the whole acquisition (Medium: 16 384 frames, ~1 s on 16
    # cores) while the run stays within a few minutes, else over the first --ref-frames positions
    n = min(cfg.S, 16384) if args.steps + args.warmup <= 150 else args.ref_frames
    prep = oracle_prepare(cfg, n)
    for _ in range(args.warmup):
        oracle_pass(cfg, prep)
    t0 = time.perf_counter()
    secs = [oracle_pass(cfg, prep) for _ in range(args.steps)]
    wall = time.perf_counter() - t0
    v = n / statistics.median(secs)
    cores = len(os.sched_getaffinity(0))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * n / v,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded forward model + Poisson, synth/)",
        "config": {"workload": cfg.name, "scan": [cfg.Sy, cfg.Sx], "detector": [cfg.Q, cfg.Q], "K": cfg.K,
                   "sample_frames": n, "global_batch": n},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"first {n} scan positions of {cfg.name}"
                                   f"{' (the whole scan)' if n == cfg.S else ''}: projection + FFT "
                                   f"accumulation + Wiener readout + IDFT, float64 NumPy, median of {args.steps}",
                         **host_info()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="wdd", choices=["wdd", "reference"])
    ap.add_argument("--config", default="medium")
    ap.add_argument("--batch", type=int, default=0, help="override the workload's batch (experiments only)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--acq-per-graph", type=int, default=4,
                    help="acquisitions per captured graph (consecutive ones overlap readout and projection)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-frames", type=int, default=2048)
    ap.add_argument("--e2e-steps", type=int, default=5)

    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2212_01309_b200 as wdd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    cfg = CONFIGS[args.config]
    batch = args.batch or cfg.batch or cfg.S
    rows = np.array_split(np.arange(cfg.Sy), world)[rank]
    idx = (rows[:, None] * cfg.Sx + np.arange(cfg.Sx)[None, :]).reshape(-1).astype(np.int32)
    frames = Acquisition(cfg).frames_parallel(idx)
    dev = torch.from_numpy(frames).to(f"cuda:{local}")
    pinned = torch.from_numpy(frames).pin_memory()
    frame_bytes = cfg.Q * cfg.Q * frames.dtype.itemsize

    plan = wdd.Plan.from_config(cfg, device=local)
    if world > 1:
        obj = [wdd.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        plan.set_comm(world, rank, obj[0])
    out = torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device=f"cuda:{local}")
    stream = torch.cuda.Stream(device=local)      # graphs cannot capture the legacy default stream
    torch.cuda.synchronize()
    torch.cuda.set_stream(stream)
    batches = [(a, min(a + batch, len(idx))) for a in range(0, len(idx), batch)]

    def step_eager():
        plan.reset()
        for a, b in batches:
            plan.ingest(dev[a:b], idx[a:b], stream)
        plan.readout(out)

    # launches per step (library kernels only; cuFFT's own kernels not counted)
    plan.launch_count(reset=True)
    step_eager()
    launches_per_step = plan.launch_count(reset=True)
    torch.cuda.synchronize()

    # A graph holds `acq_per_graph` consecutive acquisitions: inside it each acquisition's first
    # projection overlaps the previous acquisition's readout (the plan alternates two coefficient
    # stores across resets), as back-to-back scans do in a live session; graph launches themselves
    # serialise.  `run(n)` performs exactly n steps (acquisitions).
    A = max(1, args.acq_per_graph)
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
            return
        for _ in range(n // A):
            plan.graph_launch(graph_for(A), stream)
        if n % A:
            plan.graph_launch(graph_for(n % A), stream)

    if not args.no_graph:
        graph_for(A)
        if args.steps % A:
            graph_for(args.steps % A)
    run(max(3, args.warmup))
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
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = cfg.S * args.steps / (ms / 1e3)

    # ---- projection stage alone: a second graph with the same reset + ingests and no readout
    # (the flush runs at readout), replayed and timed with events on the plan stream.  Batches
    # overlap on the GPU (PDL), so the stage time, not an isolated launch, is what the kernel costs.
    plan.capture_begin(stream)
    plan.reset()
    for a, b in batches:
        plan.ingest(dev[a:b], idx[a:b], stream)
    h_ing = plan.capture_end()
    for _ in range(3):
        plan.graph_launch(h_ing, stream)
    plan.reset()
    torch.cuda.synchronize()
    reps = max(10, min(args.steps, 100))
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(reps):
        plan.graph_launch(h_ing, stream)
    p1.record(stream)
    torch.cuda.synchronize()
    plan.reset()
    proj_ms_step = p0.elapsed_time(p1) / reps

    # ---- per-kernel device times (eager pass with event pairs around every launch; batches do
    # not overlap here, so these are isolated-launch costs)
    prof_steps = min(args.steps, 20)
    plan.profile_enable(True)
    for _ in range(prof_steps):
        step_eager()
    torch.cuda.synchronize()
    kern = {}
    for name in ("project", "rowdft", "flush", "readout", "finalize"):
        tot, cnt = plan.profile_read(name)
        kern[name] = {"ms_total": tot, "launches": cnt, "ms_per_launch": tot / cnt if cnt else None}
    plan.profile_enable(False)
    peaks, peak_src = _peaks()
    info = plan.info()
    n_launch = len(batches)
    frames_per_launch = len(idx) / n_launch
    bytes_per_launch = frames_per_launch * (frame_bytes + cfg.K * 4)   # frames read + C written
    proj_ms_launch = proj_ms_step / n_launch
    achieved = bytes_per_launch / (proj_ms_launch * 1e-3) / 1e9
    share = proj_ms_step / ms_step
    # whole-step algorithmic roofline (SURVEY §8(d) bytes per frame; every stage is HBM-bound):
    # frame + C write/read (8K) + row staging R write/read (16 n_vx K / Sx) + G written once and
    # the bank read once by the fused readout (2 x 8 n_act K / S)
    b_step = (frame_bytes + 8 * cfg.K + 16 * info["n_vx"] * cfg.K / cfg.Sx
              + 16 * info["n_act"] * cfg.K / cfg.S)
    roof_fps = peaks["hbm_gbs"] * 1e9 / b_step

    # ---- end to end through the public API from pinned host memory (H2D + compute + D2H)
    out_host = np.empty((cfg.Sy, cfg.Sx), dtype=np.complex64)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step_e2e():
        plan.reset()
        for a, b in batches:
            plan.ingest_host(pinned[a:b], idx[a:b], stream)
        plan.readout_host(out_host)

    step_e2e()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.e2e_steps):
        step_e2e()
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    e2e_value = cfg.S * args.e2e_steps / (e_ms / 1e3)

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            # the whole acquisition (Medium: 16 384 frames, ~2 s per pass), median of 5 passes:
            # about 10 s of CPU work
            n_cpu = min(cfg.S, max(args.ref_frames, 16384))
            v, cores, t = oracle_baseline(cfg, n_cpu, repeats=5)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                   "sample": f"first {n_cpu} scan positions of {cfg.name} (the whole scan for Medium): "
                             f"projection + FFT accumulation + Wiener readout + IDFT, float64 NumPy, "
                             f"median of 5 passes ({t:.1f} s each)", **host_info()}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": (value / PAPER_FPS[cfg.name]) if cfg.name in PAPER_FPS else None,
            "vs_baseline_ref": "paper P:815, 12412 frames/s on a 32-core CPU (context, not the target)",
            "dtype": "fp16x2+f32",
            "data": "synthetic (seeded forward model + Poisson, synth/); frames resident in HBM",
            "config": {"workload": cfg.name, "scan": [cfg.Sy, cfg.Sx], "detector": [cfg.Q, cfg.Q],
                       "K": cfg.K, "batch": batch, "global_batch": cfg.S, "parallelism": f"rows/{world}",
                       "l2": "inputs larger than L2 (537 MB of frames per step)",
                       "graph": not args.no_graph, "acquisitions_per_graph": None if args.no_graph else A},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": _traffic(cfg.name), "kernel": "project_kernel",
                         "peak_source": peak_src, "bytes_per_launch": bytes_per_launch,
                         "ms_per_launch": proj_ms_launch, "launches_per_step": n_launch,
                         "share_of_step": share},
            "kernels_isolated": kern,
            "step_roofline": {"bytes_per_frame": b_step, "frames_per_s_at_hbm": roof_fps,
                              "frac": value / roof_fps,
                              "frame_bytes_only_frames_per_s": peaks["hbm_gbs"] * 1e9 / frame_bytes},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(len(idx) * frame_bytes),
                    "d2h_bytes_per_step": int(cfg.S * 8)},
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
