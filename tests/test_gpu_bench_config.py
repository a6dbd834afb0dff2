"""Box at full size in exactly the launch configuration bench.py times (the headline line): a
1 GiB device pool of 8 192 forward-model frames from the GPU simulator, cycled over the 1 048 576
scan positions in 8 192-frame `wdd_ingest` calls on a plan with ingest_overlap = 1, reset + 128
ingests + readout captured as ONE CUDA graph and replayed.

What the oracle can say about it: the pool is 8 scan rows, so the acquisition is periodic along sy
with period 8, and the scan DFT of a period-8 signal of length 1024 is supported on vy = 128 m:

    G[(128 m, vx), k] = sqrt(128) * G8[(m, vx), k],      G = 0 at every other vy,

with G8 the oracle's accumulator of the 8 x 1024 scan of the pool frames (eq:outer_prod, P:424,
`oracle.accumulate_fft` with norm 1/sqrt(8 * 1024)).  The test does not trust that identity on its
own: sampled rows of G (on and off the support) are also computed by the oracle's direct sum
over all 1 048 576 scan positions, G[v] = sum_s f_s[v] c_s (`oracle.scan_phase`, block by block).
Then, as in Algorithm 2: o_v = sum_k G[v,k] K_v[k] with the oracle's Wiener bank at
the supported active v (the active set itself is the oracle's, from tests/golden/fullsize_box.npz),
and O = conj(IDFT2(o)).  Compared whole: G on the support, G off the support (zero up to float32
rounding), the spectrum and the image, relative L2 <= 1e-4 (north star); the replays and the eager
run bit-identical.  Errors are appended to gpurun_out/fullsize_parity.jsonl.

Live the same way (bench.py --config live): the 1 GiB pool is 16 of its 512 scan rows, ingested in
1 024-frame batches with a readout every 64 rows on a plan with pipelined readouts
(readout_async), the whole acquisition (512 ingests, 8 readouts) one graph.  All 8 readouts of the
replays must be bit-identical to the eager run's; the last one (whole scan, period 16: support
vy = 32 m) is compared whole with the oracle as above."""
import json
import os
import time

import numpy as np
import pytest

import oracle as O
from synth import CONFIGS

pytestmark = pytest.mark.gpu
TOL = 1e-4
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def test_box_graph_replay_of_cycled_pool_matches_oracle():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    from paper_2212_01309_b200 import build
    build.build()
    import paper_2212_01309_b200 as wdd
    from synth.gpu import GpuAcquisition

    cfg = CONFIGS["box"]
    batch = pool_n = (1 << 30) // (cfg.Q * cfg.Q * 2)       # bench.py's defaults: a 1 GiB pool, one pool per ingest
    assert batch == 8192 and pool_n % cfg.Sx == 0 and cfg.S % pool_n == 0
    rows_p = pool_n // cfg.Sx                               # 8 scan rows per pool cycle
    rep = cfg.Sy // rows_p                                  # 128 cycles
    sim = GpuAcquisition(cfg, device="cuda:0")
    pool = torch.cat([sim.frames(np.arange(a, a + 4096)) for a in range(0, pool_n, 4096)])
    torch.cuda.synchronize()

    plan = wdd.Plan.from_config(cfg, device=0, ingest_overlap=True)
    out = torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device="cuda:0")
    stream = torch.cuda.Stream(device=0)
    torch.cuda.synchronize()
    torch.cuda.set_stream(stream)
    try:
        def step():
            plan.reset()
            for a in range(0, cfg.S, batch):
                plan.ingest(pool, np.arange(a, a + batch, dtype=np.int32), stream)
            plan.readout(out, wait=False)

        plan.launch_count(reset=True)
        step()                                              # eager
        launches = plan.launch_count(reset=True)
        torch.cuda.synchronize()
        img_eager = out.cpu().numpy()
        plan.capture_begin(stream)
        step()
        h = plan.capture_end()
        imgs = []
        for _ in range(2):                                  # back-to-back replays, as the bench runs them
            out.zero_()
            plan.graph_launch(h, stream)
            plan.graph_launch(h, stream)
            torch.cuda.synchronize()
            imgs.append(out.cpu().numpy())
        assert launches >= cfg.S // batch + 3               # 128 projections + the flush / image kernels
        assert np.array_equal(imgs[0], img_eager) and np.array_equal(imgs[1], img_eager)
        G_gpu, act = plan.get_accumulator()
        spec = plan.readout_spectrum().cpu().numpy().reshape(-1)
        torch.cuda.synchronize()
    finally:
        torch.cuda.set_stream(torch.cuda.default_stream())

    # ---- oracle: coefficients of the 8 192 pool frames, their 8 x 1024 scan DFT
    g = O.geometry(cfg)
    Psi = O.hg_basis(cfg.Q, cfg.L, g.sigma)
    fr = pool.cpu().numpy()
    C8 = np.concatenate([O.vec(O.project(fr[a:a + 256].astype(np.float64), Psi)) for a in range(0, pool_n, 256)])
    G8 = O.accumulate_fft(C8, np.arange(pool_n), rows_p, cfg.Sx)          # [(m, vx), k]
    gold_act = np.load(os.path.join(ROOT, "tests", "golden", "fullsize_box.npz"))["act"]
    assert np.array_equal(np.sort(act), gold_act)                        # the oracle's active set
    vy, vx = act // cfg.Sx, act % cfg.Sx
    on = vy % rep == 0
    G_on_ref = np.sqrt(rep) * G8[(vy[on] // rep) * cfg.Sx + vx[on]]

    # the periodicity identity itself, pinned on sampled rows by the oracle's direct sum over the
    # whole scan (on the support: against the identity; off it: exactly cancelling phases)
    rng = np.random.default_rng(5)
    s_on = rng.choice(np.nonzero(on)[0], 6, replace=False)
    s_off = rng.choice(np.nonzero(~on)[0], 6, replace=False)
    samp = np.concatenate([s_on, s_off])
    G_dir = np.zeros((len(samp), cfg.K), dtype=np.complex128)
    for b in range(rep):
        G_dir += O.scan_phase(act[samp], np.arange(b * pool_n, (b + 1) * pool_n), cfg.Sy, cfg.Sx) @ C8
    pos_on = {int(i): k for k, i in enumerate(np.nonzero(on)[0])}
    ident = rel(G_dir[:6], G_on_ref[[pos_on[int(i)] for i in s_on]])
    assert ident < 1e-11, ident
    scale = float(np.sqrt(np.mean(np.abs(G_on_ref) ** 2)))
    assert np.max(np.abs(G_dir[6:])) < 1e-9 * scale

    idx_t = torch.from_numpy(samp).cuda()
    e = {"config": "box_bench_launch_config", "launches_per_step": int(launches),
         "G_sampled_direct": rel(G_gpu[idx_t[:6]].cpu().numpy(), G_dir[:6])}
    on_t = torch.from_numpy(np.nonzero(on)[0]).cuda()
    G_on = G_gpu[on_t].cpu().numpy()
    e["G_support"] = rel(G_on, G_on_ref)
    e["G_support_ac"] = rel(G_on[:, 1:], G_on_ref[:, 1:])
    off_t = torch.from_numpy(np.nonzero(~on)[0]).cuda()
    # off the support G is zero: what float32 leaves there, relative to the supported rows
    off_sq = 0.0
    for a in range(0, len(off_t), 65536):
        blk = G_gpu[off_t[a:a + 65536]]
        off_sq += float((blk.real.double() ** 2 + blk.imag.double() ** 2).sum().item())
    e["G_off_support_over_support"] = float(np.sqrt(off_sq) / np.linalg.norm(G_on_ref))

    W = O.wiener_bank(g, Psi, act[on], cfg.Sy, cfg.Sx, cfg.eps)
    o_ref = O.readout_spectrum(G_on_ref, W, act[on], cfg.Sy, cfg.Sx)
    O_ref = O.image_from_spectrum(o_ref)
    inactive = np.ones(cfg.S, bool)
    inactive[act] = False
    assert float(np.max(np.abs(spec[inactive]), initial=0.0)) == 0.0
    e["o"] = rel(spec, o_ref.reshape(-1))
    e["o_support"] = rel(spec[act[on]], o_ref.reshape(-1)[act[on]])
    e["O"] = rel(img_eager, O_ref)
    e["O_mean_removed"] = rel(img_eager - img_eager.mean(), O_ref - O_ref.mean())
    plan.close()

    e["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    print(json.dumps(e))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "fullsize_parity.jsonl"), "a") as f:
        f.write(json.dumps(e) + "\n")
    for k in ("G_sampled_direct", "G_support", "G_support_ac", "G_off_support_over_support", "o", "o_support",
              "O", "O_mean_removed"):
        assert e[k] < TOL, (k, e[k])


def test_live_graph_replay_of_cycled_pool_matches_oracle():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    from paper_2212_01309_b200 import build
    build.build()
    import paper_2212_01309_b200 as wdd
    from synth.gpu import GpuAcquisition

    cfg = CONFIGS["live"]
    batch = cfg.batch
    pool_n = (1 << 30) // (cfg.Q * cfg.Q * 2)               # bench.py's default 1 GiB pool
    assert batch == 1024 and pool_n == 8192 and pool_n % cfg.Sx == 0 and cfg.S % pool_n == 0
    rows_p = pool_n // cfg.Sx                               # 16 scan rows per pool cycle
    rep = cfg.Sy // rows_p                                  # 32 cycles
    n_ro = cfg.Sy // cfg.readout_rows
    sim = GpuAcquisition(cfg, device="cuda:0")
    pool = torch.cat([sim.frames(np.arange(a, a + 4096)) for a in range(0, pool_n, 4096)])
    torch.cuda.synchronize()

    plan = wdd.Plan.from_config(cfg, device=0, ingest_overlap=True, readout_async=True)
    outs = [torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device="cuda:0") for _ in range(n_ro)]
    stream = torch.cuda.Stream(device=0)
    torch.cuda.synchronize()
    torch.cuda.set_stream(stream)
    try:
        def step():
            plan.reset()
            done = k = 0
            for a in range(0, cfg.S, batch):
                plan.ingest(pool[a % pool_n:a % pool_n + batch], np.arange(a, a + batch, dtype=np.int32), stream)
                rows = (a + batch) // cfg.Sx
                if rows - done >= cfg.readout_rows:
                    done = rows
                    plan.readout(outs[k], wait=False)
                    k += 1
            assert k == n_ro

        step()                                              # eager
        plan.readout_wait(stream)
        torch.cuda.synchronize()
        eager = [o.cpu().numpy() for o in outs]
        assert not np.array_equal(eager[0], eager[-1])
        plan.capture_begin(stream)
        step()
        h = plan.capture_end()
        for _ in range(2):                                  # back-to-back replays, as the bench runs them
            for o in outs:
                o.zero_()
            plan.graph_launch(h, stream)
            plan.graph_launch(h, stream)
            plan.readout_wait(stream)
            torch.cuda.synchronize()
            for k, o in enumerate(outs):
                assert np.array_equal(o.cpu().numpy(), eager[k]), ("replay", k)
        G_gpu, act = plan.get_accumulator()
        spec = plan.readout_spectrum().cpu().numpy().reshape(-1)
        torch.cuda.synchronize()
    finally:
        torch.cuda.set_stream(torch.cuda.default_stream())

    g = O.geometry(cfg)
    Psi = O.hg_basis(cfg.Q, cfg.L, g.sigma)
    fr = pool.cpu().numpy()
    C16 = np.concatenate([O.vec(O.project(fr[a:a + 256].astype(np.float64), Psi)) for a in range(0, pool_n, 256)])
    G16 = O.accumulate_fft(C16, np.arange(pool_n), rows_p, cfg.Sx)
    gold_act = np.load(os.path.join(ROOT, "tests", "golden", "fullsize_live.npz"))["act"]
    assert np.array_equal(np.sort(act), gold_act)
    vy, vx = act // cfg.Sx, act % cfg.Sx
    on = vy % rep == 0
    G_on_ref = np.sqrt(rep) * G16[(vy[on] // rep) * cfg.Sx + vx[on]]
    rng = np.random.default_rng(6)
    s_on = rng.choice(np.nonzero(on)[0], 6, replace=False)
    s_off = rng.choice(np.nonzero(~on)[0], 6, replace=False)
    samp = np.concatenate([s_on, s_off])
    G_dir = np.zeros((len(samp), cfg.K), dtype=np.complex128)
    for b in range(rep):
        G_dir += O.scan_phase(act[samp], np.arange(b * pool_n, (b + 1) * pool_n), cfg.Sy, cfg.Sx) @ C16
    pos_on = {int(i): k for k, i in enumerate(np.nonzero(on)[0])}
    assert rel(G_dir[:6], G_on_ref[[pos_on[int(i)] for i in s_on]]) < 1e-11
    scale = float(np.sqrt(np.mean(np.abs(G_on_ref) ** 2)))
    assert np.max(np.abs(G_dir[6:])) < 1e-9 * scale

    e = {"config": "live_bench_launch_config",
         "G_sampled_direct": rel(G_gpu[torch.from_numpy(s_on).cuda()].cpu().numpy(), G_dir[:6])}
    G_on = G_gpu[torch.from_numpy(np.nonzero(on)[0]).cuda()].cpu().numpy()
    e["G_support"] = rel(G_on, G_on_ref)
    e["G_support_ac"] = rel(G_on[:, 1:], G_on_ref[:, 1:])
    # off the support the eight 64-row flushes cancel only up to the GEMM flush's rounding
    off_t = torch.from_numpy(np.nonzero(~on)[0]).cuda()
    off_sq = 0.0
    for a in range(0, len(off_t), 32768):
        blk = G_gpu[off_t[a:a + 32768]]
        off_sq += float((blk.real.double() ** 2 + blk.imag.double() ** 2).sum().item())
    e["G_off_support_over_support"] = float(np.sqrt(off_sq) / np.linalg.norm(G_on_ref))
    W = O.wiener_bank(g, Psi, act[on], cfg.Sy, cfg.Sx, cfg.eps)
    o_ref = O.readout_spectrum(G_on_ref, W, act[on], cfg.Sy, cfg.Sx)
    O_ref = O.image_from_spectrum(o_ref)
    inactive = np.ones(cfg.S, bool)
    inactive[act] = False
    assert float(np.max(np.abs(spec[inactive]), initial=0.0)) == 0.0
    e["o"] = rel(spec, o_ref.reshape(-1))
    e["o_support"] = rel(spec[act[on]], o_ref.reshape(-1)[act[on]])
    e["O"] = rel(eager[-1], O_ref)
    e["O_mean_removed"] = rel(eager[-1] - eager[-1].mean(), O_ref - O_ref.mean())
    plan.close()
    e["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    print(json.dumps(e))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "fullsize_parity.jsonl"), "a") as f:
        f.write(json.dumps(e) + "\n")
    for k in ("G_sampled_direct", "G_support", "G_support_ac", "G_off_support_over_support", "o", "o_support",
              "O", "O_mean_removed"):
        assert e[k] < TOL, (k, e[k])
