"""Back-to-back acquisitions with overlap: a reset after ingests swaps the plan's two coefficient
stores, so the next acquisition's first projection is launched programmatically (PDL) behind the
previous acquisition's readout instead of after it.  The readouts must be bit-identical to the
same acquisitions run one at a time with a device synchronisation in between (same kernels, same
arithmetic: any race on the coefficient store, R, G or the partial readouts shows up as a
difference), both eagerly and inside one captured CUDA graph (bench.py's step graph).  Plans with
readout_async run each readout on their readout stream while the plan stream goes on with the
next acquisition: the same bit-identity must hold."""
import numpy as np
import pytest

from synth import CONFIGS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    from paper_2212_01309_b200 import build
    build.build()
    import paper_2212_01309_b200 as wdd
    return torch, wdd


def _check_overlap(torch, wdd, cfg, batch, n_acq, readout_async=False, accumulator="G", cadence=0):
    from synth.sparse import dense_frames_torch, sparse_events
    idx = np.arange(cfg.S)
    b = batch
    acqs = [dense_frames_torch(*sparse_events(seed, idx, cfg.Q), cfg.Q, "cuda") for seed in range(11, 11 + n_acq)]
    plan = wdd.Plan.from_config(cfg, ingest_overlap=True, readout_async=readout_async, accumulator=accumulator)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    def acquire(fr, out):
        # cadence > 0: a readout (into out, overwritten) after every `cadence` batches as well
        plan.reset()
        for i, a in enumerate(range(0, cfg.S, b)):
            plan.ingest(fr[a:a + b], idx[a:a + b].astype(np.int32), stream)
            if cadence and (i + 1) % cadence == 0 and a + b < cfg.S:
                plan.readout(out, wait=False)
        plan.readout(out, wait=False)

    iso = []
    for fr in acqs:
        out = torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device="cuda")
        acquire(fr, out)
        torch.cuda.synchronize()
        iso.append(out.cpu().numpy())
    assert not np.array_equal(iso[0], iso[1])
    if readout_async and not cadence:   # the pipelined plan's isolated images are the ordinary plan's
        ref = wdd.Plan.from_config(cfg, ingest_overlap=True, accumulator=accumulator)
        ref.reset()
        for a in range(0, cfg.S, b):
            ref.ingest(acqs[0][a:a + b], idx[a:a + b].astype(np.int32), stream)
        img = ref.readout()
        torch.cuda.synchronize()
        assert np.array_equal(img.cpu().numpy(), iso[0])
        ref.close()

    # eager, no synchronisation between the acquisitions
    outs = [torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device="cuda") for _ in acqs]
    for fr, out in zip(acqs, outs):
        acquire(fr, out)
    torch.cuda.synchronize()
    for k, out in enumerate(outs):
        assert np.array_equal(out.cpu().numpy(), iso[k]), ("eager", k)

    # one graph holding the acquisitions, replayed twice
    gouts = [torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device="cuda") for _ in acqs]
    plan.capture_begin(stream)
    for fr, out in zip(acqs, gouts):
        acquire(fr, out)
    h = plan.capture_end()
    for _ in range(2):
        for out in gouts:
            out.zero_()
        plan.graph_launch(h, stream)
        torch.cuda.synchronize()
        for k, out in enumerate(gouts):
            assert np.array_equal(out.cpu().numpy(), iso[k]), ("graph", k)
    plan.sync()
    torch.cuda.set_stream(torch.cuda.default_stream())


@pytest.mark.parametrize("name", ["medium", "large"])
def test_overlapped_acquisitions_match_isolated(env, name):
    torch, wdd = env
    cfg = CONFIGS[name]
    _check_overlap(torch, wdd, cfg, cfg.batch or 16384, 3)


@pytest.mark.parametrize("Sy,Sx,batch", [(2, 2, 1), (2, 2, 4), (16, 16, 32), (32, 32, 1024)])
def test_many_small_overlapped_acquisitions(env, Sy, Sx, batch):
    # small scans: the first projection of an acquisition does not fill the GPU, so nothing but
    # the launch protocol keeps acquisition k + 2's projection from writing the coefficient store
    # that acquisition k's row FFT still reads (the row FFT triggers its dependents only once its
    # C tiles are in shared memory)
    torch, wdd = env
    _check_overlap(torch, wdd, CONFIGS["medium"].with_(Sy=Sy, Sx=Sx), batch, 12)


@pytest.mark.parametrize("name,Sy,batch,acc,cadence", [("medium", 128, 512, "G", 0), ("medium", 128, 512, "G", 8),
                                                        ("medium", 128, 512, "spectrum", 4), ("medium", 2, 1, "G", 0),
                                                        ("medium", 32, 256, "G", 1), ("large", 256, 16384, "G", 0)])
def test_pipelined_readouts_match_isolated(env, name, Sy, batch, acc, cadence):
    # readout_async: each readout runs on the plan's readout stream while the next acquisition's
    # projections run on the plan stream (mid-acquisition readouts too, Live cadence)
    torch, wdd = env
    cfg = CONFIGS[name]
    cfg = cfg.with_(Sy=Sy, Sx=Sy) if Sy != cfg.Sy else cfg
    _check_overlap(torch, wdd, cfg, batch, 12 if cfg.S <= 1024 else 4, readout_async=True, accumulator=acc,
                   cadence=cadence)


def test_overlapped_acquisitions_without_wide_first_launch():
    # WDD_PROJ_WIDE_FIRST=0: the first projection of an acquisition takes the narrow grid (the
    # environment knob is read once per process, hence the subprocess)
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import importlib.util, torch, paper_2212_01309_b200 as w; from synth import CONFIGS; "
            "s = importlib.util.spec_from_file_location('ovl', 'tests/test_gpu_overlap.py'); "
            "t = importlib.util.module_from_spec(s); s.loader.exec_module(t); "
            "t._check_overlap(torch, w, CONFIGS['medium'].with_(Sy=32, Sx=32), 256, 12); "
            "t._check_overlap(torch, w, CONFIGS['medium'], 512, 4); print('ok')")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, WDD_PROJ_WIDE_FIRST="0"))
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_readout_async_api(env):
    # a shard group keeps its collectives on the plan stream: rejected at create; readout(wait=True)
    # orders torch's current stream after the readout stream (no device synchronisation in between)
    torch, wdd = env
    cfg = CONFIGS["medium"].with_(Sy=32, Sx=32)
    with pytest.raises(wdd.WddError):
        wdd.Plan.from_config(cfg, k_shards=2, k_rank=0, readout_async=True)
    from synth.sparse import dense_frames_torch, sparse_events
    idx = np.arange(cfg.S)
    fr = dense_frames_torch(*sparse_events(5, idx, cfg.Q), cfg.Q, "cuda")
    ref = wdd.Plan.from_config(cfg)
    ref.ingest(fr, idx.astype(np.int32))
    want = ref.readout().cpu().numpy()
    plan = wdd.Plan.from_config(cfg, readout_async=True)
    for _ in range(3):
        plan.reset()
        plan.ingest(fr, idx.astype(np.int32))
        img = plan.readout()                  # wait=True: the copy below is stream-ordered after it
        host = torch.empty_like(img, device="cpu").pin_memory()
        host.copy_(img, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        assert np.array_equal(host.numpy(), want)
    plan.close()
    ref.close()
