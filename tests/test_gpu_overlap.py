"""Back-to-back acquisitions with overlap: a reset after ingests swaps the plan's two coefficient
stores, so the next acquisition's first projection is launched programmatically (PDL) behind the
previous acquisition's readout instead of after it.  The readouts must be bit-identical to the
same acquisitions run one at a time with a device synchronisation in between (same kernels, same
arithmetic: any race on the coefficient store, R, G or the partial readouts shows up as a
difference), both eagerly and inside one captured CUDA graph (bench.py's step graph)."""
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


@pytest.mark.parametrize("name", ["medium", "large"])
def test_overlapped_acquisitions_match_isolated(env, name):
    torch, wdd = env
    from synth.sparse import dense_frames_torch, sparse_events
    cfg = CONFIGS[name]
    idx = np.arange(cfg.S)
    b = cfg.batch or 16384
    acqs = [dense_frames_torch(*sparse_events(seed, idx, cfg.Q), cfg.Q, "cuda") for seed in (11, 12, 13)]
    plan = wdd.Plan.from_config(cfg)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    def acquire(fr, out):
        plan.reset()
        for a in range(0, cfg.S, b):
            plan.ingest(fr[a:a + b], idx[a:a + b].astype(np.int32), stream)
        plan.readout(out)

    iso = []
    for fr in acqs:
        out = torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device="cuda")
        acquire(fr, out)
        torch.cuda.synchronize()
        iso.append(out.cpu().numpy())
    assert not np.array_equal(iso[0], iso[1])

    # eager, no synchronisation between the acquisitions
    outs = [torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device="cuda") for _ in acqs]
    for fr, out in zip(acqs, outs):
        acquire(fr, out)
    torch.cuda.synchronize()
    for k, out in enumerate(outs):
        assert np.array_equal(out.cpu().numpy(), iso[k]), ("eager", k)

    # one graph holding the three acquisitions, replayed twice
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
