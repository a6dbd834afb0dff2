"""GPU parity of the spectrum-only accumulator (wdd_plan_opts.accumulator = 1):
each flush adds its increment of the Wiener readout to a running o instead of updating G.  The
readout is linear in G (Algorithm 2, o_v = sum_k G[v,k] K_v[k]), so every readout must
equal the float64 oracle on the frames ingested so far, and G formed on demand must equal the
oracle's G -- same tolerance as the G-mode tests (relative L2 <= 1e-4)."""
import numpy as np
import pytest

import oracle as O
from synth import CONFIGS, Acquisition

pytestmark = pytest.mark.gpu
TOL = 1e-4


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    return torch


@pytest.fixture(scope="module")
def wdd():
    from paper_2212_01309_b200 import build
    build.build()
    import paper_2212_01309_b200 as w
    return w


def _oracle(cfg, fr, idx):
    return O.reduced_wdd(fr, idx, O.geometry(cfg), cfg.Sy, cfg.Sx, cfg.L, cfg.eps, return_all=True)


def _setup(torch, name):
    cfg = CONFIGS[name]
    idx = np.arange(cfg.S)
    fr = Acquisition(cfg, noise=True).frames_parallel(idx)
    return cfg, idx, fr, torch.from_numpy(np.ascontiguousarray(fr)).cuda()


@pytest.mark.parametrize("name", ["tiny", "medium"])
def test_spectrum_full_scan(wdd, torch_cuda, name):
    torch = torch_cuda
    cfg, idx, fr, fr_dev = _setup(torch, name)
    ref = _oracle(cfg, fr, idx)
    plan = wdd.Plan.from_config(cfg, accumulator="spectrum")
    b = cfg.batch or cfg.S
    for a in range(0, cfg.S, b):
        plan.ingest(fr_dev[a:a + b], idx[a:a + b])
    out = plan.readout()
    torch.cuda.synchronize()
    o1 = out.cpu().numpy()
    assert rel(o1, ref["O"]) < TOL
    out2 = plan.readout()                      # nothing new: the running o is unchanged
    torch.cuda.synchronize()
    assert np.array_equal(out2.cpu().numpy(), o1)
    G, act = plan.get_accumulator()            # formed on demand from the coefficient store
    assert rel(G.cpu().numpy(), ref["G"][act]) < TOL
    out3 = plan.readout()                      # forming G does not disturb o
    torch.cuda.synchronize()
    assert np.array_equal(out3.cpu().numpy(), o1)
    plan.sync()


@pytest.mark.parametrize("rows_per_readout", [1, 3, 8])
def test_spectrum_live_cadence(wdd, torch_cuda, rows_per_readout):
    # frames in scan order, readout every r rows: the GEMM flush (few rows) and the FFT flush both
    # feed the running o; every readout equals the oracle on the frames so far
    torch = torch_cuda
    cfg, idx, fr, fr_dev = _setup(torch, "tiny")
    plan = wdd.Plan.from_config(cfg, accumulator="spectrum")
    g_plan = wdd.Plan.from_config(cfg)
    step = rows_per_readout * cfg.Sx
    for n, a in enumerate(range(0, cfg.S, step)):
        b = min(cfg.S, a + step)
        plan.ingest(fr_dev[a:b], idx[a:b])
        g_plan.ingest(fr_dev[a:b], idx[a:b])
        out = plan.readout()
        out_g = g_plan.readout()
        torch.cuda.synchronize()
        assert rel(out.cpu().numpy(), out_g.cpu().numpy()) < 1e-5, b
        if n % 4 == 0 or b == cfg.S:
            assert rel(out.cpu().numpy(), _oracle(cfg, fr[:b], idx[:b])["O"]) < TOL, b


def test_spectrum_partial_rows_random_order(wdd, torch_cuda):
    # random arrival order with readouts in between: rows are flushed several times, partially
    torch = torch_cuda
    cfg, idx, fr, fr_dev = _setup(torch, "tiny")
    rng = np.random.default_rng(11)
    perm = rng.permutation(cfg.S)
    cuts = np.sort(rng.choice(np.arange(1, cfg.S), size=7, replace=False))
    plan = wdd.Plan.from_config(cfg, accumulator="spectrum")
    seen = []
    for k, part in enumerate(np.split(perm, cuts)):
        plan.ingest(fr_dev[torch.from_numpy(part).cuda()].contiguous(), part)
        seen.extend(part.tolist())
        if k % 2 == 1:
            out = plan.readout()
            torch.cuda.synchronize()
            s = np.asarray(seen)
            assert rel(out.cpu().numpy(), _oracle(cfg, fr[s], s)["O"]) < TOL, k
    G, act = plan.get_accumulator()
    ref = _oracle(cfg, fr, idx)
    assert rel(G.cpu().numpy(), ref["G"][act]) < TOL
    out = plan.readout()
    torch.cuda.synchronize()
    assert rel(out.cpu().numpy(), ref["O"]) < TOL


def test_spectrum_reset_and_rejects_non_pow2(wdd, torch_cuda):
    torch = torch_cuda
    cfg, idx, fr, fr_dev = _setup(torch, "tiny")
    plan = wdd.Plan.from_config(cfg, accumulator="spectrum")
    plan.ingest(fr_dev[:300], idx[:300])
    plan.readout()
    plan.reset()
    plan.ingest(fr_dev, idx)
    out = plan.readout()
    torch.cuda.synchronize()
    assert rel(out.cpu().numpy(), _oracle(cfg, fr, idx)["O"]) < TOL
    with pytest.raises(wdd.WddError):
        wdd.Plan.from_config(cfg.with_(Sy=24), accumulator="spectrum")
