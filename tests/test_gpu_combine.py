"""GPU parity of the multi-rank combine (§8 a7) with a real NCCL communicator, and of the readout
variants built on it, against the float64 oracle.

One GPU is available to this build, so the communicator has one rank: wdd_set_comm(1, 0, id)
creates a real NCCL communicator and wdd_readout then takes the combine path exactly as on N
ranks -- the flush's partial readouts are summed into o (n_act, accumulator order) and allreduced
(combine = 0), or the partial G is allreduced and read out (combine = 1, the north star's literal
"partial G ... NCCL-allreduced"), or the running spectrum is allreduced (spectrum-only
accumulator).  Linearity ("trivial parallelization", "merge function sums up the
contributions") makes the N-rank result the sum of N such partial results; the world-size-2
version of this test (tests/test_gpu_multirank.py) runs where two GPUs are visible.

Also here: readout of the spectrum (before the image transform) and the image transform
of a given spectrum, and the ingest_overlap = 0 contract (frames written by a kernel
enqueued right before the ingest)."""
import numpy as np
import pytest

import oracle as O
from synth import CONFIGS, Acquisition

pytestmark = pytest.mark.gpu
TOL = 1e-4


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    from paper_2212_01309_b200 import build
    build.build()
    import paper_2212_01309_b200 as w
    return torch, w


def _data(name):
    cfg = CONFIGS[name]
    idx = np.arange(cfg.S)
    fr = Acquisition(cfg, noise=True).frames_parallel(idx)
    ref = O.reduced_wdd(fr, idx, O.geometry(cfg), cfg.Sy, cfg.Sx, cfg.L, cfg.eps, return_all=True)
    return cfg, idx, fr, ref


_CACHE = {}


def _cached(name):
    if name not in _CACHE:
        _CACHE[name] = _data(name)
    return _CACHE[name]


def _comm_plan(wdd, cfg, **kw):
    plan = wdd.Plan.from_config(cfg, **kw)
    plan.set_comm(1, 0, wdd.nccl_unique_id())
    return plan


@pytest.mark.parametrize("name", ["tiny", "medium"])
@pytest.mark.parametrize("combine,accumulator", [(0, "G"), (1, "G"), (0, "spectrum")])
def test_one_rank_comm_readout_matches_oracle(env, name, combine, accumulator):
    torch, wdd = env
    cfg, idx, fr, ref = _cached(name)
    plan = _comm_plan(wdd, cfg, combine=combine, accumulator=accumulator)
    dev = torch.from_numpy(np.ascontiguousarray(fr)).cuda()
    b = min(cfg.batch or 256, cfg.S // 4)
    half = (cfg.S // 2) // b * b
    for a in range(0, half, b):
        plan.ingest(dev[a:a + b], idx[a:a + b])
    # a partial readout through the combine path, then the rest of the scan
    mid = plan.readout()
    torch.cuda.synchronize()
    ref_mid = O.reduced_wdd(fr[:half], idx[:half], O.geometry(cfg), cfg.Sy, cfg.Sx, cfg.L, cfg.eps)
    assert rel(mid.cpu().numpy(), ref_mid) < TOL
    for a in range(half, cfg.S, b):
        plan.ingest(dev[a:a + b], idx[a:a + b])
    out = plan.readout()
    spec = plan.readout_spectrum()                   # after the combine
    own = plan.readout_spectrum(combine=False)       # this rank's partial spectrum
    img2 = plan.image_from_spectrum(spec)
    torch.cuda.synchronize()
    assert rel(out.cpu().numpy(), ref["O"]) < TOL
    assert rel(spec.cpu().numpy(), ref["o"]) < TOL
    assert rel(own.cpu().numpy(), ref["o"]) < TOL
    assert rel(img2.cpu().numpy(), ref["O"]) < TOL
    # inactive v carry exactly zero in the spectrum
    inactive = np.ones(cfg.S, bool)
    inactive[ref["active"]] = False
    assert np.all(spec.cpu().numpy().reshape(-1)[inactive] == 0)
    G, act = plan.get_accumulator()
    assert rel(G.cpu().numpy(), ref["G"][act]) < TOL
    # non-mutating and deterministic through the collective
    out2 = plan.readout()
    torch.cuda.synchronize()
    assert np.array_equal(out2.cpu().numpy(), out.cpu().numpy())
    info = plan.info()
    assert info["nranks"] == 1 and info["rank"] == 0


def test_one_rank_comm_inside_graph(env):
    # the NCCL combine captured in a CUDA graph (bench.py replays whole acquisitions this way)
    torch, wdd = env
    cfg, idx, fr, ref = _cached("tiny")
    plan = _comm_plan(wdd, cfg)
    dev = torch.from_numpy(np.ascontiguousarray(fr)).cuda()
    st = torch.cuda.Stream()
    out = torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device="cuda")
    plan.capture_begin(st)
    plan.reset()
    for a in range(0, cfg.S, 256):
        plan.ingest(dev[a:a + 256], idx[a:a + 256], st)
    plan.readout(out)
    h = plan.capture_end()
    for _ in range(3):
        out.zero_()
        plan.graph_launch(h, st)
        torch.cuda.synchronize()
        assert rel(out.cpu().numpy(), ref["O"]) < TOL


def test_live_row_subset_with_comm(env):
    # Live geometry (512^2 scan, 256^2 detector, K = 1024) on a seeded row subset -- 16 contiguous
    # rows plus 16 random rows, read out after each group (SURVEY §8(d) fast CI variant) -- through
    # the one-rank combine, against the oracle at 48 sampled active v (eq:outer_prod at those v,
    # bank of Algorithm 1 at those v; the full Live bank is a minute of host time)
    torch, wdd = env
    from synth.sparse import dense_frames_torch, sparse_events
    cfg = CONFIGS["live"]
    g = O.geometry(cfg)
    Psi = O.hg_basis(cfg.Q, cfg.L, g.sigma)
    plan = _comm_plan(wdd, cfg)
    act = plan.active_set()
    rng = np.random.default_rng(77)
    v_s = np.concatenate([[0], rng.choice(act[act != 0], 47, replace=False)]).astype(np.int64)
    W = O.wiener_bank(g, Psi, v_s, cfg.Sy, cfg.Sx, cfg.eps)
    rows_a = np.arange(200, 216)
    rows_b = np.sort(rng.choice(np.setdiff1d(np.arange(cfg.Sy), rows_a), 16, replace=False))
    G_ref = np.zeros((len(v_s), cfg.K), dtype=np.complex128)
    for rows in (rows_a, rows_b):
        idx = (rows[:, None] * cfg.Sx + np.arange(cfg.Sx)[None, :]).reshape(-1)
        for a in range(0, len(idx), cfg.batch):
            ib = idx[a:a + cfg.batch]
            pix, cnt = sparse_events(31, ib, cfg.Q)
            plan.ingest(dense_frames_torch(pix, cnt, cfg.Q, "cuda"), ib)
            G_ref += O.accumulate_at(O.project_events(pix, cnt, Psi), ib, v_s, cfg.Sy, cfg.Sx)
        spec = plan.readout_spectrum().cpu().numpy().reshape(-1)
        assert rel(spec[v_s], np.sum(G_ref * W, axis=1)) < TOL
        img = plan.readout().cpu().numpy()
        o_img = np.fft.fft2(np.conj(img.astype(np.complex128)), norm="ortho").reshape(-1)
        assert rel(o_img[v_s], np.sum(G_ref * W, axis=1)) < TOL


@pytest.mark.parametrize("overlap", [False, True])
def test_frames_from_a_kernel_right_before_ingest(env, overlap):
    # ingest_overlap = 0 (default): the frames may be written by a kernel enqueued on the stream
    # right before wdd_ingest -- here every batch is produced by a device copy (a kernel) from a
    # scrambled source into ONE reused buffer, so a projection reading early would see the
    # previous batch's frames.  ingest_overlap = 1 requires frames complete before the previous
    # library call; the test then produces each batch into its own buffer ahead of time.
    torch, wdd = env
    cfg, idx, fr, ref = _cached("medium")
    src = torch.from_numpy(np.ascontiguousarray(fr)).cuda()
    plan = wdd.Plan.from_config(cfg, ingest_overlap=overlap)
    st = torch.cuda.Stream()
    b = cfg.batch
    with torch.cuda.stream(st):
        if overlap:
            bufs = [src[a:a + b].clone() for a in range(0, cfg.S, b)]
            for k, a in enumerate(range(0, cfg.S, b)):
                plan.ingest(bufs[k], idx[a:a + b], st)
        else:
            buf = torch.empty_like(src[:b])
            for a in range(0, cfg.S, b):
                buf.copy_(src[a:a + b])                 # a kernel writes the frames ...
                plan.ingest(buf, idx[a:a + b], st)      # ... right before the ingest reads them
        out = plan.readout()
    torch.cuda.synchronize()
    assert rel(out.cpu().numpy(), ref["O"]) < TOL


def test_float_frames_range_flag_and_dynamic_range(env):
    # f32 frames are split into fp16 hi + lo planes; values beyond fp16 (|x| > 65504, inf, NaN)
    # cannot be represented and are reported by wdd_check (sticky flag) instead of silently
    # corrupting G.  A frame spanning 1e-3 .. 6e4 (eight decades) stays within the tolerance.
    torch, wdd = env
    cfg = CONFIGS["tiny"]
    g = O.geometry(cfg)
    Psi = O.hg_basis(cfg.Q, cfg.L, g.sigma)
    rng = np.random.default_rng(5)
    fr = (10.0 ** rng.uniform(-3, np.log10(6e4), size=(64, cfg.Q, cfg.Q))).astype(np.float32)
    plan = wdd.Plan.from_config(cfg)
    C = plan.project(torch.from_numpy(fr).cuda()).cpu().numpy()
    plan.check()                                           # in range: no error
    Co = O.vec(O.project(fr.astype(np.float64), Psi))
    assert rel(C, Co) < 1e-5
    bad = fr[:4].copy()
    bad[1, 3, 7] = 7e4
    plan.ingest(torch.from_numpy(bad).cuda(), np.arange(4))
    with pytest.raises(wdd.WddError) as e:
        plan.check()
    assert e.value.name == "WDD_E_RANGE"
    plan.check()                                           # the flag was cleared by the report
    nan = fr[:2].copy()
    nan[0, 0, 0] = np.nan
    plan.reset()
    plan.ingest(torch.from_numpy(nan).cuda(), np.arange(2))
    with pytest.raises(wdd.WddError):
        plan.readout_host()
