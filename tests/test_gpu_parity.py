"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle on the same seeded
inputs.  Tolerance (BASELINE.json north star): relative L2 <= 1e-4 on G and on the complex
image; integer work (active set, accumulator order) bit-exact."""
import math

import numpy as np
import pytest

import oracle as O
from synth import CONFIGS, Acquisition

pytestmark = pytest.mark.gpu
TOL = 1e-4


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


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


def _frames(cfg, idx, noise=True):
    return Acquisition(cfg, noise=noise).frames_parallel(np.asarray(idx))


def _to_dev(torch, fr):
    t = torch.from_numpy(np.ascontiguousarray(fr))
    if t.dtype == torch.uint16:
        pass
    return t.cuda()


@pytest.mark.parametrize("name", ["tiny", "medium"])
def test_plan_tables(wdd, torch_cuda, name):
    cfg = CONFIGS[name]
    plan = wdd.Plan.from_config(cfg)
    g = O.geometry(cfg)
    basis, _, act = plan.tables()
    assert np.max(np.abs(basis - O.hg_basis(cfg.Q, cfg.L, g.sigma))) < 1e-13
    oact = O.active_set(g, cfg.Sy, cfg.Sx)
    assert np.array_equal(np.sort(act), oact)                    # bit-exact set
    key = (act % cfg.Sx).astype(np.int64) * cfg.S + act           # accumulator order (vx, vy)
    assert np.all(np.diff(key) > 0)
    info = plan.info()
    assert info["n_act"] == len(oact)
    assert info["n_vx"] == len(np.unique(oact % cfg.Sx))


@pytest.mark.parametrize("name", ["tiny", "medium", "large"])
def test_bank_matches_oracle(wdd, torch_cuda, name):
    # the plan's bank is built on the GPU in float64 (bank.cu); tables() runs the same kernel
    cfg = CONFIGS[name]
    plan = wdd.Plan.from_config(cfg)
    g = O.geometry(cfg)
    _, W, act = plan.tables(bank=True)
    rng = np.random.default_rng(0)
    sel = np.sort(rng.choice(len(act), size=min(len(act), 300), replace=False))
    Wo = O.wiener_bank(g, O.hg_basis(cfg.Q, cfg.L, g.sigma), act[sel], cfg.Sy, cfg.Sx, cfg.eps)
    assert rel(W[sel], Wo) < 1e-10


def _check_project(wdd, torch, cfg, fr):
    plan = wdd.Plan.from_config(cfg)
    C = plan.project(_to_dev(torch, fr)).cpu().numpy()
    g = O.geometry(cfg)
    Co = O.vec(O.project(fr.astype(np.float64), O.hg_basis(cfg.Q, cfg.L, g.sigma)))
    return rel(C, Co), np.max(np.abs(C - Co)) / np.max(np.abs(Co))


@pytest.mark.parametrize("name,n", [("tiny", 37), ("tiny", 1024), ("medium", 515), ("large", 130), ("live", 33),
                                    ("box", 17)])
def test_projection_parity(wdd, torch_cuda, name, n):
    cfg = CONFIGS[name]
    fr = _frames(cfg, np.arange(n) * 7 % cfg.S)
    r, mx = _check_project(wdd, torch_cuda, cfg, fr)
    assert r < 1e-5 and mx < 1e-5, (r, mx)


@pytest.mark.parametrize("Q,L", [(32, 8), (64, 16), (64, 24), (128, 16), (128, 32), (256, 32), (256, 24)])
def test_projection_high_counts_and_float(wdd, torch_cuda, Q, L):
    # counts >= 1024 exercise the second (high-bit) plane; float frames the fp16 residual plane.
    base = CONFIGS["medium"].with_(Q=Q, L=L, Sy=16, Sx=16)
    rng = np.random.default_rng(Q + L)
    fr16 = rng.integers(0, 65535, size=(9, Q, Q), dtype=np.uint16)
    r, mx = _check_project(wdd, torch_cuda, base, fr16)
    assert r < 1e-5 and mx < 1e-5, (r, mx)
    fr32 = (rng.random((9, Q, Q)) * 1000.0).astype(np.float32)
    r, mx = _check_project(wdd, torch_cuda, base.with_(dtype="f32"), fr32)
    assert r < 1e-5 and mx < 1e-5, (r, mx)


@pytest.mark.parametrize("Q,L", [(128, 16), (256, 32), (64, 8)])
def test_projection_sparse_high_counts(wdd, torch_cuda, Q, L):
    # counts >= 1024 in only a few detector rows: some converter warps need the second count
    # plane while others have already released their rows (mixed per-warp paths)
    base = CONFIGS["medium"].with_(Q=Q, L=L, Sy=16, Sx=16)
    rng = np.random.default_rng(7 * Q + L)
    fr = rng.poisson(3.0, size=(21, Q, Q)).astype(np.uint16)
    for f in range(fr.shape[0]):
        for _ in range(3):
            fr[f, rng.integers(0, Q), rng.integers(0, Q)] = rng.integers(1024, 65535)
    r, mx = _check_project(wdd, torch_cuda, base, fr)
    assert r < 1e-5 and mx < 1e-5, (r, mx)


def _ingest_batches(torch, plan, fr_dev, idx, batch):
    for a in range(0, len(idx), batch):
        plan.ingest(fr_dev[a:a + batch], idx[a:a + batch])


def _oracle_all(cfg, fr, idx):
    g = O.geometry(cfg)
    return O.reduced_wdd(fr, idx, g, cfg.Sy, cfg.Sx, cfg.L, cfg.eps, return_all=True)


@pytest.mark.parametrize("name", ["tiny", "medium"])
def test_full_scan_parity(wdd, torch_cuda, name):
    torch = torch_cuda
    cfg = CONFIGS[name]
    idx = np.arange(cfg.S)
    fr = _frames(cfg, idx)
    ref = _oracle_all(cfg, fr, idx)
    plan = wdd.Plan.from_config(cfg)
    fr_dev = _to_dev(torch, fr)
    _ingest_batches(torch, plan, fr_dev, idx, cfg.batch or cfg.S)
    G, act = plan.get_accumulator()
    G = G.cpu().numpy()
    assert rel(G, ref["G"][act]) < TOL
    out = plan.readout()
    torch.cuda.synchronize()
    Oimg = out.cpu().numpy()
    assert rel(Oimg, ref["O"]) < TOL
    # non-mutating: a second readout is bit-identical
    out2 = plan.readout()
    torch.cuda.synchronize()
    assert np.array_equal(out2.cpu().numpy(), Oimg)
    plan.sync()   # raises if a device-side wait timed out


def test_live_equals_offline_random_partitions(wdd, torch_cuda):
    torch = torch_cuda
    cfg = CONFIGS["tiny"]
    idx = np.arange(cfg.S)
    fr = _frames(cfg, idx)
    fr_dev = _to_dev(torch, fr)
    off = wdd.Plan.from_config(cfg)
    off.ingest(fr_dev, idx)
    G_off, _ = off.get_accumulator()
    rng = np.random.default_rng(3)
    perm = rng.permutation(cfg.S)
    live = wdd.Plan.from_config(cfg)
    cuts = np.sort(rng.choice(np.arange(1, cfg.S), size=9, replace=False))
    for k, part in enumerate(np.split(perm, cuts)):
        live.ingest(fr_dev[torch.from_numpy(part).cuda()].contiguous(), part)
        if k == 4:  # a readout in the middle must not disturb the running sum
            live.readout()
    G_live, _ = live.get_accumulator()
    assert rel(G_live.cpu().numpy(), G_off.cpu().numpy()) < 1e-5
    ref = _oracle_all(cfg, fr, idx)
    out = live.readout()
    torch.cuda.synchronize()
    assert rel(out.cpu().numpy(), ref["O"]) < TOL


def test_partial_rows_and_partial_readout(wdd, torch_cuda):
    # contiguous chunks that split scan rows, read out at 10 % and 55 % of the scan
    torch = torch_cuda
    cfg = CONFIGS["tiny"]
    idx = np.arange(cfg.S)
    fr = _frames(cfg, idx)
    fr_dev = _to_dev(torch, fr)
    plan = wdd.Plan.from_config(cfg)
    bounds = [0, 45, 102, 563, cfg.S]
    for a, b in zip(bounds, bounds[1:]):
        plan.ingest(fr_dev[a:b], idx[a:b])
        ref = _oracle_all(cfg, fr[:b], idx[:b])
        out = plan.readout()
        torch.cuda.synchronize()
        assert rel(out.cpu().numpy(), ref["O"]) < TOL, b


def test_rejects_duplicates_and_range_without_effect(wdd, torch_cuda):
    torch = torch_cuda
    cfg = CONFIGS["tiny"]
    fr = _frames(cfg, np.arange(8))
    fr_dev = _to_dev(torch, fr)
    plan = wdd.Plan.from_config(cfg)
    plan.ingest(fr_dev[:4], np.arange(4))
    G0, _ = plan.get_accumulator()
    with pytest.raises(wdd.WddError) as e:
        plan.ingest(fr_dev[4:8], [4, 5, 6, 4])
    assert e.value.name == "WDD_E_DUP"
    with pytest.raises(wdd.WddError) as e:
        plan.ingest(fr_dev[4:8], [4, 5, 2, 7])
    assert e.value.name == "WDD_E_DUP"
    with pytest.raises(wdd.WddError) as e:
        plan.ingest(fr_dev[4:8], [4, 5, 6, cfg.S])
    assert e.value.name == "WDD_E_RANGE"
    plan.ingest(fr_dev[:0], [])
    G1, _ = plan.get_accumulator()
    assert torch.equal(G0, G1)
    plan.ingest(fr_dev[4:8], [4, 5, 6, 7])  # the rejected indices are still available
    assert plan.info()["frames_ingested"] == 8
    plan.reset()
    G2, _ = plan.get_accumulator()
    assert float(G2.abs().max()) == 0.0
    plan.ingest(fr_dev[:4], np.arange(4))


def test_contiguous_run_bookkeeping(wdd, torch_cuda):
    # contiguous calls take word-wise host bookkeeping (seen bitmap, pending masks): runs that start
    # and end inside 32- / 64-bit words and scan rows, a run hitting an ingested position in its
    # middle (DUP, nothing marked), runs crossing the scan end or starting past it (RANGE); the
    # accumulator and image must equal the same frames ingested as scattered (non-run) calls
    torch = torch_cuda
    cfg = CONFIGS["tiny"]   # 32 x 32: one 32-bit mask word per row, two rows per 64-bit seen word
    idx = np.arange(cfg.S)
    fr = _frames(cfg, idx)
    fr_dev = _to_dev(torch, fr)
    runs = [(0, 1), (1, 31), (31, 33), (33, 65), (65, 130), (130, 131), (131, 700), (700, cfg.S)]
    plan = wdd.Plan.from_config(cfg)
    plan.ingest(fr_dev[65:130], idx[65:130])
    with pytest.raises(wdd.WddError) as e:
        plan.ingest(fr_dev[40:100], idx[40:100])          # overlaps 65 .. 99
    assert e.value.name == "WDD_E_DUP"
    with pytest.raises(wdd.WddError) as e:
        plan.ingest(fr_dev[cfg.S - 3:], np.arange(cfg.S - 3, cfg.S + 0) + 1)   # ends past the scan
    assert e.value.name == "WDD_E_RANGE"
    with pytest.raises(wdd.WddError) as e:
        plan.ingest(fr_dev[:2], np.array([cfg.S, cfg.S + 1]))
    assert e.value.name == "WDD_E_RANGE"
    with pytest.raises(wdd.WddError) as e:
        plan.ingest(fr_dev[:2], np.array([-1, 0]))
    assert e.value.name == "WDD_E_RANGE"
    for a, b in runs:
        if (a, b) != (65, 130):
            plan.ingest(fr_dev[a:b], idx[a:b])
    assert plan.info()["frames_ingested"] == cfg.S
    out = plan.readout()
    G, _ = plan.get_accumulator()
    # the same frames as scattered calls (every call permuted: never a run)
    ref_plan = wdd.Plan.from_config(cfg)
    rng = np.random.default_rng(7)
    perm = rng.permutation(cfg.S)
    for c in np.array_split(perm, 9):
        c = c if len(c) < 2 or not np.all(np.diff(c) == 1) else c[::-1]
        ref_plan.ingest(fr_dev[torch.from_numpy(c).long().cuda()].contiguous(), c)
    out_ref = ref_plan.readout()
    G_ref, _ = ref_plan.get_accumulator()
    torch.cuda.synchronize()
    assert rel(G.cpu().numpy(), G_ref.cpu().numpy()) < 1e-6
    assert rel(out.cpu().numpy(), out_ref.cpu().numpy()) < 1e-6
    ref = _oracle_all(cfg, fr, idx)
    assert rel(out.cpu().numpy(), ref["O"]) < TOL


def test_normalize_flag(wdd, torch_cuda):
    torch = torch_cuda
    cfg = CONFIGS["tiny"]
    idx = np.arange(cfg.S)
    fr = _frames(cfg, idx)
    plan = wdd.Plan.from_config(cfg, normalize=True)
    plan.ingest(_to_dev(torch, fr), idx)
    out = plan.readout()
    torch.cuda.synchronize()
    ref = O.reduced_wdd(fr, idx, O.geometry(cfg), cfg.Sy, cfg.Sx, cfg.L, cfg.eps, normalize=True)
    assert rel(out.cpu().numpy(), ref) < TOL


def test_host_ingest_equals_device_ingest(wdd, torch_cuda):
    torch = torch_cuda
    cfg = CONFIGS["medium"]
    idx = np.arange(4096)
    fr = _frames(cfg, idx)
    a = wdd.Plan.from_config(cfg)
    a.ingest(_to_dev(torch, fr), idx)
    b = wdd.Plan.from_config(cfg)
    pinned = torch.from_numpy(fr).pin_memory()
    for s in range(0, len(idx), 512):
        b.ingest_host(pinned[s:s + 512], idx[s:s + 512])
    Ga, _ = a.get_accumulator()
    Gb, _ = b.get_accumulator()
    torch.cuda.synchronize()
    assert torch.equal(Ga, Gb)
    host = b.readout_host()
    dev = a.readout()
    torch.cuda.synchronize()
    assert np.array_equal(host, dev.cpu().numpy())


def test_phase_recovery_medium(wdd, torch_cuda):
    torch = torch_cuda
    cfg = CONFIGS["medium"]
    acq = Acquisition(cfg)
    idx = np.arange(cfg.S)
    fr = acq.frames_parallel(idx)
    plan = wdd.Plan.from_config(cfg)
    _ingest_batches(torch, plan, _to_dev(torch, fr), idx, cfg.batch)
    out = plan.readout().cpu().numpy()
    ph = np.angle(out * np.conj(out.mean()))
    assert np.corrcoef(ph.ravel(), acq.phase().ravel())[0, 1] > 0.94


@pytest.mark.parametrize("Sy,Sx", [(24, 40), (32, 20), (20, 32)])
def test_non_power_of_two_scan(wdd, torch_cuda, Sy, Sx):
    # non-power-of-two scan axes take the DFT-matrix kernels for that axis (rowdft / flush)
    torch = torch_cuda
    cfg = CONFIGS["tiny"].with_(Sy=Sy, Sx=Sx)
    idx = np.arange(cfg.S)
    fr = _frames(cfg, idx)
    ref = _oracle_all(cfg, fr, idx)
    plan = wdd.Plan.from_config(cfg)
    _ingest_batches(torch, plan, _to_dev(torch, fr), idx, 100)
    G, act = plan.get_accumulator()
    assert rel(G.cpu().numpy(), ref["G"][act]) < TOL
    out = plan.readout()
    torch.cuda.synchronize()
    assert rel(out.cpu().numpy(), ref["O"]) < TOL


@pytest.mark.parametrize("rows_per_readout", [1, 2, 5, 8, 16])
def test_live_readout_cadence(wdd, torch_cuda, rows_per_readout):
    # frames arrive in scan order; a readout every r rows flushes r staged rows into G (few rows:
    # DFT-matrix rank update; more: FFT along y with the missing rows as zeros).  Every readout
    # must equal the oracle on the frames ingested so far.
    torch = torch_cuda
    cfg = CONFIGS["tiny"]
    idx = np.arange(cfg.S)
    fr = _frames(cfg, idx)
    fr_dev = _to_dev(torch, fr)
    plan = wdd.Plan.from_config(cfg)
    step = rows_per_readout * cfg.Sx
    for a in range(0, cfg.S, step):
        b = min(cfg.S, a + step)
        plan.ingest(fr_dev[a:b], idx[a:b])
        out = plan.readout()
        torch.cuda.synchronize()
        if (a // step) % 3 == 0 or b == cfg.S:
            ref = _oracle_all(cfg, fr[:b], idx[:b])
            assert rel(out.cpu().numpy(), ref["O"]) < TOL, b
    G, act = plan.get_accumulator()
    assert rel(G.cpu().numpy(), _oracle_all(cfg, fr, idx)["G"][act]) < TOL


def test_medium_live_cadence_pruned_flush(wdd, torch_cuda):
    # 128-row scan read out every 32 rows: each flush is an aligned block of 2^5 rows, which takes
    # the pruned y transform (4 FFTs of 32 points instead of one of 128)
    torch = torch_cuda
    cfg = CONFIGS["medium"]
    idx = np.arange(cfg.S)
    fr = _frames(cfg, idx)
    fr_dev = _to_dev(torch, fr)
    plan = wdd.Plan.from_config(cfg)
    step = 32 * cfg.Sx
    for a in range(0, cfg.S, step):
        for b in range(a, a + step, cfg.batch):
            plan.ingest(fr_dev[b:b + cfg.batch], idx[b:b + cfg.batch])
        out = plan.readout()
    torch.cuda.synchronize()
    ref = _oracle_all(cfg, fr, idx)
    assert rel(out.cpu().numpy(), ref["O"]) < TOL
    G, act = plan.get_accumulator()
    assert rel(G.cpu().numpy(), ref["G"][act]) < TOL


def test_back_to_back_acquisitions_same_plan(wdd, torch_cuda):
    # reset -> full scan -> readout, three times on one plan without host synchronisation in
    # between: the launches of one acquisition must not overtake the flush / readout of the last
    torch = torch_cuda
    cfg = CONFIGS["tiny"]
    idx = np.arange(cfg.S)
    fr = _frames(cfg, idx)
    fr_dev = _to_dev(torch, fr)
    plan = wdd.Plan.from_config(cfg)
    s = torch.cuda.Stream()
    outs = []
    for _ in range(3):
        plan.reset()
        for a in range(0, cfg.S, 128):
            plan.ingest(fr_dev[a:a + 128], idx[a:a + 128], s)
        out = torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device="cuda")
        with torch.cuda.stream(s):
            plan.readout(out)
        outs.append(out)
    torch.cuda.synchronize()
    ref = _oracle_all(cfg, fr, idx)["O"]
    for o in outs:
        assert rel(o.cpu().numpy(), ref) < TOL
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


@pytest.mark.parametrize("accumulator", ["G", "spectrum"])
def test_multi_plan_row_shards_sum_to_single_plan(wdd, torch_cuda, accumulator):
    # SURVEY §4 item 5, "multi-GPU without a cluster": three plans on one device ingest disjoint
    # row shards (bench.py's sharding); the sum of their accumulators and of their spectra -- what
    # the NCCL combine of wdd_readout adds up -- equals one plan that ingested everything
    # (linearity of Algorithm 2).
    torch = torch_cuda
    cfg = CONFIGS["medium"].with_(Sy=32, Sx=32)
    idx = np.arange(cfg.S)
    fr_dev = _to_dev(torch, _frames(cfg, idx))
    whole = wdd.Plan.from_config(cfg, accumulator=accumulator)
    _ingest_batches(torch, whole, fr_dev, idx, 100)
    G1, act = whole.get_accumulator()
    img1 = whole.readout()
    Gs, spec = 0, 0
    for rows in np.array_split(np.arange(cfg.Sy), 3):
        sh = (rows[:, None] * cfg.Sx + np.arange(cfg.Sx)[None, :]).reshape(-1)
        p = wdd.Plan.from_config(cfg, accumulator=accumulator)
        _ingest_batches(torch, p, fr_dev[sh[0]:sh[-1] + 1], sh, 77)      # (a shard is a run of rows)
        G, a2 = p.get_accumulator()
        assert np.array_equal(a2, act)
        Gs = Gs + G.cpu().numpy().astype(np.complex128)
        im = p.readout().cpu().numpy().astype(np.complex128)
        spec = spec + np.fft.fft2(np.conj(im), norm="ortho")
    torch.cuda.synchronize()
    assert rel(Gs, G1.cpu().numpy()) < 1e-5
    spec1 = np.fft.fft2(np.conj(img1.cpu().numpy().astype(np.complex128)), norm="ortho")
    assert rel(spec, spec1) < 1e-5
