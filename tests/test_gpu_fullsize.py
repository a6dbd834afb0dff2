"""GPU parity at BASELINE.json's full sizes (Large, Live, Box), in the launch configuration of
each workload (Live: 1024-frame batches with a readout every 64 scan rows; Large: one single
ingest; Box: the whole 1024 x 1024 scan on one GPU).

The frames are seeded sparse counting-detector frames (synth/sparse.py): the forward simulator
would need minutes of host time per workload, and the projection's cost does not depend on
frame content.  The oracle evaluates, one sampled scan frequency at a time,
  G[v, :] = sum_s f_s[v] H(I_s)          (eq:outer_prod P:424, H of P:361 on the frame events)
  o_v     = sum_k G[v, k] K_v[k]          (bank of Algorithm 1)
and the GPU's o_v is read back from its image (o = DFT2_unitary(conj O), the inverse of P:531).
Tolerance: relative L2 <= 1e-4 (north star); the active set is compared bit-exactly."""
import numpy as np
import pytest

import oracle as O
from synth import CONFIGS
from synth.sparse import dense_frames_torch, sparse_events

pytestmark = pytest.mark.gpu
TOL = 1e-4
SEED = 1234
N_SAMPLE = 48


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


def _run(env, name, batch, readout_rows):
    torch, wdd = env
    cfg = CONFIGS[name]
    g = O.geometry(cfg)
    Psi = O.hg_basis(cfg.Q, cfg.L, g.sigma)
    plan = wdd.Plan.from_config(cfg)
    act = plan.active_set()
    rng = np.random.default_rng(SEED)
    v_s = np.concatenate([[0], rng.choice(act[act != 0], N_SAMPLE - 1, replace=False)]).astype(np.int64)
    assert 0 in set(act.tolist())
    G_ref = np.zeros((len(v_s), cfg.K), dtype=np.complex128)
    mid = None
    rows_done = 0
    for a in range(0, cfg.S, batch):
        idx = np.arange(a, min(cfg.S, a + batch))
        pix, cnt = sparse_events(SEED, idx, cfg.Q)
        plan.ingest(dense_frames_torch(pix, cnt, cfg.Q, "cuda"), idx)
        G_ref += O.accumulate_at(O.project_events(pix, cnt, Psi), idx, v_s, cfg.Sy, cfg.Sx)
        rows = (idx[-1] + 1) // cfg.Sx
        if readout_rows and rows - rows_done >= readout_rows:
            rows_done = rows
            out = plan.readout()
            if mid is None:                        # first live readout: a partial scan
                torch.cuda.synchronize()
                mid = (out.cpu().numpy(), G_ref.copy())
    G_gpu, order = plan.get_accumulator()
    pos = {int(v): i for i, v in enumerate(order)}
    G_s = G_gpu[torch.from_numpy(np.array([pos[int(v)] for v in v_s])).cuda()].cpu().numpy()
    W = O.wiener_bank(g, Psi, v_s, cfg.Sy, cfg.Sx, cfg.eps)
    out = plan.readout()
    torch.cuda.synchronize()
    return dict(cfg=cfg, plan=plan, act=act, v_s=v_s, G_ref=G_ref, G_s=G_s, W=W,
                img=out.cpu().numpy(), mid=mid)


def _check(r):
    cfg, v_s = r["cfg"], r["v_s"]
    e_G = rel(r["G_s"], r["G_ref"])
    assert e_G < TOL, e_G
    # G without the DC-dominated v = 0 row and k = 0 column: the small entries must hold too
    e_G_ac = rel(r["G_s"][1:, 1:], r["G_ref"][1:, 1:])
    assert e_G_ac < TOL, e_G_ac
    o_ref = np.sum(r["G_ref"] * r["W"], axis=1)
    o_gpu = np.fft.fft2(np.conj(r["img"].astype(np.complex128)), norm="ortho").reshape(-1)
    e_o = rel(o_gpu[v_s], o_ref)
    assert e_o < TOL, e_o
    inactive = np.ones(cfg.S, bool)
    inactive[r["act"]] = False
    # the image carries no energy at inactive frequencies beyond float32 rounding of the image
    assert np.max(np.abs(o_gpu[inactive])) < 1e-5 * np.max(np.abs(o_gpu)), "energy at inactive v"
    if r["mid"] is not None:
        img, G_mid = r["mid"]
        o_mid = np.fft.fft2(np.conj(img.astype(np.complex128)), norm="ortho").reshape(-1)
        assert rel(o_mid[v_s], np.sum(G_mid * r["W"], axis=1)) < TOL
    return e_G, e_G_ac, e_o


def test_large_single_pass(env):
    cfg = CONFIGS["large"]
    r = _run(env, "large", cfg.S, 0)        # "Ingest in a single pass"
    print("large", _check(r))


def test_live_streaming_cadence(env):
    cfg = CONFIGS["live"]
    r = _run(env, "live", cfg.batch, cfg.readout_rows)   # 1024-frame batches, readout every 64 rows
    print("live", _check(r))
    # the exact active set at full size (bit-exact integer work)
    assert np.array_equal(np.sort(r["act"]), O.active_set(O.geometry(cfg), cfg.Sy, cfg.Sx))


def test_box_full_scan_one_gpu(env):
    r = _run(env, "box", 16384, 0)
    print("box", _check(r))


@pytest.mark.parametrize("accumulator", ["G", "spectrum"])
def test_live_repeated_scans_deterministic(env, accumulator):
    # The Live cadence runs the pipelined tensor-core flush (rgemm_kernel): a warp-specialised
    # kernel with several barrier rings.  Three back-to-back scans on one plan, every readout of
    # every scan compared bit for bit with the first scan's: a synchronisation error anywhere in
    # the ring protocol shows up as a changed byte (or a hang / fault) long before it shows up in a
    # relative-L2 comparison.
    torch, wdd = env
    cfg = CONFIGS["live"]
    pool_n = 4096
    pool = dense_frames_torch(*sparse_events(SEED, np.arange(pool_n), cfg.Q), cfg.Q, "cuda")
    plan = wdd.Plan.from_config(cfg, accumulator=accumulator)
    scans = []
    for _ in range(3):
        plan.reset()
        outs = []
        done = 0
        for a in range(0, cfg.S, cfg.batch):
            plan.ingest(pool[a % pool_n:a % pool_n + cfg.batch], np.arange(a, a + cfg.batch, dtype=np.int32))
            rows = (a + cfg.batch) // cfg.Sx
            if rows - done >= cfg.readout_rows:
                done = rows
                outs.append(plan.readout().clone())
        torch.cuda.synchronize()
        scans.append(torch.stack(outs).cpu().numpy())
    assert scans[0].shape[0] == cfg.Sy // cfg.readout_rows
    assert np.all(np.isfinite(scans[0]))
    for s in scans[1:]:
        assert np.array_equal(s, scans[0])
