"""GPU parity of coefficient-sharded rank groups (include/wdd.h "coefficient-sharded
rank groups") against the float64 oracle.

A group of n plans (k_shards = n, k_rank = r) splits the coefficient rows a of H(I): every
plan's projection stores each frame's coefficient rows of shard o directly into plan o's
coefficient store, and every plan flushes and reads out only its own coefficients.  The Wiener
readout o_v = sum_k G[v,k] K_v[k] is a sum over k, so the shards' partial spectra add
up to the oracle's o, and their G slices concatenate to the oracle's G (eq:outer_prod).

One GPU is available, so the group's plans live in one process on one device, linked with
wdd_link_shards (the same kernels and the same stores a multi-GPU group reaches through
cudaIpcOpenMemHandle, which test_two_process_ipc_group exercises with two processes on the one
device); the partial spectra are summed here instead of by NCCL, and every call runs on one stream,
which orders each plan's ingests before the readouts.  The frames are partitioned by scan-row
blocks (Box) or round-robin batches (Live), SURVEY §8(e)."""
import os
import socket

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


def _group(wdd, cfg, n, **kw):
    plans = [wdd.Plan.from_config(cfg, k_shards=n, k_rank=r, **kw) for r in range(n)]
    wdd.link_shards(plans)
    return plans


def _ingest(plans, owner, fr_dev, idx):
    for q, p in enumerate(plans):
        if q == owner:
            p.ingest(fr_dev, idx)
        else:
            p.ingest_remote(idx)


def _spectrum(torch, plans):
    return sum(p.readout_spectrum(combine=False).to(torch.complex128) for p in plans)


def _G(plans):
    parts = [p.get_accumulator() for p in plans]
    for p, (G, _) in zip(plans, parts):
        assert G.shape[1] == p.k_count
    assert [p.k_lo for p in plans] == list(np.cumsum([0] + [p.k_count for p in plans[:-1]]))
    return np.concatenate([G.cpu().numpy() for G, _ in parts], axis=1), parts[0][1]


def _oracle(cfg, fr, idx):
    return O.reduced_wdd(fr, idx, O.geometry(cfg), cfg.Sy, cfg.Sx, cfg.L, cfg.eps, return_all=True)


@pytest.mark.parametrize("n", [2, 3, 4])
@pytest.mark.parametrize("accumulator", ["G", "spectrum"])
def test_row_blocks_medium(env, n, accumulator):
    # Box-style partition: rank r ingests scan-row block r in 512-frame batches; a readout of the
    # partial scan after every block, then the whole scan
    torch, wdd = env
    cfg = CONFIGS["medium"]
    idx = np.arange(cfg.S)
    fr = Acquisition(cfg).frames_parallel(idx)
    dev = torch.from_numpy(fr).cuda()
    plans = _group(wdd, cfg, n, accumulator=accumulator)
    assert sum(p.k_count for p in plans) == cfg.K
    blocks = np.array_split(np.arange(cfg.Sy), n)
    done = 0
    for r, rows in enumerate(blocks):
        sel = (rows[:, None] * cfg.Sx + np.arange(cfg.Sx)[None, :]).reshape(-1)
        for a in range(0, len(sel), 512):
            s = sel[a:a + 512]
            _ingest(plans, r, dev[s[0]:s[-1] + 1], s)
        done = sel[-1] + 1
        if r < n - 1:
            spec = _spectrum(torch, plans).cpu().numpy()
            ref = _oracle(cfg, fr[:done], idx[:done])
            assert rel(spec, ref["o"]) < TOL, (r, rel(spec, ref["o"]))
    ref = _oracle(cfg, fr, idx)
    spec = _spectrum(torch, plans)
    img = plans[0].image_from_spectrum(spec.to(torch.complex64))
    assert rel(spec.cpu().numpy(), ref["o"]) < TOL
    assert rel(img.cpu().numpy(), ref["O"]) < TOL
    G, act = _G(plans)
    assert rel(G, ref["G"][act]) < TOL


@pytest.mark.parametrize("n", [2, 8])
def test_round_robin_batches_tiny(env, n):
    # Live-style partition (batch b on rank b mod n), float32 frames, L = 8: n = 8 gives every rank a
    # single coefficient row a (k_count = 8); readouts at 25 / 50 / 100 % of the scan
    torch, wdd = env
    cfg = CONFIGS["tiny"]
    idx = np.arange(cfg.S)
    fr = Acquisition(cfg).frames(idx)
    dev = torch.from_numpy(fr).cuda()
    plans = _group(wdd, cfg, n)
    for b, a in enumerate(range(0, cfg.S, 64)):
        _ingest(plans, b % n, dev[a:a + 64], idx[a:a + 64])
        if a + 64 in (256, 512, cfg.S):
            ref = _oracle(cfg, fr[:a + 64], idx[:a + 64])
            assert rel(_spectrum(torch, plans).cpu().numpy(), ref["o"]) < TOL, a
    G, act = _G(plans)
    assert rel(G, _oracle(cfg, fr, idx)["G"][act]) < TOL


def test_back_to_back_acquisitions_alternate_stores(env):
    # three acquisitions on one group without synchronisation: every reset flips every plan's
    # store parity, and the projections of the next acquisition write the other store of every
    # peer while the previous readout may still read this one
    torch, wdd = env
    cfg = CONFIGS["medium"]
    idx = np.arange(cfg.S)
    plans = _group(wdd, cfg, 2, ingest_overlap=True)
    specs, refs = [], []
    frames = [Acquisition(cfg.with_(seed=40 + k)).frames_parallel(idx) for k in range(3)]
    devs = [torch.from_numpy(f).cuda() for f in frames]
    half = cfg.S // 2
    for k in range(3):
        for p in plans:
            p.reset()
        for b, a in enumerate(range(0, cfg.S, 512)):
            _ingest(plans, 0 if a < half else 1, devs[k][a:a + 512], idx[a:a + 512])
        specs.append(_spectrum(torch, plans))
    torch.cuda.synchronize()
    for k in range(3):
        ref = _oracle(cfg, frames[k], idx)
        assert rel(specs[k].cpu().numpy(), ref["o"]) < TOL, k


def _sampled(cfg, plan, seed=77, n=48):
    act = plan.active_set()
    rng = np.random.default_rng(seed)
    return np.concatenate([[0], rng.choice(act[act != 0], n - 1, replace=False)]).astype(np.int64)


@pytest.mark.parametrize("name,n,rows,step", [("live", 4, 32, 16), ("box", 8, 16, 16), ("box", 3, 12, 6)])
def test_full_geometry_row_subset(env, name, n, rows, step):
    # Live (K = 1024, 4 shards of 256 coefficients: the pipelined tensor-core flush) and Box
    # (K = 576, 8 shards of 72 / 3 shards of 192) geometries on a contiguous row subset, round-robin
    # 1024-frame batches, read out every `step` rows; oracle at 48 sampled active v
    torch, wdd = env
    from synth.sparse import dense_frames_torch, sparse_events
    cfg = CONFIGS[name]
    g = O.geometry(cfg)
    Psi = O.hg_basis(cfg.Q, cfg.L, g.sigma)
    plans = _group(wdd, cfg, n)
    v_s = _sampled(cfg, plans[0])
    W = O.wiener_bank(g, Psi, v_s, cfg.Sy, cfg.Sx, cfg.eps)
    G_ref = np.zeros((len(v_s), cfg.K), dtype=np.complex128)
    r0 = cfg.Sy // 3
    b = 0
    for blk in range(r0, r0 + rows, step):
        sel = np.arange(blk * cfg.Sx, (blk + step) * cfg.Sx)
        for a in range(0, len(sel), 1024):
            s = sel[a:a + 1024]
            pix, cnt = sparse_events(5, s, cfg.Q, max_count=3000)      # counts >= 1024 too
            _ingest(plans, b % n, dense_frames_torch(pix, cnt, cfg.Q, "cuda"), s)
            b += 1
            G_ref += O.accumulate_at(O.project_events(pix, cnt, Psi), s, v_s, cfg.Sy, cfg.Sx)
        spec = _spectrum(torch, plans).cpu().numpy().reshape(-1)
        assert rel(spec[v_s], np.sum(G_ref * W, axis=1)) < TOL, blk
    G, act = _G(plans)
    pos = {int(v): i for i, v in enumerate(act)}
    assert rel(G[[pos[int(v)] for v in v_s]], G_ref) < TOL


def test_group_with_one_rank_communicators(env):
    # every plan of the group has a (one-rank) NCCL communicator, so readouts and accumulator reads
    # take the shard-group path: the barrier collective (empty ordinary kernel, one-element
    # allreduce, empty kernel) before the flush, and the allreduce of o -- the identity on one rank,
    # so each plan still returns its own shard's spectrum; their sum is the oracle's
    torch, wdd = env
    cfg = CONFIGS["medium"]
    idx = np.arange(cfg.S)
    fr = Acquisition(cfg).frames_parallel(idx)
    dev = torch.from_numpy(fr).cuda()
    plans = _group(wdd, cfg, 2)
    for p in plans:
        p.set_comm(1, 0, wdd.nccl_unique_id())
    for k in range(2):                                  # two acquisitions: resets swap the stores
        for p in plans:
            p.reset()
        for b, a in enumerate(range(0, cfg.S, 512)):
            _ingest(plans, b % 2, dev[a:a + 512], idx[a:a + 512])
        spec = sum(p.readout_spectrum().to(torch.complex128) for p in plans)
        imgs = [p.readout() for p in plans]
        ref = _oracle(cfg, fr, idx)
        assert rel(spec.cpu().numpy(), ref["o"]) < TOL, k
        G, act = _G(plans)
        assert rel(G, ref["G"][act]) < TOL, k
        # each plan's image is the image of its own shard's spectrum
        for p, im in zip(plans, imgs):
            own = p.readout_spectrum(combine=False)
            assert rel(im.cpu().numpy(), p.image_from_spectrum(own).cpu().numpy()) < 1e-6


def test_shard_errors(env):
    torch, wdd = env
    cfg = CONFIGS["tiny"]
    with pytest.raises(wdd.WddError) as e:
        wdd.Plan.from_config(cfg, k_shards=2, k_rank=2)
    assert e.value.name == "WDD_E_ARG"
    with pytest.raises(wdd.WddError):
        wdd.Plan.from_config(cfg, k_shards=9, k_rank=0)            # more shards than rows a (L = 8)
    p = wdd.Plan.from_config(cfg, k_shards=2, k_rank=0)
    fr = torch.zeros((4, cfg.Q, cfg.Q), dtype=torch.float32, device="cuda")
    with pytest.raises(wdd.WddError) as e:
        p.ingest(fr, np.arange(4))                                  # peers not linked yet
    assert e.value.name == "WDD_E_STATE"
    q = wdd.Plan.from_config(cfg)
    with pytest.raises(wdd.WddError) as e:
        q.ingest_remote(np.arange(4))                               # not a shard plan
    assert e.value.name == "WDD_E_STATE"
    p1 = wdd.Plan.from_config(cfg, k_shards=2, k_rank=1)
    wdd.link_shards([p, p1])
    p.ingest_remote(np.arange(4))
    with pytest.raises(wdd.WddError) as e:
        p.ingest(fr, np.arange(4))                                  # already marked by the remote call
    assert e.value.name == "WDD_E_DUP"


# ------------------------------------------------------------------ two processes, IPC store handles
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import paper_2212_01309_b200 as wdd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = CONFIGS["medium"]
    idx = np.arange(cfg.S)
    fr = Acquisition(cfg).frames(idx[:cfg.S]) if rank == 0 else None
    obj = [fr]
    dist.broadcast_object_list(obj, src=0)
    dev = torch.from_numpy(obj[0]).cuda()
    plan = wdd.Plan.from_config(cfg, k_shards=world, k_rank=rank)
    hs = [None] * world
    dist.all_gather_object(hs, plan.shard_store_handle())
    plan.set_shard_peers(world, rank, hs)
    rows = np.array_split(np.arange(cfg.Sy), world)
    for r, rr in enumerate(rows):
        sel = (rr[:, None] * cfg.Sx + np.arange(cfg.Sx)[None, :]).reshape(-1).astype(np.int32)
        for a in range(0, len(sel), 512):
            s = sel[a:a + 512]
            if r == rank:
                plan.ingest(dev[s[0]:s[-1] + 1], s)
            else:
                plan.ingest_remote(s)
    torch.cuda.synchronize()          # this process's projections (and their peer stores) are done
    dist.barrier()                    # ... and the other's
    spec = plan.readout_spectrum(combine=False).cpu().numpy()
    G, act = plan.get_accumulator()
    q.put((rank, spec, G.cpu().numpy(), act, plan.k_lo, plan.k_count))
    torch.cuda.synchronize()
    dist.barrier()                    # nobody unmaps a store a peer may still write
    plan.close()
    dist.destroy_process_group()


def test_two_process_ipc_group(env):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r = q.get(timeout=600)
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = CONFIGS["medium"]
    idx = np.arange(cfg.S)
    ref = _oracle(cfg, Acquisition(cfg).frames(idx), idx)
    spec = res[0][0].astype(np.complex128) + res[1][0]
    assert rel(spec, ref["o"]) < TOL
    G = np.concatenate([res[0][1], res[1][1]], axis=1)
    assert res[0][3] == 0 and res[1][3] == res[0][4] and res[0][4] + res[1][4] == cfg.K
    assert rel(G, ref["G"][res[0][2]]) < TOL
