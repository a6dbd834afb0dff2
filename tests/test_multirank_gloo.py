"""World-size-2 checks of the multi-rank combine on CPU (gloo): the scan rows are split across
ranks exactly as bench.py does, each rank forms its partial accumulator and Wiener-filtered
spectrum with the oracle, and an allreduce of the spectra equals the single-rank result
(linearity of Algorithm 2, "merge ... sums up the contributions")."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import oracle as O
    from synth import CONFIGS, Acquisition
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = CONFIGS["tiny"]
    g = O.geometry(cfg)
    rows = np.array_split(np.arange(cfg.Sy), world)[rank]          # bench.py's sharding
    idx = (rows[:, None] * cfg.Sx + np.arange(cfg.Sx)[None, :]).reshape(-1)
    fr = Acquisition(cfg).frames(idx)
    Psi = O.hg_basis(cfg.Q, cfg.L, g.sigma)
    C = O.vec(O.project(fr.astype(np.float64), Psi))
    G = O.accumulate_fft(C, idx, cfg.Sy, cfg.Sx)
    act = O.active_set(g, cfg.Sy, cfg.Sx)
    W = O.wiener_bank(g, Psi, act, cfg.Sy, cfg.Sx, cfg.eps)
    o = torch.from_numpy(O.readout_spectrum(G[act], W, act, cfg.Sy, cfg.Sx))
    o_re, o_im = o.real.contiguous(), o.imag.contiguous()
    dist.all_reduce(o_re)
    dist.all_reduce(o_im)
    Gt = torch.from_numpy(G[act].real.copy())
    dist.all_reduce(Gt)
    if rank == 0:
        q.put((o_re.numpy() + 1j * o_im.numpy(), Gt.numpy(), len(idx)))
    dist.destroy_process_group()


def test_two_rank_row_shards_allreduce_equals_single_rank():
    import oracle as O
    from synth import CONFIGS, Acquisition
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    o_sum, G_sum, n0 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = CONFIGS["tiny"]
    idx = np.arange(cfg.S)
    r = O.reduced_wdd(Acquisition(cfg).frames(idx), idx, O.geometry(cfg), cfg.Sy, cfg.Sx, cfg.L, cfg.eps,
                      return_all=True)
    assert n0 == cfg.S // 2
    assert np.max(np.abs(o_sum - r["o"])) < 1e-10 * np.max(np.abs(r["o"]))
    assert np.max(np.abs(G_sum - r["G"][r["active"]].real)) < 1e-10 * np.max(np.abs(r["G"]))
    O_img = O.image_from_spectrum(o_sum)
    assert np.max(np.abs(O_img - r["O"])) < 1e-10 * np.max(np.abs(r["O"]))


def _shard_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import oracle as O
    import bench
    from synth import CONFIGS, Acquisition
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    # bench.py's schedules (the multi-GPU host logic): every scan position is ingested by exactly
    # one rank and marked remote by every other; all ranks read out at the same points
    for cfg, part, batch in ((CONFIGS["medium"], "rows", 512), (CONFIGS["live"], "rr", 1024),
                             (CONFIGS["box"], "rows", 8192)):
        sch = bench._schedule(cfg, world, rank, batch, part)
        own = np.concatenate([s[2] for s in sch if s[0] == "ingest"])
        rem = np.concatenate([s[2] for s in sch if s[0] == "remote"])
        marks = [i for i, s in enumerate(sch) if s[0] == "readout"]
        gathered = [None] * world
        dist.all_gather_object(gathered, (own, rem, marks))
        out[cfg.name] = gathered
    # the coefficient-shard decomposition of the readout (wdd.h shard groups): rank r owns rows
    # a in [r L / n, (r+1) L / n) of H(I); its partial readout over those k, allreduced, is o
    cfg = CONFIGS["tiny"]
    idx = np.arange(cfg.S)
    r_all = O.reduced_wdd(Acquisition(cfg).frames(idx), idx, O.geometry(cfg), cfg.Sy, cfg.Sx, cfg.L, cfg.eps,
                          return_all=True)
    a0, a1 = rank * cfg.L // world, (rank + 1) * cfg.L // world
    ks = slice(a0 * cfg.L, a1 * cfg.L)
    o = np.zeros(cfg.S, dtype=np.complex128)
    o[r_all["active"]] = np.sum(r_all["G"][r_all["active"]][:, ks] * r_all["W"][:, ks], axis=1)
    t = torch.from_numpy(np.stack([o.real, o.imag]))
    dist.all_reduce(t)
    out["o"] = (t[0].numpy() + 1j * t[1].numpy(), r_all["o"].reshape(-1), (a0, a1))
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


def test_two_rank_shard_schedules_and_coefficient_split():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from synth import CONFIGS
    for name in ("medium", "live", "box"):
        cfg = CONFIGS[name]
        (own0, rem0, m0), (own1, rem1, m1) = out[name]
        assert m0 == m1
        assert len(np.intersect1d(own0, own1)) == 0
        assert np.array_equal(np.sort(np.concatenate([own0, own1])), np.arange(cfg.S))
        assert np.array_equal(np.sort(rem0), np.sort(own1)) and np.array_equal(np.sort(rem1), np.sort(own0))
    o_sum, o_ref, _ = out["o"]
    assert np.max(np.abs(o_sum - o_ref)) < 1e-12 * np.max(np.abs(o_ref))
