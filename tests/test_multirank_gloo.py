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
