"""World-size-2 GPU parity of the NCCL combine (§8 a7, §8(e)): two processes, one GPU each, split
the scan rows (bench.py's sharding), each ingests its rows into its own plan, and the collective
wdd_readout must give every rank the oracle's image of the whole scan (the merge
sums the partitions).  Needs two visible GPUs; skipped otherwise (this build's boxes have one --
tests/test_gpu_combine.py runs the same path on a one-rank communicator)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, variant, q):
    import torch
    import torch.distributed as dist
    import paper_2212_01309_b200 as wdd
    from synth import CONFIGS, Acquisition
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    cfg = CONFIGS["medium"]
    rows = np.array_split(np.arange(cfg.Sy), world)[rank]
    idx = (rows[:, None] * cfg.Sx + np.arange(cfg.Sx)[None, :]).reshape(-1).astype(np.int32)
    fr = torch.from_numpy(Acquisition(cfg).frames_parallel(idx)).cuda()
    combine, acc = variant
    plan = wdd.Plan.from_config(cfg, device=rank, combine=combine, accumulator=acc)
    obj = [wdd.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    plan.set_comm(world, rank, obj[0])
    for a in range(0, len(idx), cfg.batch):
        plan.ingest(fr[a:a + cfg.batch], idx[a:a + cfg.batch])
    img = plan.readout().cpu().numpy()
    q.put((rank, img))
    plan.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("variant", [(0, "G"), (1, "G"), (0, "spectrum")])
def test_two_gpu_row_shards_match_oracle(variant):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import oracle as O
    from paper_2212_01309_b200 import build
    from synth import CONFIGS, Acquisition
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, variant, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = CONFIGS["medium"]
    idx = np.arange(cfg.S)
    ref = O.reduced_wdd(Acquisition(cfg).frames_parallel(idx), idx, O.geometry(cfg), cfg.Sy, cfg.Sx, cfg.L,
                        cfg.eps)
    for r in (0, 1):
        e = float(np.linalg.norm(res[r] - ref) / np.linalg.norm(ref))
        assert e < TOL, (r, e)
    assert np.array_equal(res[0], res[1])


def _shard_worker(rank, world, port, q):
    # coefficient-sharded group over NCCL: store handles all-gathered, peers opened with CUDA IPC,
    # round-robin batches (batch b on rank b mod world), collective readouts
    import torch
    import torch.distributed as dist
    import paper_2212_01309_b200 as wdd
    from synth import CONFIGS, Acquisition
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    cfg = CONFIGS["medium"]
    idx = np.arange(cfg.S, dtype=np.int32)
    fr = torch.from_numpy(Acquisition(cfg).frames_parallel(idx)).cuda()
    plan = wdd.Plan.from_config(cfg, device=rank, k_shards=world, k_rank=rank)
    obj = [wdd.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    plan.set_comm(world, rank, obj[0])
    hs = [None] * world
    dist.all_gather_object(hs, plan.shard_store_handle())
    plan.set_shard_peers(world, rank, hs)
    outs = []
    for _ in range(2):
        plan.reset()
        for b, a in enumerate(range(0, cfg.S, cfg.batch)):
            if b % world == rank:
                plan.ingest(fr[a:a + cfg.batch], idx[a:a + cfg.batch])
            else:
                plan.ingest_remote(idx[a:a + cfg.batch])
        outs.append(plan.readout().cpu().numpy())
    q.put((rank, outs))
    torch.cuda.synchronize()
    dist.barrier()
    plan.close()
    dist.destroy_process_group()


def test_two_gpu_coefficient_shards_match_oracle():
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import oracle as O
    from paper_2212_01309_b200 import build
    from synth import CONFIGS, Acquisition
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = CONFIGS["medium"]
    idx = np.arange(cfg.S)
    ref = O.reduced_wdd(Acquisition(cfg).frames_parallel(idx), idx, O.geometry(cfg), cfg.Sy, cfg.Sx, cfg.L,
                        cfg.eps)
    for r in (0, 1):
        for img in res[r]:
            e = float(np.linalg.norm(img - ref) / np.linalg.norm(ref))
            assert e < TOL, (r, e)
    assert np.array_equal(res[0][1], res[1][1])


@pytest.mark.parametrize("combine", ["kshard", "partial"])
def test_bench_two_gpus(combine):
    # bench.py under torchrun on two GPUs (the driver's multi-GPU launch), one short Medium run
    import json
    import subprocess
    import sys
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--config", "medium", "--steps", "4", "--warmup", "3", "--no-cpu-baseline", "--combine", combine]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["combine"] == combine
