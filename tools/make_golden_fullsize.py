#!/usr/bin/env python
"""Write tests/golden/fullsize_{large,live,box}.npz: float64 ORACLE values for the whole-array
full-size parity tests (tests/test_gpu_fullsize.py).  Calls only oracle/ (the method) and synth/
(the seeded input generator); nothing here comes from the CUDA path.

Inputs: the seeded sparse counting-detector frames of synth/sparse.py (the GPU side materialises
the same frames on the device).  Per config:
  large  one pass over all 65 536 frames, counts up to 3000 (the projection's second count plane);
         stores the whole spectrum o_v = sum_k G[v,k] K_v[k] at every active v
  live   1024-frame batches, a readout every 64 scan rows (8 readouts); stores o after each
         readout (the frames ingested so far), complex64
  box    the whole 1024 x 1024 scan; stores o (complex64) and G (eq:outer_prod) at every
         active v of 8 whole scan-frequency columns vx, complex64
G is the oracle's FFT accumulation (accumulate_fft, the unitary 2-D scan DFT of the zero-filled
coefficient stack) evaluated in coefficient chunks; the bank is the oracle's wiener_bank
(Algorithm 1) over the oracle's active set.  complex64 storage rounds the float64 values by at most
6e-8 relative, far below the 1e-4 tolerance.

    python tools/make_golden_fullsize.py [large|live|box ...] [--workers 8]
"""
import argparse
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from synth import CONFIGS  # noqa: E402
from synth.sparse import sparse_events  # noqa: E402

SPEC = {  # config -> (sparse-event seed, max count)
    "large": (21, 3000),
    "live": (22, 200),
    "box": (23, 200),
}
OUT = os.path.join(ROOT, "tests", "golden")


def _bank_chunk(args):
    name, v = args
    cfg = CONFIGS[name]
    g = O.geometry(cfg)
    return O.wiener_bank(g, O.hg_basis(cfg.Q, cfg.L, g.sigma), v, cfg.Sy, cfg.Sx, cfg.eps)


def _proj_chunk(args):
    name, seed, mc, idx = args
    cfg = CONFIGS[name]
    g = O.geometry(cfg)
    pix, cnt = sparse_events(seed, idx, cfg.Q, max_count=mc)
    return O.project_events(pix, cnt, O.hg_basis(cfg.Q, cfg.L, g.sigma))


def bank(pool, name, act):
    parts = pool.map(_bank_chunk, [(name, c) for c in np.array_split(act, 256)])
    return np.concatenate(parts, axis=0)


def project(pool, name, idx):
    seed, mc = SPEC[name]
    parts = pool.map(_proj_chunk, [(name, seed, mc, c) for c in np.array_split(idx, max(1, len(idx) // 4096))])
    return np.concatenate(parts, axis=0)


def spectrum(cfg, C, idx, act, W, kc=64, keep=None):
    """o over the active v (and G at the `keep` rows) from coefficient stack C at positions idx,
    G by the oracle's unitary FFT accumulation, one chunk of kc coefficients at a time."""
    o = np.zeros(len(act), dtype=np.complex128)
    Gk = None if keep is None else np.zeros((len(keep), cfg.K), dtype=np.complex128)
    for k0 in range(0, cfg.K, kc):
        G = O.accumulate_fft(C[:, k0:k0 + kc], idx, cfg.Sy, cfg.Sx)
        o += np.sum(G[act] * W[:, k0:k0 + kc], axis=1)
        if keep is not None:
            Gk[:, k0:k0 + kc] = G[keep]
    return o, Gk


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["large", "live", "box"])
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    args = ap.parse_args()
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    with Pool(args.workers) as pool:
        for name in args.configs:
            t0 = time.time()
            cfg = CONFIGS[name]
            seed, mc = SPEC[name]
            act = O.active_set(O.geometry(cfg), cfg.Sy, cfg.Sx)
            W = bank(pool, name, act)
            print(name, "bank", W.shape, f"{time.time() - t0:.0f} s", flush=True)
            meta = dict(seed=seed, max_count=mc, act=act.astype(np.int32))
            if name == "large":
                idx = np.arange(cfg.S)
                C = project(pool, name, idx)
                o, _ = spectrum(cfg, C, idx, act, W, kc=128)
                np.savez(os.path.join(OUT, "fullsize_large.npz"), o=o, **meta)
            elif name == "live":
                rows = cfg.readout_rows
                outs = []
                o = np.zeros(len(act), dtype=np.complex128)
                for r0 in range(0, cfg.Sy, rows):
                    idx = np.arange(r0 * cfg.Sx, (r0 + rows) * cfg.Sx)
                    C = project(pool, name, idx)
                    ob, _ = spectrum(cfg, C, idx, act, W, kc=64)
                    o = o + ob
                    outs.append(o.astype(np.complex64))
                    print(name, "readout", len(outs), f"{time.time() - t0:.0f} s", flush=True)
                np.savez(os.path.join(OUT, "fullsize_live.npz"), o_readouts=np.stack(outs), **meta)
            else:
                idx = np.arange(cfg.S)
                C = project(pool, name, idx)
                print(name, "projected", f"{time.time() - t0:.0f} s", flush=True)
                vx = act % cfg.Sx
                cols, lens = np.unique(vx, return_counts=True)
                # 8 whole columns spread over the scan frequencies, from the shorter half of the
                # columns (keeps the stored file small; every column runs the same kernels)
                short = cols[lens <= np.median(lens)]
                pick = short[np.round(np.linspace(0, len(short) - 1, 8)).astype(int)]
                keep_rows = np.nonzero(np.isin(vx, pick))[0]
                o, Gk = spectrum(cfg, C, idx, act, W, kc=32, keep=act[keep_rows])
                np.savez(os.path.join(OUT, "fullsize_box.npz"), o=o.astype(np.complex64), cols_vx=pick,
                         G_cols_v=act[keep_rows], G_cols=Gk.astype(np.complex64), **meta)
            print(name, "done", f"{time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
