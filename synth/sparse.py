"""Seeded sparse counting-detector frames for full-size parity runs (test-input generator only).

At the Large / Live / Box sizes (65 536 to 1 048 576 frames of up to 256 x 256 pixels) the
forward simulator costs minutes of host time and the frames do not fit host memory at once.
These frames keep the counting-detector format of the real workloads (uint16 counts, DC pixel at
(Q/2, Q/2)) with a bright-field cluster plus scattered electrons, but are described by a short
list of (pixel, count) events per frame, so both sides can regenerate any batch cheaply:
the GPU side materialises dense frames on the device batch by batch, the oracle evaluates the
projection on the events directly.  No arithmetic of the reconstruction method lives here.

Recipe: frame s holds `events` electrons-hits; a fraction `bf` of them inside the disc of radius
`r_bf` px around the centre (uniform in the disc), the rest uniform over the detector; counts
U{1..max_count}.  Random numbers come from default_rng([seed, 7, block]) for blocks of
`BLOCK` consecutive scan positions, so any batch aligned to the block grid is reproducible.
"""
from __future__ import annotations

import numpy as np

BLOCK = 1024


def _block(seed, b, Q, events, r_bf, bf, max_count):
    rng = np.random.default_rng([seed, 7, b])
    n_bf = int(round(events * bf))
    ang = rng.random((BLOCK, n_bf)) * 2 * np.pi
    rad = np.sqrt(rng.random((BLOCK, n_bf))) * r_bf
    my_bf = np.clip(np.rint(Q // 2 + rad * np.sin(ang)), 0, Q - 1).astype(np.int64)
    mx_bf = np.clip(np.rint(Q // 2 + rad * np.cos(ang)), 0, Q - 1).astype(np.int64)
    my_df = rng.integers(0, Q, size=(BLOCK, events - n_bf))
    mx_df = rng.integers(0, Q, size=(BLOCK, events - n_bf))
    pix = np.concatenate([my_bf * Q + mx_bf, my_df * Q + mx_df], axis=1)
    cnt = rng.integers(1, max_count + 1, size=(BLOCK, events)).astype(np.uint16)
    return pix, cnt


def sparse_events(seed, idx, Q, events=12, r_bf=None, bf=0.75, max_count=200):
    """Events of the frames at scan positions `idx` (any order): pixel indices my*Q + mx (int64)
    and counts (uint16), each of shape (len(idx), events).  Duplicate pixels add."""
    idx = np.asarray(idx, dtype=np.int64)
    if r_bf is None:
        r_bf = 0.2 * Q
    pix = np.empty((len(idx), events), dtype=np.int64)
    cnt = np.empty((len(idx), events), dtype=np.uint16)
    blocks = idx // BLOCK
    for b in np.unique(blocks):
        sel = np.nonzero(blocks == b)[0]
        p, c = _block(seed, int(b), Q, events, r_bf, bf, max_count)
        pix[sel] = p[idx[sel] % BLOCK]
        cnt[sel] = c[idx[sel] % BLOCK]
    return pix, cnt


def dense_frames_numpy(pix, cnt, Q):
    """Dense (n, Q, Q) uint16 frames of the events (host; small cases and pins only)."""
    n = pix.shape[0]
    out = np.zeros((n, Q * Q), dtype=np.uint32)
    np.add.at(out, (np.repeat(np.arange(n), pix.shape[1]), pix.reshape(-1)), cnt.reshape(-1).astype(np.uint32))
    assert out.max(initial=0) < 65536
    return out.astype(np.uint16).reshape(n, Q, Q)


def dense_frames_torch(pix, cnt, Q, device):
    """Same frames materialised on a CUDA device with torch (index_put with accumulation)."""
    import torch
    n = pix.shape[0]
    p = torch.from_numpy(pix).to(device)
    c = torch.from_numpy(cnt.astype(np.int32)).to(device)
    flat = torch.zeros(n * Q * Q, dtype=torch.int32, device=device)
    base = (torch.arange(n, device=device, dtype=torch.int64) * (Q * Q))[:, None]
    flat.index_put_(((base + p).reshape(-1),), c.reshape(-1), accumulate=True)
    return flat.to(torch.uint16).reshape(n, Q, Q)
