"""Seeded forward simulator for synthetic 4D-STEM frames (test-input generator only).

Recipe:
  * object  O = exp(i*phi), phi = sum_a A_a exp(-d_a(r)^2 / (2*0.3^2)), d_a the periodic
    minimum-image distance on the Sy*D x Sx*D torus, sampled at pixel D (the scan step);
    positions ~ U[0, FOV)^2, amplitudes ~ U[lo, hi); rng = default_rng([seed, 0]).
  * probe   p_hat(q) = 1[|q|^2 <= (alpha/lambda)^2] * exp(-i*pi*lambda*df*|q|^2) on the detector
    grid q_m = (m - Q/2)/(Q*D); real-space probe P = centred unitary IDFT of p_hat.
  * frame s=(sy,sx): exit[j,i] = P[j,i] * O[(sy+j-Q/2) mod Sy, (sx+i-Q/2) mod Sx],
    I_s = |centred unitary DFT(exit)|^2  (the paper's eq:forward),
  * dose    counts ~ Poisson(dose * I_s / sum(I_s)) with rng = default_rng([seed, 1, s])
    (the paper's Poisson(nu * I~_s)); counter-based, so any subset of frames
    can be regenerated independently and in parallel.
This module is shared by both sides of every parity test and contains no step of the
reconstruction method itself.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

from .configs import Config


def _cdft2(x):
    """Centred unitary 2-D DFT over the last two axes (DC at index Q/2)."""
    return np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(x, axes=(-2, -1)), norm="ortho"),
                           axes=(-2, -1))


def _cidft2(x):
    return np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(x, axes=(-2, -1)), norm="ortho"),
                           axes=(-2, -1))


class Acquisition:
    """One seeded synthetic acquisition for a Config.

    frames(idx) returns the diffraction patterns for flattened scan indices
    s = sy*Sx + sx (row-major, y outer) as an (n, Q, Q) array in the config's storage
    dtype (uint16 counts or float32), or float64 noise-free intensities scaled to the
    dose when noise=False.
    """

    def __init__(self, cfg: Config, noise: bool = True):
        self.cfg = cfg
        self.noise = noise
        self._phi = None
        self._obj = None
        self._probe = None

    # -- object ---------------------------------------------------------------------
    def phase(self) -> np.ndarray:
        """phi on the Sy x Sx scan raster (radians)."""
        if self._phi is None:
            c = self.cfg
            rng = np.random.default_rng([c.seed, 0])
            Ly, Lx = c.Sy * c.step_A, c.Sx * c.step_A
            pos = rng.uniform(0.0, 1.0, size=(c.n_atoms, 2)) * np.array([Ly, Lx])
            amp = rng.uniform(c.amp_lo, c.amp_hi, size=c.n_atoms)
            phi = np.zeros((c.Sy, c.Sx))
            s2 = 2.0 * c.atom_sigma_A ** 2
            h = int(math.ceil(6.0 * c.atom_sigma_A / c.step_A))
            hy, hx = min(h, (c.Sy - 1) // 2), min(h, (c.Sx - 1) // 2)
            dy = np.arange(-hy, hy + 1)
            dx = np.arange(-hx, hx + 1)
            for (ya, xa), A in zip(pos, amp):
                iy0, ix0 = int(round(ya / c.step_A)), int(round(xa / c.step_A))
                ry = (iy0 + dy) * c.step_A - ya
                rx = (ix0 + dx) * c.step_A - xa
                g = A * np.exp(-(ry[:, None] ** 2 + rx[None, :] ** 2) / s2)
                phi[np.ix_((iy0 + dy) % c.Sy, (ix0 + dx) % c.Sx)] += g
            self._phi = phi
        return self._phi

    def object(self) -> np.ndarray:
        if self._obj is None:
            self._obj = np.exp(1j * self.phase())
        return self._obj

    # -- probe ----------------------------------------------------------------------
    def probe(self) -> np.ndarray:
        """Real-space probe P (Q x Q complex), centred at (Q/2, Q/2)."""
        if self._probe is None:
            c = self.cfg
            lam = c.wavelength_A
            dq = 1.0 / (c.Q * c.step_A)
            q = (np.arange(c.Q) - c.Q // 2) * dq
            q2 = q[:, None] ** 2 + q[None, :] ** 2
            qa = c.alpha_rad / lam
            ph = np.where(q2 <= qa * qa, np.exp(-1j * math.pi * lam * c.defocus_A * q2), 0.0)
            self._probe = _cidft2(ph)
        return self._probe

    # -- frames ---------------------------------------------------------------------
    def intensities(self, idx) -> np.ndarray:
        """Noise-free |cDFT2(P * O_patch)|^2 for scan indices idx (float64, (n,Q,Q))."""
        c = self.cfg
        idx = np.asarray(idx, dtype=np.int64)
        O = self.object()
        P = self.probe()
        sy, sx = idx // c.Sx, idx % c.Sx
        j = np.arange(c.Q) - c.Q // 2
        rows = (sy[:, None] + j[None, :]) % c.Sy          # (n, Q)
        cols = (sx[:, None] + j[None, :]) % c.Sx          # (n, Q)
        patch = O[rows[:, :, None], cols[:, None, :]]     # (n, Q, Q)
        return np.abs(_cdft2(P[None] * patch)) ** 2

    def frames(self, idx, chunk: int = 256) -> np.ndarray:
        c = self.cfg
        idx = np.asarray(idx, dtype=np.int64)
        if not self.noise:
            out = np.empty((len(idx), c.Q, c.Q))
        else:
            out = np.empty((len(idx), c.Q, c.Q),
                           dtype=np.uint16 if c.dtype == "u16" else np.float32)
        for a in range(0, len(idx), chunk):
            sub = idx[a:a + chunk]
            I = self.intensities(sub)
            lam = c.dose * I / I.sum(axis=(1, 2), keepdims=True)
            if not self.noise:
                out[a:a + len(sub)] = lam
                continue
            for t, s in enumerate(sub):
                cnt = np.random.default_rng([c.seed, 1, int(s)]).poisson(lam[t])
                if c.dtype == "u16":
                    assert cnt.max() < 65536, "count overflows uint16"
                out[a + t] = cnt
        return out

    def frames_parallel(self, idx, workers: int | None = None) -> np.ndarray:
        """frames(idx) computed in a process pool (same values, counter-based RNG)."""
        idx = np.asarray(idx, dtype=np.int64)
        workers = workers or min(32, os.cpu_count() or 1)
        if workers <= 1 or len(idx) < 2048:
            return self.frames(idx)
        parts = np.array_split(idx, workers * 4)
        with ProcessPoolExecutor(max_workers=workers) as ex:
            res = list(ex.map(_frames_worker, [(self.cfg, self.noise, p) for p in parts]))
        return np.concatenate(res, axis=0)


def _frames_worker(args):
    cfg, noise, idx = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    return Acquisition(cfg, noise).frames(idx)
