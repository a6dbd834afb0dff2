"""End-to-end pins for the oracle: reduced WDD (Algorithm 2) and full WDD (eq:deconv_mat).

  * DFT-basis substitution: the R-oracle run with the complex DFT basis (L = Q) equals the
    F-oracle exactly -- pins scan DFT, bank, Wiener, zero-frequency extraction, IFFT and
    conj of the reduced machinery against the conventional algorithm.
  * Convergence as K grows (BASELINE north star), read as the truncated Fourier basis
    converging monotonically to full WDD, exact at L = Q (R-conv in DESIGN.md).
  * Recovery of the known synthetic phase object, and sign pins (P:122-126 validation intent).
  * Live == offline.
"""
import math

import numpy as np
import pytest

import oracle as O
from synth import Acquisition


def _corr(Oimg, phi):
    ph = np.angle(Oimg * np.conj(Oimg.mean()))
    return float(np.corrcoef(ph.ravel(), phi.ravel())[0, 1])


def _run(td, frames, L=None, Psi=None, **kw):
    cfg = td["cfg"]
    g = O.geometry(cfg)
    return O.reduced_wdd(frames, td["idx"], g, cfg.Sy, cfg.Sx, L or cfg.L, cfg.eps, Psi=Psi, **kw)


def test_dft_basis_substitution_equals_full_wdd(tiny_data):
    cfg = tiny_data["cfg"]
    g = O.geometry(cfg)
    I4 = tiny_data["clean"].reshape(cfg.Sy, cfg.Sx, cfg.Q, cfg.Q)
    Of = O.full_wdd(I4, g, cfg.eps)
    Or = _run(tiny_data, tiny_data["clean"], L=cfg.Q, Psi=O.fourier_basis(cfg.Q))
    assert np.linalg.norm(Or - Of) / np.linalg.norm(Of) < 1e-12


def test_truncated_fourier_basis_converges_to_full_wdd(tiny_data):
    cfg = tiny_data["cfg"]
    g = O.geometry(cfg)
    I4 = tiny_data["clean"].reshape(cfg.Sy, cfg.Sx, cfg.Q, cfg.Q)
    Of = O.full_wdd(I4, g, cfg.eps)
    act = O.active_set(g, cfg.Sy, cfg.Sx)
    errs = []
    for L in (8, 16, 24, 28, 32):
        Or = _run(tiny_data, tiny_data["clean"], L=L, Psi=O.fourier_basis(cfg.Q, L), active=act)
        a, b = Or - Or.mean(), Of - Of.mean()
        errs.append(np.linalg.norm(a - b) / np.linalg.norm(b))
    assert all(e2 < e1 for e1, e2 in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-12


def test_phase_recovery_full_and_reduced(tiny_data):
    cfg = tiny_data["cfg"]
    g = O.geometry(cfg)
    phi = tiny_data["phi"]
    I4 = tiny_data["clean"].reshape(cfg.Sy, cfg.Sx, cfg.Q, cfg.Q)
    assert _corr(O.full_wdd(I4, g, cfg.eps), phi) >= 0.99
    assert _corr(_run(tiny_data, tiny_data["clean"]), phi) >= 0.94
    assert _corr(_run(tiny_data, tiny_data["noisy"]), phi) >= 0.80


def test_sign_pins():
    # Missing conj flips the phase; a swapped-conj bank (conj(p(q)) p(q+q_hat)) destroys
    # the recovery (corr 0.94 -> -0.24 here).  Needs an aberrated probe so p_hat is complex.
    from synth import CONFIGS
    cfg = CONFIGS["tiny"].with_(defocus_A=100.0)
    acq = Acquisition(cfg, noise=False)
    idx = np.arange(cfg.S)
    g = O.geometry(cfg)
    phi = acq.phase()
    r = O.reduced_wdd(acq.frames(idx), idx, g, cfg.Sy, cfg.Sx, cfg.L, cfg.eps, return_all=True)
    assert _corr(r["O"], phi) > 0.9
    no_conj = np.fft.ifft2(r["o"], norm="ortho")
    assert _corr(no_conj, phi) < -0.9
    W_swapped = np.zeros_like(r["W"])
    for i, v in enumerate(r["active"]):
        qh = O.wdd.scan_shift(v, cfg.Sy, cfg.Sx, cfg.step_A)
        Y = np.conj(O.probe_hat(g)) * O.probe_hat(g, qh)
        H = O.vec(O.project(Y, r["Psi"]))
        W_swapped[i] = np.conj(H) / (np.abs(H) ** 2 + cfg.eps)
    o = O.readout_spectrum(r["G"][r["active"]], W_swapped, r["active"], cfg.Sy, cfg.Sx)
    assert _corr(O.image_from_spectrum(o), phi) < _corr(r["O"], phi) - 0.6


def test_normalised_full_wdd_of_phase_object_is_flat(tiny_data):
    # eq:extract divides by sqrt of the q_hat=0, q=0 value; for a pure phase object
    # the noise-free full-WDD amplitude is then flat.
    cfg = tiny_data["cfg"]
    I4 = tiny_data["clean"].reshape(cfg.Sy, cfg.Sx, cfg.Q, cfg.Q)
    On = O.full_wdd(I4, O.geometry(cfg), cfg.eps, normalize=True)
    a = np.abs(On)
    assert a.std() / a.mean() < 1e-2


def test_live_equals_offline(tiny_data):
    # Algorithm 2 processes frames one at a time; partial sums in any order.
    cfg = tiny_data["cfg"]
    g = O.geometry(cfg)
    Psi = O.hg_basis(cfg.Q, cfg.L, g.sigma)
    fr = tiny_data["noisy"].astype(np.float64)
    C = O.vec(O.project(fr, Psi))
    rng = np.random.default_rng(9)
    perm = rng.permutation(cfg.S)
    G = np.zeros((cfg.S, cfg.K), dtype=np.complex128)
    for part in np.array_split(perm, 7):
        G += O.accumulate_fft(C[part], part, cfg.Sy, cfg.Sx)
    off = O.accumulate_fft(C, np.arange(cfg.S), cfg.Sy, cfg.Sx)
    assert np.max(np.abs(G - off)) < 1e-10 * np.max(np.abs(off))


def test_partial_readouts_are_finite(tiny_data):
    cfg = tiny_data["cfg"]
    g = O.geometry(cfg)
    n = cfg.S // 10
    Oimg = O.reduced_wdd(tiny_data["noisy"][:n], np.arange(n), g, cfg.Sy, cfg.Sx, cfg.L, cfg.eps)
    assert np.all(np.isfinite(Oimg))


def test_generator_is_counter_based():
    # any subset regenerates identically (seeded per frame), so both parity sides see the same frames.
    from synth import CONFIGS
    cfg = CONFIGS["tiny"]
    a = Acquisition(cfg).frames(np.arange(40))
    b = Acquisition(cfg).frames(np.arange(20, 40))
    assert np.array_equal(a[20:], b)


def test_wavelength_textbook_values():
    from synth import wavelength_A
    assert abs(wavelength_A(300) - 0.019687) < 2e-6
    assert abs(wavelength_A(200) - 0.025079) < 2e-6
    assert abs(wavelength_A(60) - 0.048661) < 2e-6


@pytest.mark.slow
def test_medium_phase_recovery():
    from synth import CONFIGS
    cfg = CONFIGS["medium"]
    acq = Acquisition(cfg)
    idx = np.arange(cfg.S)
    Oimg = O.reduced_wdd(acq.frames_parallel(idx), idx, O.geometry(cfg), cfg.Sy, cfg.Sx, cfg.L, cfg.eps)
    assert _corr(Oimg, acq.phase()) >= 0.94
