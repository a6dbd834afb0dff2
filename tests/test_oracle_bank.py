"""Pins for the oracle's probe, autocorrelation, active set and Wiener bank
(Algorithm 1 `Algo:PreCompute` P:441-463; intersection geometry P:465-500)."""
import math

import numpy as np
import pytest

import oracle as O
from synth import CONFIGS


def _geom(name):
    return O.geometry(CONFIGS[name])


def test_zero_shift_autocorrelation_is_aperture_intensity():
    # Y_0 = p_hat conj(p_hat) = |p_hat|^2 = 1 inside the aperture, 0 outside.
    g = _geom("medium")
    Y0 = O.autocorrelation(g, 0, 128, 128)
    q = g.q_grid()
    disc = (q[:, None] ** 2 + q[None, :] ** 2) <= g.q_alpha ** 2
    assert np.max(np.abs(Y0 - disc)) < 1e-15


def test_aperture_pixel_count_matches_disc_area():
    # Number of detector pixels inside the aperture ~ pi R^2 (R = alpha/lambda/dq).
    for name in ["tiny", "medium", "live"]:
        g = _geom(name)
        n = int(np.count_nonzero(O.autocorrelation(g, 0, 8, 8)))
        assert abs(n - math.pi * g.R ** 2) <= 2 * math.pi * g.R * 0.5 + 4, (name, n)


def _lens_area(R, d):
    if d >= 2 * R:
        return 0.0
    return 2 * R * R * math.acos(d / (2 * R)) - 0.5 * d * math.sqrt(4 * R * R - d * d)


@pytest.mark.parametrize("vy,vx", [(0, 5), (3, 0), (7, 11), (20, 9), (-30, 4)])
def test_overlap_lens_area_medium(vy, vx):
    # Medium has S = Q, so q_hat_v shifts the aperture by exactly v~ pixels (R8);
    # the nonzero support of Y_v is the lens of two radius-R discs at distance |v~|.
    g = _geom("medium")
    S = 128
    v = (vy % S) * S + (vx % S)
    n = int(np.count_nonzero(O.autocorrelation(g, v, S, S)))
    A = _lens_area(g.R, math.hypot(vy, vx))
    assert abs(n - A) <= 2 * math.pi * g.R * 0.6 + 4, (n, A)


def test_active_set_equals_brute_force_over_all_frequencies():
    # active_set's prefiltered pixel test == "Y_v has a nonzero pixel" checked on every v.
    cfg = CONFIGS["tiny"]
    g = O.geometry(cfg)
    brute = [v for v in range(cfg.S) if np.any(O.autocorrelation(g, v, cfg.Sy, cfg.Sx))]
    assert np.array_equal(O.active_set(g, cfg.Sy, cfg.Sx), np.array(brute))


@pytest.mark.parametrize("name", ["medium", "large", "live", "box"])
def test_active_set_equals_aperture_self_correlation(name):
    # An independent construction of the exact active set (R9): in units of the scan
    # frequency, the shift q_hat_v is v~ Q / S detector pixels (R8), an integer on the grid refined by
    # F = S / Q.  There, v is active iff v~ = d - a for an aperture pixel a (coarse pixels, scaled by
    # F) and a point d of the aperture disc (fine grid): the support of the cross-correlation of the
    # two indicator arrays, computed by FFT convolution -- no per-v pixel test as in active_set.
    from scipy.signal import fftconvolve
    cfg = CONFIGS[name]
    g = O.geometry(cfg)
    assert cfg.Sy == cfg.Sx and cfg.Sy % cfg.Q == 0
    F = cfg.Sy // cfg.Q
    Rf = g.R * F                                            # disc radius on the fine grid
    h = int(np.ceil(Rf)) + 1
    w = np.arange(-h, h + 1)
    D = (w[:, None] ** 2 + w[None, :] ** 2 <= Rf * Rf).astype(np.float64)
    A = np.zeros_like(D)
    u = np.arange(cfg.Q) - cfg.Q // 2                      # coarse pixel coordinates
    uu = u[np.abs(u) * F <= h]
    inside = uu[:, None] ** 2 + uu[None, :] ** 2 <= g.R * g.R
    iy, ix = np.nonzero(inside)
    A[uu[iy] * F + h, uu[ix] * F + h] = 1.0
    corr = fftconvolve(D, A[::-1, ::-1])                    # corr[t] = sum_a A[a] D[a + t]
    ty, tx = np.nonzero(corr > 0.5)
    ty, tx = ty - 2 * h, tx - 2 * h
    v = np.sort((ty % cfg.Sy) * cfg.Sx + (tx % cfg.Sx))
    assert np.array_equal(v, O.active_set(g, cfg.Sy, cfg.Sx))


@pytest.mark.parametrize("name,n_act", [("tiny", 517), ("medium", 7425), ("large", 29593)])
def test_active_set_counts_and_symmetry(name, n_act):
    # Counts recorded in SURVEY.md Appendix A E6 (exact discrete test).  Symmetry: Y_{-v}(q) =
    # conj(Y_v(q - q_hat_v)) so v and -v are active together; superset of the continuous disc
    # |q_hat| <= 2 q_alpha (triangle inequality).
    cfg = CONFIGS[name]
    g = O.geometry(cfg)
    act = O.active_set(g, cfg.Sy, cfg.Sx)
    assert len(act) == n_act
    vy, vx = act // cfg.Sx, act % cfg.Sx
    neg = ((-vy) % cfg.Sy) * cfg.Sx + ((-vx) % cfg.Sx)
    assert set(neg.tolist()) == set(act.tolist())
    fy = O.signed_freq(cfg.Sy)[vy] / (cfg.Sy * cfg.step_A)
    fx = O.signed_freq(cfg.Sx)[vx] / (cfg.Sx * cfg.step_A)
    assert np.all(np.hypot(fy, fx) <= 2 * g.q_alpha * (1 + 1e-12))


def test_wiener_scalar_identity_and_bound():
    # K_v = conj(H)/(|H|^2 + eps): K*H = |H|^2/(|H|^2+eps) in [0,1), and
    # |K| <= 1/(2 sqrt(eps)) (AM-GM), attained when |H|^2 = eps.
    cfg = CONFIGS["tiny"]
    g = O.geometry(cfg)
    Psi = O.hg_basis(cfg.Q, cfg.L, g.sigma)
    act = O.active_set(g, cfg.Sy, cfg.Sx)
    W = O.wiener_bank(g, Psi, act, cfg.Sy, cfg.Sx, cfg.eps)
    H = np.stack([O.vec(O.project(O.autocorrelation(g, v, cfg.Sy, cfg.Sx), Psi)) for v in act])
    prod = W * H
    assert np.max(np.abs(prod.imag)) < 1e-15
    assert np.all(prod.real >= 0) and np.all(prod.real < 1)
    assert np.max(np.abs(W)) <= 1 / (2 * math.sqrt(cfg.eps)) * (1 + 1e-12)
    # the zero-shift filter is real (Y_0 real, basis real)
    assert np.max(np.abs(W[0].imag)) < 1e-15


def test_paper_pruning_example_golden():
    # tests/golden/paper_pruning_example.txt: P:497-499 prints S_hat = 0.47 S for
    # theta = 32 mrad, Delta = 0.026 nm, lambda = 2.508 pm (eq:low_correlation).
    from pathlib import Path
    vals = {}
    for line in (Path(__file__).parent / "golden" / "paper_pruning_example.txt").read_text().splitlines():
        if line and not line.startswith("#"):
            k, v = line.split("=")
            vals[k.strip()] = float(v)
    r = O.pruning_bound_paper(vals["step_A"], vals["theta_rad"], vals["wavelength_A"])
    assert abs(r - vals["ratio_printed"]) <= 0.005


def test_paper_pruning_bound_is_not_an_exclusion_bound():
    # R9: the printed bound is the inscribed-square half-width.  With the paper's own example
    # geometry, on-axis frequencies up to 2*Delta*theta/lambda*S stay active, beyond 0.47 S.
    S, step, theta, lam = 64, 0.26, 0.032, 0.02508
    g = O.Geometry(Q=64, step_A=step, wavelength_A=lam, alpha_rad=theta)
    act = O.active_set(g, S, S)
    fx = np.abs(O.signed_freq(S)[act % S])
    bound = O.pruning_bound_paper(step, theta, lam) * S
    assert fx.max() > bound
    assert fx.max() <= 2 * step * theta / lam * S + 1
