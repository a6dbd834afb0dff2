"""Pins for the oracle's Hermite-Gauss basis.

Each test ties oracle.hermite_functions / hg_basis / project to something other than the
oracle's own formula: numpy's Hermite-polynomial evaluator, the harmonic-oscillator
eigen-equation, numpy's FFT, and orthonormality-derived identities.
"""
import math

import numpy as np
import pytest
from numpy.polynomial import hermite as npH

import oracle as O
from synth import CONFIGS

CFG_QL = [(c.Q, c.L) for c in CONFIGS.values()]


def _explicit_hermite_function(n, u):
    """psi_n(u) = H_n(u) exp(-u^2/2) / sqrt(2^n n! sqrt(pi)) via numpy's physicists' H_n."""
    coef = np.zeros(n + 1)
    coef[n] = 1.0
    return npH.hermval(u, coef) * np.exp(-u * u / 2) / math.sqrt(2.0 ** n * math.factorial(n) * math.sqrt(math.pi))


def test_recurrence_matches_explicit_hermite_polynomials():
    # psi_n = H_n(x/sigma) exp(-x^2/2sigma^2), "proper L2-normalization".
    u = np.linspace(-6, 6, 241)
    psi = O.hermite_functions(u, 21)
    for n in range(21):
        ref = _explicit_hermite_function(n, u)
        assert np.max(np.abs(psi[:, n] - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_ho_eigen_equation_and_energies():
    # eqn:HO-eigenvalueproblem / eqn:HO-eigenenergy with sigma = 1:
    # -psi''/2 + u^2 psi/2 = (n + 1/2) psi.  Second derivative by central differences.
    h = 1e-3
    u = np.arange(-9, 9 + h / 2, h)
    psi = O.hermite_functions(u, 12)
    d2 = (psi[2:] - 2 * psi[1:-1] + psi[:-2]) / h ** 2
    uu = u[1:-1, None]
    lhs = -0.5 * d2 + 0.5 * uu ** 2 * psi[1:-1]
    for n in range(12):
        assert np.max(np.abs(lhs[:, n] - (n + 0.5) * psi[1:-1, n])) < 1e-4


@pytest.mark.parametrize("Q,L", CFG_QL)
def test_gram_orthonormal_at_default_sigma(Q, L):
    # R1/R3: sigma0 = sqrt(Q/2pi), continuous-normalised functions sampled on pixels.
    Psi = O.hg_basis(Q, L, math.sqrt(Q / (2 * math.pi)))
    assert np.max(np.abs(Psi.T @ Psi - np.eye(L))) <= 1e-10


@pytest.mark.parametrize("Q,L", CFG_QL)
def test_parity_even_odd(Q, L):
    # Fig. 2 caption: each psi_n is even or odd about the centre pixel c = Q/2.
    Psi = O.hg_basis(Q, L, math.sqrt(Q / (2 * math.pi)))
    c = Q // 2
    d = np.arange(1, c)
    for n in range(L):
        assert np.allclose(Psi[c + d, n], (-1) ** n * Psi[c - d, n], atol=1e-15, rtol=0)


@pytest.mark.parametrize("Q,L,tol", [(32, 8, 1e-5), (128, 16, 1e-12), (128, 32, 1e-12),
                                     (256, 32, 1e-12), (256, 24, 1e-12)])
def test_dft_eigenfunction_property(Q, L, tol):
    # eqn:eigenfunction-of-FT: F psi_n = i^n psi_n for sigma = 1, width sigma -> 1/sigma.
    # With the e^{-i2pi} DFT of P:403 the eigenvalue is (-i)^n (R4).  Centred unitary DFT
    # by numpy.fft; sigma' = Q/(2 pi sigma).
    sigma = 1.1 * math.sqrt(Q / (2 * math.pi)) if Q >= 128 else math.sqrt(Q / (2 * math.pi))
    Psi = O.hg_basis(Q, L, sigma)
    Psi2 = O.hg_basis(Q, L, Q / (2 * math.pi * sigma))
    F = np.fft.fftshift(np.fft.fft(np.fft.ifftshift(Psi, axes=0), axis=0, norm="ortho"), axes=0)
    for n in range(L):
        err = np.linalg.norm(F[:, n] - (-1j) ** n * Psi2[:, n]) / np.linalg.norm(Psi2[:, n])
        assert err <= tol, (n, err)


def test_single_mode_projects_to_unit_coefficient():
    # H(A) = psi_x^T A^T psi_y.  A[my, mx] = Psi[mx, a0] Psi[my, b0] is the (n_x=a0, n_y=b0)
    # CHO eigenfunction (eqn:CHO-eigenfunction) -> one unit coefficient at k = a0*L + b0 (R5).
    Q, L = 64, 8
    Psi = O.hg_basis(Q, L, math.sqrt(Q / (2 * math.pi)))
    a0, b0 = 5, 2
    A = np.outer(Psi[:, b0], Psi[:, a0])          # rows my, cols mx
    C = O.vec(O.project(A, Psi))
    expect = np.zeros(L * L)
    expect[a0 * L + b0] = 1.0
    assert np.max(np.abs(C - expect)) < 1e-12


def test_projection_linear_and_in_span_roundtrip():
    rng = np.random.default_rng(5)
    Q, L = 64, 8
    Psi = O.hg_basis(Q, L, math.sqrt(Q / (2 * math.pi)))
    A, B = rng.normal(size=(2, Q, Q))
    assert np.allclose(O.project(2 * A - 3 * B, Psi), 2 * O.project(A, Psi) - 3 * O.project(B, Psi),
                       atol=1e-12)
    # in-span A = Psi_y C^T Psi_x^T ... reconstructs C exactly (orthonormal columns)
    Cm = rng.normal(size=(L, L))                  # [a, b]
    A = Psi @ Cm.T @ Psi.T                        # A[my, mx] = sum_ab Psi[my,b] C[a,b] Psi[mx,a]
    assert np.max(np.abs(O.project(A, Psi) - Cm)) < 1e-12


def test_mirror_symmetric_frame_has_no_odd_x_coefficients():
    # A frame even under mx -> 2c - mx projects to zero on odd n_x = a (parity of psi_a).
    rng = np.random.default_rng(7)
    Q, L = 32, 8
    c = Q // 2
    A = rng.random((Q, Q))
    A[:, c + 1:] = A[:, c - 1:0:-1]                # mirror about column c (col 0 has no partner)
    A[:, 0] = 0.0
    H = O.project(A, O.hg_basis(Q, L, math.sqrt(Q / (2 * math.pi))))
    assert np.max(np.abs(H[1::2, :])) < 1e-12 * np.max(np.abs(H))
    assert np.max(np.abs(H[0::2, :])) > 1e-3
