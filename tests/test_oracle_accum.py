"""Pins for the oracle's scan-frequency accumulation G (eq:outer_prod)."""
import math

import numpy as np

import oracle as O


def _rand_C(rng, n, K):
    return rng.normal(size=(n, K))


def test_fft_equals_streaming_outer_products():
    # I_hat = F_2D I computed by FFT must equal sum_s f_s i_s^T summed one
    # scan point at a time -- two different algorithms for the same matrix product.
    rng = np.random.default_rng(1)
    Sy, Sx, K = 6, 10, 5
    idx = rng.permutation(Sy * Sx)[:37]
    C = _rand_C(rng, len(idx), K)
    Gf = O.accumulate_fft(C, idx, Sy, Sx)
    Gs = O.accumulate_stream(C, idx, Sy, Sx)
    assert np.max(np.abs(Gf - Gs)) < 1e-12


def test_dft_matrix_kron_definition():
    # F_2D = F (x) F with F[f, x] = e^{-i 2 pi f x / N} / sqrt(N):
    # build it explicitly with np.kron and compare with accumulate_fft on the full scan.
    rng = np.random.default_rng(2)
    Sy, Sx, K = 4, 6, 3
    Fy = np.exp(-2j * np.pi * np.outer(np.arange(Sy), np.arange(Sy)) / Sy) / math.sqrt(Sy)
    Fx = np.exp(-2j * np.pi * np.outer(np.arange(Sx), np.arange(Sx)) / Sx) / math.sqrt(Sx)
    F2 = np.kron(Fy, Fx)
    I = _rand_C(rng, Sy * Sx, K)
    assert np.max(np.abs(F2 @ I - O.accumulate_fft(I, np.arange(Sy * Sx), Sy, Sx))) < 1e-12


def test_frame_at_origin_gives_flat_rows():
    # f_{s=0} = (1,...,1)/sqrt(S): every row of G equals C_0 / sqrt(S).
    rng = np.random.default_rng(3)
    Sy, Sx, K = 8, 8, 4
    c0 = rng.normal(size=(1, K))
    G = O.accumulate_fft(c0, [0], Sy, Sx)
    assert np.max(np.abs(G - c0 / math.sqrt(Sy * Sx))) < 1e-14


def test_unitarity_parseval():
    rng = np.random.default_rng(4)
    Sy, Sx, K = 8, 12, 6
    C = _rand_C(rng, Sy * Sx, K)
    G = O.accumulate_fft(C, np.arange(Sy * Sx), Sy, Sx)
    assert abs(np.linalg.norm(G) - np.linalg.norm(C)) < 1e-10 * np.linalg.norm(C)


def test_partition_and_order_invariance():
    # "trivial to split into partial sums"; merge "in any particular order".
    rng = np.random.default_rng(5)
    Sy, Sx, K = 8, 8, 5
    C = _rand_C(rng, Sy * Sx, K)
    full = O.accumulate_fft(C, np.arange(Sy * Sx), Sy, Sx)
    perm = rng.permutation(Sy * Sx)
    cuts = np.sort(rng.choice(np.arange(1, Sy * Sx), size=5, replace=False))
    parts = np.split(perm, cuts)
    acc = sum(O.accumulate_fft(C[p], p, Sy, Sx) for p in parts[::-1])
    assert np.max(np.abs(acc - full)) < 1e-12


def test_zero_frame_leaves_accumulator_unchanged():
    Sy, Sx, K = 4, 4, 3
    rng = np.random.default_rng(6)
    C = _rand_C(rng, 5, K)
    idx = np.arange(5)
    a = O.accumulate_fft(C, idx, Sy, Sx)
    b = O.accumulate_fft(np.vstack([C, np.zeros((1, K))]), np.r_[idx, 9], Sy, Sx)
    assert np.array_equal(a, b)
