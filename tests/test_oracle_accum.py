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


def test_accumulate_at_equals_fft_rows():
    # G at selected frequencies (explicit phase rows, integer angle reduction) == the rows of the
    # FFT-computed G (a different algorithm) on a non-square scan with a random index subset.
    rng = np.random.default_rng(11)
    Sy, Sx, K = 12, 20, 6
    idx = rng.permutation(Sy * Sx)[:150]
    C = _rand_C(rng, len(idx), K)
    v = rng.choice(Sy * Sx, size=17, replace=False)
    assert np.max(np.abs(O.accumulate_at(C, idx, v, Sy, Sx) - O.accumulate_fft(C, idx, Sy, Sx)[v])) < 1e-12


def test_scan_phase_large_indices_equals_fft_of_impulse():
    # f_s[v] at 1024 x 1024 against an independent computation: the unitary 2-D FFT of
    # a unit impulse at scan position s is exactly the column f_s of F_2D; checked at every v for
    # scan positions near the ends of both axes (large products vy*sy, integer angle reduction).
    Sy = Sx = 1024
    for s in (1023 * Sx + 1022, 7, 1024 * 1024 - 1, 511 * Sx + 513):
        imp = np.zeros((Sy, Sx))
        imp[s // Sx, s % Sx] = 1.0
        ref = np.fft.fft2(imp, norm="ortho").reshape(-1)
        f = O.scan_phase(np.arange(Sy * Sx), [s], Sy, Sx)[:, 0]
        assert np.max(np.abs(f - ref)) < 1e-15


def test_project_events_equals_dense_projection():
    # the sparse-event form of H equals the dense projection of the same frames
    from synth.sparse import dense_frames_numpy, sparse_events
    Q, L = 32, 8
    Psi = O.hg_basis(Q, L, math.sqrt(Q / (2 * math.pi)))
    pix, cnt = sparse_events(5, np.arange(40), Q, events=9)
    pix[0, 1] = pix[0, 0]                       # a duplicated pixel must add
    dense = dense_frames_numpy(pix, cnt, Q).astype(np.float64)
    assert np.max(np.abs(O.project_events(pix, cnt, Psi) - O.vec(O.project(dense, Psi)))) < 1e-10
