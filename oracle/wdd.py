"""Float64 oracle for the Live-WDD hot path.  TEST INFRASTRUCTURE ONLY (see __init__).

Every function cites the PAPER.md passage (P:line) it writes out.  Readings of the
paper where it is silent or garbled are numbered R1..R19 in DESIGN.md §3 and cited here.

Notation (paper): detector N x N (here Q x Q), L Hermite-Gauss orders per axis, K = L^2,
scan S = Sy x Sx positions s = sy*Sx + sx, scan frequencies v = vy*Sx + vx in FFT order.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "Geometry", "geometry", "hermite_functions", "hg_basis", "fourier_basis",
    "signed_freq", "probe_hat", "autocorrelation", "project", "vec",
    "accumulate_fft", "accumulate_stream", "active_set", "wiener_bank",
    "readout_spectrum", "image_from_spectrum", "reduced_wdd", "full_wdd",
    "pruning_bound_paper", "cdft2", "cidft2", "project_events", "scan_phase", "accumulate_at",
]


# ---------------------------------------------------------------------------------------
# Geometry (P:481-484 pixel conversion; R7, R8, R17)
# ---------------------------------------------------------------------------------------
class Geometry:
    """Derived acquisition quantities (all lengths in Angstrom, frequencies in 1/A).

    dq      detector pixel in reciprocal space: 1/(Q*step) unless det_px_rad given (R17)
    q_alpha aperture radius alpha/lambda (R7: alpha, not sin(alpha))
    R       aperture radius in detector pixels, q_alpha/dq ("radius of the circle in pixel R")
    c       basis / DC centre pixel Q/2 (R2)
    sigma   Hermite-Gauss width in pixels, sqrt(Q/(2*pi)) unless overridden (R1)
    """

    def __init__(self, Q, step_A, wavelength_A, alpha_rad, defocus_A=0.0,
                 det_px_rad=0.0, sigma_px=0.0):
        self.Q = int(Q)
        self.step_A = float(step_A)
        self.wavelength_A = float(wavelength_A)
        self.alpha_rad = float(alpha_rad)
        self.defocus_A = float(defocus_A)
        self.dq = det_px_rad / wavelength_A if det_px_rad > 0 else 1.0 / (Q * step_A)
        self.q_alpha = alpha_rad / wavelength_A
        self.R = self.q_alpha / self.dq
        self.c = Q // 2
        self.sigma = sigma_px if sigma_px > 0 else math.sqrt(Q / (2.0 * math.pi))

    def q_grid(self):
        """Detector coordinates q_m = (m - c)*dq, m = 0..Q-1 (DC at pixel c)."""
        return (np.arange(self.Q) - self.c) * self.dq


def geometry(cfg, **kw) -> Geometry:
    return Geometry(cfg.Q, cfg.step_A, cfg.wavelength_A, cfg.alpha_rad, cfg.defocus_A, **kw)


# ---------------------------------------------------------------------------------------
# Hermite-Gauss basis (P:168-174 eqn:HO-eigenfunction, P:195-214 eqn:CHO-eigenfunction,
# P:346-358 sampled matrix psi_x; R1-R3)
# ---------------------------------------------------------------------------------------
def hermite_functions(u, L):
    """L2-normalised Hermite functions psi_n(u) = H_n(u) e^{-u^2/2} / sqrt(2^n n! sqrt(pi)),
    n = 0..L-1 (P:168-174 with its "proper L2-normalization").  Evaluated with the
    three-term recurrence psi_n = sqrt(2/n) u psi_{n-1} - sqrt((n-1)/n) psi_{n-2}, which is
    the Hermite-polynomial recurrence H_n = 2u H_{n-1} - 2(n-1) H_{n-2} divided by the
    normalisation (no factorials, no overflow).  Returns shape u.shape + (L,)."""
    u = np.asarray(u, dtype=np.float64)
    out = np.empty(u.shape + (L,))
    out[..., 0] = math.pi ** -0.25 * np.exp(-0.5 * u * u)
    if L > 1:
        out[..., 1] = math.sqrt(2.0) * u * out[..., 0]
    for n in range(2, L):
        out[..., n] = math.sqrt(2.0 / n) * u * out[..., n - 1] - math.sqrt((n - 1.0) / n) * out[..., n - 2]
    return out


def hg_basis(Q, L, sigma, center=None):
    """Sampled basis matrix psi_x in R^{Q x L}: Psi[m, n] = psi_n((m - c)/sigma)/sqrt(sigma),
    the continuous-normalised functions of width sigma sampled at pixel centres (R3)."""
    c = Q // 2 if center is None else center
    u = (np.arange(Q) - c) / sigma
    return hermite_functions(u, L) / math.sqrt(sigma)


def fourier_basis(Q, L=None):
    """Complex DFT basis Psi_F[m, n] = Q^{-1/2} exp(+2 pi i (m-c)(n-c)/Q) restricted to the L
    columns with smallest |n - c| (all Q columns when L is None).  Used only by the
    DFT-basis-substitution pin (R-oracle with this basis == F-oracle) and the
    convergence-as-K-grows pin."""
    c = Q // 2
    m = np.arange(Q) - c
    F = np.exp(2j * math.pi * np.outer(m, m) / Q) / math.sqrt(Q)
    if L is None or L >= Q:
        return F
    cols = np.argsort(np.abs(m), kind="stable")[:L]
    return F[:, np.sort(cols)]


# ---------------------------------------------------------------------------------------
# Scan frequencies, probe, autocorrelation (R7, R8, R15)
# ---------------------------------------------------------------------------------------
def signed_freq(S):
    """Signed frequency index v~ of FFT-ordered index v (numpy.fft.fftfreq * S; R15)."""
    return np.rint(np.fft.fftfreq(S) * S).astype(np.int64)


def probe_hat(geom: Geometry, shift=(0.0, 0.0)):
    """Fourier-space probe p_hat(q + shift) on the detector grid (Algorithm 1 initialisation,
    P:445-447 "circular aperture ... generated from the radius"), with the north-star defocus
    phase (R7): p_hat(q) = 1[|q|^2 <= q_alpha^2] exp(-i pi lambda df |q|^2).  Indexed [my, mx]."""
    q = geom.q_grid()
    qy = q[:, None] + shift[0]
    qx = q[None, :] + shift[1]
    q2 = qy * qy + qx * qx
    inside = q2 <= geom.q_alpha * geom.q_alpha
    return np.where(inside, np.exp(-1j * math.pi * geom.wavelength_A * geom.defocus_A * q2), 0.0)


def scan_shift(v, Sy, Sx, step_A):
    """q_hat_v = (v~y/(Sy*step), v~x/(Sx*step)) in 1/A (P:481-484 per axis, R8)."""
    vy, vx = int(v) // Sx, int(v) % Sx
    fy, fx = signed_freq(Sy)[vy], signed_freq(Sx)[vx]
    return (fy / (Sy * step_A), fx / (Sx * step_A))


def autocorrelation(geom: Geometry, v, Sy, Sx):
    """Y_v[my, mx] = p_hat(q) * conj(p_hat(q + q_hat_v))  (Algorithm 1 line 3)."""
    qh = scan_shift(v, Sy, Sx, geom.step_A)
    return probe_hat(geom) * np.conj(probe_hat(geom, qh))


# ---------------------------------------------------------------------------------------
# Projection H and vectorisation (R5)
# ---------------------------------------------------------------------------------------
def project(A, Psi):
    """H(A) = psi_x^T A^T psi_y  in C^{L x L}, with psi_x = psi_y = Psi (R2).
    Works on a stack (..., Q, Q); entry [a, b] = sum_{my,mx} Psi[mx,a] Psi[my,b] A[my,mx]
    (a = n_x, b = n_y)."""
    A = np.asarray(A)
    return np.matmul(np.matmul(Psi.T, np.swapaxes(A, -1, -2)), Psi)


def vec(H):
    """vec: C^{L x L} -> C^{L^2}, k = a*L + b (row-major over [n_x][n_y], R5)."""
    H = np.asarray(H)
    return H.reshape(H.shape[:-2] + (H.shape[-1] * H.shape[-2],))


# ---------------------------------------------------------------------------------------
# Accumulation G(q_hat, k) (P:399-426 eq:outer_prod; Algorithm 2 lines 2-4)
# ---------------------------------------------------------------------------------------
def accumulate_fft(C, idx, Sy, Sx):
    """G = F_2D i over the ingested scan positions, F_2D = F (x) F unitary,
    computed as a unitary 2-D FFT of the zero-filled coefficient stack (P:416-420,
    I_hat = F_2D I).  Returns G[v, k], v = vy*Sx + vx (FFT order).  Duplicate indices add."""
    C = np.asarray(C)
    K = C.shape[-1]
    Z = np.zeros((Sy * Sx, K), dtype=np.result_type(C.dtype, np.float64))
    np.add.at(Z, np.asarray(idx), C)
    G = np.fft.fft2(Z.reshape(Sy, Sx, K), axes=(0, 1), norm="ortho")
    return G.reshape(Sy * Sx, K)


def accumulate_stream(C, idx, Sy, Sx):
    """G = sum_s f_s i_s^T  (eq:outer_prod): f_s is the s-th column of F_2D,
    f_s[v] = exp(-2 pi i (vy*sy/Sy + vx*sx/Sx)) / sqrt(Sy*Sx), summed one
    scan point at a time as Algorithm 2 does.  Slow; for pins only."""
    C = np.asarray(C)
    vy = np.arange(Sy)[:, None]
    vx = np.arange(Sx)[None, :]
    G = np.zeros((Sy * Sx, C.shape[-1]), dtype=np.complex128)
    for s, c in zip(np.asarray(idx), C):
        sy, sx = int(s) // Sx, int(s) % Sx
        f = np.exp(-2j * math.pi * (vy * sy / Sy + vx * sx / Sx)) / math.sqrt(Sy * Sx)
        G += np.outer(f.reshape(-1), c)
    return G


def project_events(pix, cnt, Psi):
    """H(I_s) of P:361 evaluated directly on a sparse frame given as events (pixel my*Q + mx,
    count): entry [a, b] = sum_events count * Psi[mx, a] * Psi[my, b] -- the same double sum
    as project(), restricted to the nonzero pixels.  Returns vec(H) per frame, shape (n, L*L)."""
    Q, L = Psi.shape
    pix = np.asarray(pix, dtype=np.int64)
    w = np.asarray(cnt, dtype=np.float64)
    my, mx = pix // Q, pix % Q
    H = np.einsum("ne,nea,neb->nab", w, Psi[mx], Psi[my], optimize=True)
    return vec(H)


def scan_phase(v_list, idx, Sy, Sx):
    """f_s[v] = exp(-2 pi i (vy*sy/Sy + vx*sx/Sx)) / sqrt(Sy*Sx) for the listed v
    (rows) and scan positions idx (columns).  The angle is reduced exactly in integers
    ((vy*sy) mod Sy, (vx*sx) mod Sx) before the float64 cos/sin."""
    v = np.asarray(v_list, dtype=np.int64)[:, None]
    s = np.asarray(idx, dtype=np.int64)[None, :]
    vy, vx, sy, sx = v // Sx, v % Sx, s // Sx, s % Sx
    ang = 2.0 * math.pi * (((vy * sy) % Sy) / Sy + ((vx * sx) % Sx) / Sx)
    return (np.cos(ang) - 1j * np.sin(ang)) / math.sqrt(Sy * Sx)


def accumulate_at(C, idx, v_list, Sy, Sx):
    """Rows v_list of G = sum_s f_s c_s^T (eq:outer_prod) for coefficient vectors C (n, K)
    at scan positions idx: G[v, :] = sum_s f_s[v] C[s, :]."""
    return scan_phase(v_list, idx, Sy, Sx) @ np.asarray(C, dtype=np.float64)


# ---------------------------------------------------------------------------------------
# Active set and Wiener bank (Algorithm 1 + intersection condition; R9, R10)
# ---------------------------------------------------------------------------------------
def active_set(geom: Geometry, Sy, Sx):
    """Sorted flattened v with Y_v not identically zero, i.e. the shifted apertures share at
    least one detector pixel (exact discrete form of s_y^2 + s_x^2 <= 4R^2; R9).
    Candidate prefilter |q_hat_v| <= 2 q_alpha is implied by the triangle inequality (a
    superset, not a heuristic); the pixel test is inclusive (<=) in float64 (R10)."""
    q = geom.q_grid()
    qa2 = geom.q_alpha * geom.q_alpha
    my, mx = np.nonzero(q[:, None] ** 2 + q[None, :] ** 2 <= qa2)
    uy, ux = q[my], q[mx]
    fy = signed_freq(Sy) / (Sy * geom.step_A)
    fx = signed_freq(Sx) / (Sx * geom.step_A)
    lim = 2.0 * geom.q_alpha * (1.0 + 1e-9)
    cand = [(vy, vx) for vy in range(Sy) if abs(fy[vy]) <= lim
            for vx in range(Sx) if fy[vy] ** 2 + fx[vx] ** 2 <= lim * lim]
    act = []
    for vy, vx in cand:
        a = uy + fy[vy]
        b = ux + fx[vx]
        if np.any(a * a + b * b <= qa2):
            act.append(vy * Sx + vx)
    return np.array(sorted(act), dtype=np.int64)


def wiener_bank(geom: Geometry, Psi, v_list, Sy, Sx, eps):
    """K_v = conj(H(Y_v)) / (|H(Y_v)|^2 + eps), elementwise (Algorithm 1 lines 4-5),
    vectorised (R5).  Returns W[len(v_list), K] complex128."""
    L = Psi.shape[1]
    W = np.empty((len(v_list), L * L), dtype=np.complex128)
    for i, v in enumerate(v_list):
        H = vec(project(autocorrelation(geom, v, Sy, Sx), Psi))
        W[i] = np.conj(H) / (np.abs(H) ** 2 + eps)
    return W


# ---------------------------------------------------------------------------------------
# Readout (Algorithm 2 lines 6-9 and final step; R12, R13, R14)
# ---------------------------------------------------------------------------------------
def readout_spectrum(G_act, W, active, Sy, Sx):
    """o_v = sum_k (mat(t_v) o K_v)_k  -- the deconvolution D_v = mat(t_v) o K_v and
    its zero-frequency extraction "summing all elements" (R12), for the active v;
    o_v = 0 elsewhere.  Returns the Sy x Sx spectrum in FFT order."""
    o = np.zeros(Sy * Sx, dtype=np.complex128)
    o[np.asarray(active)] = np.sum(np.asarray(G_act) * np.asarray(W), axis=-1)
    return o.reshape(Sy, Sx)


def image_from_spectrum(o, normalize=False):
    """O = conj(F^{-1}(o)) with the unitary inverse DFT (R13, R14); optionally divided
    by sqrt(o[0]) (principal branch), the eq:extract normalisation."""
    O = np.conj(np.fft.ifft2(o, norm="ortho"))
    if normalize:
        O = O / np.sqrt(complex(o.reshape(-1)[0]))
    return O


def reduced_wdd(frames, idx, geom: Geometry, Sy, Sx, L, eps, Psi=None, normalize=False,
                active=None, return_all=False):
    """R-oracle: Algorithm 2 end to end with the Wiener step deferred to readout (exact by
    linearity).  frames (n, Q, Q) real; idx the scan indices."""
    if Psi is None:
        Psi = hg_basis(geom.Q, L, geom.sigma)
    C = vec(project(np.asarray(frames, dtype=np.float64), Psi))
    G = accumulate_fft(C, idx, Sy, Sx)
    if active is None:
        active = active_set(geom, Sy, Sx)
    W = wiener_bank(geom, Psi, active, Sy, Sx, eps)
    o = readout_spectrum(G[active], W, active, Sy, Sx)
    O = image_from_spectrum(o, normalize)
    if return_all:
        return dict(C=C, G=G, active=active, W=W, o=o, O=O, Psi=Psi)
    return O


# ---------------------------------------------------------------------------------------
# F-oracle: conventional WDD (eq:deconv_mat P:90-95, eq:extract P:97-106, Fig:schematic_WDD)
# ---------------------------------------------------------------------------------------
def cdft2(x):
    """Centred unitary DFT over the last two axes (F_r with DC at pixel Q/2)."""
    return np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(x, axes=(-2, -1)), norm="ortho"), axes=(-2, -1))


def cidft2(x):
    """Centred unitary inverse DFT over the last two axes (F_q^{-1})."""
    return np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(x, axes=(-2, -1)), norm="ortho"), axes=(-2, -1))


def full_wdd(I4, geom: Geometry, eps, normalize=False, return_spectrum=False):
    """Full WDD on the 4-D data I4[sy, sx, my, mx]:
       (a) F_r^ (I): unitary DFT over the scan axes (Fig:schematic_WDD (a));
       (b) W_P^v = F_q^{-1}(Y_v) with Y_v = p_hat(q) conj(p_hat(q + q_hat_v));
       (c) W_O = F_q^{-1}(F_r^ I) conj(W_P) / (|W_P|^2 + eps)  (eq:deconv_mat);
       x_v = F_r(W_O)|_{q=0}, taken as the plain sum over r (R12 scale reading);
       O = conj(F_q^^{-1}(x)) (eq:extract numerator with Algorithm 2's conj, R13)."""
    Sy, Sx = I4.shape[:2]
    Gf = np.fft.fft2(np.asarray(I4, dtype=np.float64), axes=(0, 1), norm="ortho")
    x = np.zeros((Sy, Sx), dtype=np.complex128)
    for vy in range(Sy):
        for vx in range(Sx):
            Y = autocorrelation(geom, vy * Sx + vx, Sy, Sx)
            if not np.any(Y):
                continue
            WP = cidft2(Y)
            WO = cidft2(Gf[vy, vx]) * np.conj(WP) / (np.abs(WP) ** 2 + eps)
            x[vy, vx] = WO.sum()
    O = image_from_spectrum(x, normalize)
    return (O, x) if return_spectrum else O


# ---------------------------------------------------------------------------------------
# The paper's printed pruning bound (eq:low_correlation) -- documented, unused (R9)
# ---------------------------------------------------------------------------------------
def pruning_bound_paper(step_A, theta_rad, wavelength_A):
    """S_hat / S = sqrt(2) * Delta * sin(theta) / lambda  (eq:low_correlation).
    The paper's example theta = 32 mrad, Delta = 0.026 nm, lambda = 2.508 pm gives 0.47."""
    return math.sqrt(2.0) * step_A * math.sin(theta_rad) / wavelength_A
