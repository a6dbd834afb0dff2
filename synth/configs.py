"""The five BASELINE.json workloads as concrete, seeded acquisition parameters.

Values marked "proposed" in SURVEY.md §8(d) are the survey's readings of fields the
BASELINE.json config text leaves open (kV, seeds, atom counts for Live/Box, eps).
"""
from dataclasses import dataclass, replace
import math

# CODATA 2018 exact / recommended constants (SI)
_H = 6.62607015e-34
_M_E = 9.1093837015e-31
_Q_E = 1.602176634e-19
_C = 299792458.0


def wavelength_A(kv: float) -> float:
    """Relativistic electron wavelength in Angstrom for an accelerating voltage in kV.

    lambda = h / sqrt(2 m e V (1 + e V / (2 m c^2))).  300 kV -> 0.0196875 A;
    200 kV -> 0.02508 A (the paper's "lambda = 2.508 pm").
    """
    v = kv * 1e3
    p = math.sqrt(2.0 * _M_E * _Q_E * v * (1.0 + _Q_E * v / (2.0 * _M_E * _C * _C)))
    return _H / p * 1e10


@dataclass(frozen=True)
class Config:
    name: str
    Sy: int
    Sx: int
    step_A: float          # scan step Delta (Angstrom); also the probe-window pixel
    Q: int                 # detector is Q x Q pixels, DC at (Q/2, Q/2)
    dtype: str             # "f32" or "u16" frame storage
    kv: float
    alpha_rad: float       # probe semi-convergence angle
    defocus_A: float
    n_atoms: int
    amp_lo: float
    amp_hi: float
    dose: float            # expected electrons per frame
    L: int                 # Hermite-Gauss orders per axis, K = L*L
    eps: float             # Wiener epsilon
    batch: int             # frames per wdd_ingest call (0 = whole scan in one call)
    readout_rows: int      # live readout cadence in scan rows (0 = once at the end)
    seed: int
    atom_sigma_A: float = 0.3

    @property
    def S(self) -> int:
        return self.Sy * self.Sx

    @property
    def K(self) -> int:
        return self.L * self.L

    @property
    def wavelength_A(self) -> float:
        return wavelength_A(self.kv)

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


CONFIGS = {
    # BASELINE.json configs[0]: the case the CPU oracle finishes in seconds.
    "tiny": Config("tiny", 32, 32, 0.20, 32, "f32", 300.0, 20e-3, 0.0,
                   20, 0.1, 0.5, 1e4, 8, 1e-3, 1024, 0, 0),
    # configs[1]: the paper's (128,128,128,128) at L = 16; the bench workload.
    "medium": Config("medium", 128, 128, 0.15, 128, "u16", 300.0, 25e-3, 50.0,
                     400, 0.1, 0.5, 1e5, 16, 1e-3, 512, 0, 1),
    "large": Config("large", 256, 256, 0.15, 128, "u16", 300.0, 25e-3, 100.0,
                    1600, 0.2, 1.0, 1e5, 32, 1e-3, 0, 0, 2),
    "live": Config("live", 512, 512, 0.15, 256, "u16", 300.0, 25e-3, 100.0,
                   6400, 0.2, 1.0, 5e4, 32, 1e-3, 1024, 64, 3),
    "box": Config("box", 1024, 1024, 0.15, 256, "u16", 300.0, 25e-3, 100.0,
                  25600, 0.2, 1.0, 1e5, 24, 1e-3, 0, 0, 4),
}
