"""Seeded synthetic 4D-STEM inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NONE of the method's arithmetic (no Hermite-Gauss basis, no scan
DFT, no Wiener bank, no readout).  It only produces the diffraction frames the method
consumes, following the paper's forward model (`eq:forward`) and its
Poisson dose model.  See DESIGN.md "Input recipe".
"""
from .configs import CONFIGS, Config, wavelength_A  # noqa: F401
from .generator import Acquisition  # noqa: F401
