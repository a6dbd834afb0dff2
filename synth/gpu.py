"""GPU forward simulator: the recipe of synth/generator.py with the per-frame
patch, DFT, intensity and Poisson steps on the device (synth/csrc/forward.cu, cuFFT for the DFT,
Philox4x32-10 counter-based Poisson).  The object and probe come from the host generator, so the
noise-free intensities match `Acquisition.frames(noise=False)`; the Poisson draws follow the same
distribution from a different random stream.  Test-input infrastructure only: it shares no code
with the library (paper_2212_01309_b200) or the oracle.

    sim = GpuAcquisition(cfg)            # builds synth/_lib/libwddsim.so on first use
    frames = sim.frames(idx)             # torch tensor on cuda, (n, Q, Q), cfg.dtype
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .generator import Acquisition

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "forward.cu")
_LIB = os.path.join(_HERE, "_lib", "libwddsim.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile libwddsim.so in-tree for sm_100a (nvcc, cuFFT)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        os.makedirs(os.path.dirname(_LIB), exist_ok=True)
        cmd = [os.environ.get("NVCC", "nvcc"), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
               "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-o", _LIB + f".{os.getpid()}.tmp", _SRC, "-lcufft"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc failed building libwddsim.so:\n" + res.stderr)
        os.replace(_LIB + f".{os.getpid()}.tmp", _LIB)     # (per-process temp: ranks may build at once)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.sim_frames.restype = ctypes.c_int
        _lib.sim_frames.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_int64), ctypes.c_int64, ctypes.c_double,
                                    ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    return _lib


class GpuAcquisition:
    """Frames of one seeded acquisition generated on the GPU (see module docstring)."""

    def __init__(self, cfg, device: str = "cuda"):
        import torch
        self.cfg = cfg
        host = Acquisition(cfg)
        self.obj = torch.from_numpy(host.object().astype(np.complex64)).to(device)
        self.probe = torch.from_numpy(np.ascontiguousarray(host.probe()).astype(np.complex64)).to(device)
        self.device = device

    def frames(self, idx, noise: bool = True):
        """(n, Q, Q) frames for scan indices idx: uint16 / float32 counts (cfg.dtype), or float64
        noise-free intensities scaled to the dose when noise=False."""
        import torch
        c = self.cfg
        idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64).reshape(-1))
        if noise:
            dt = torch.uint16 if c.dtype == "u16" else torch.float32
        else:
            dt = torch.float64
        out = torch.empty((len(idx), c.Q, c.Q), dtype=dt, device=self.device)
        if len(idx) == 0:
            return out
        rc = _load().sim_frames(self.obj.data_ptr(), self.probe.data_ptr(), c.Sy, c.Sx, c.Q,
                                idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), len(idx), float(c.dose),
                                int(c.seed) & 0xFFFFFFFF, 0 if c.dtype == "u16" else 1, 1 if noise else 0,
                                out.data_ptr())
        if rc == -2:
            raise OverflowError("a count overflowed uint16")
        if rc != 0:
            raise RuntimeError(f"sim_frames failed ({rc})")
        return out
