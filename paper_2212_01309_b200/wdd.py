"""Thin ctypes binding over libwdd.so (include/wdd.h).  Argument marshalling only: every step
of the hot path runs in the library's sm_100a kernels.  PyTorch supplies device memory and
streams.  There is no fallback: if the shared library is missing or a call fails, this module
raises."""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WDD_LIB") or os.path.join(_HERE, "_lib", "libwdd.so")

STATUS = {0: "WDD_OK", 1: "WDD_E_ARG", 2: "WDD_E_RANGE", 3: "WDD_E_DUP", 4: "WDD_E_NOMEM",
          5: "WDD_E_CUDA", 6: "WDD_E_NCCL", 7: "WDD_E_STATE"}
SLOTS = {"project": 0, "rowdft": 1, "flush": 2, "readout": 3, "finalize": 4}


class WddError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class _Probe(ctypes.Structure):
    _fields_ = [("wavelength_A", ctypes.c_double), ("semiangle_rad", ctypes.c_double),
                ("defocus_A", ctypes.c_double)]


class _Opts(ctypes.Structure):
    _fields_ = [("det_px_rad", ctypes.c_double), ("sigma_px", ctypes.c_double),
                ("dtype", ctypes.c_int32), ("normalize", ctypes.c_int32), ("device", ctypes.c_int32),
                ("combine", ctypes.c_int32), ("accumulator", ctypes.c_int32), ("ingest_overlap", ctypes.c_int32),
                ("k_shards", ctypes.c_int32), ("k_rank", ctypes.c_int32), ("ingest_spread", ctypes.c_int32),
                ("readout_async", ctypes.c_int32), ("reserved", ctypes.c_int32 * 1)]


class _Info(ctypes.Structure):
    _fields_ = [("Sy", ctypes.c_int32), ("Sx", ctypes.c_int32), ("Q", ctypes.c_int32), ("L", ctypes.c_int32),
                ("K", ctypes.c_int32), ("n_vx", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("normalize", ctypes.c_int32), ("n_act", ctypes.c_int64), ("dq", ctypes.c_double),
                ("q_alpha", ctypes.c_double), ("R_px", ctypes.c_double), ("sigma_px", ctypes.c_double),
                ("wavelength_A", ctypes.c_double), ("step_A", ctypes.c_double), ("eps", ctypes.c_double),
                ("bytes_G", ctypes.c_int64), ("bytes_bank", ctypes.c_int64), ("bytes_R", ctypes.c_int64),
                ("bytes_C", ctypes.c_int64), ("frames_ingested", ctypes.c_int64), ("nranks", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("proj_ctas_per_sm", ctypes.c_int32), ("k_shards", ctypes.c_int32),
                ("k_rank", ctypes.c_int32), ("k_lo", ctypes.c_int32), ("k_count", ctypes.c_int32),
                ("n_vh", ctypes.c_int32)]


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libwdd.so (raises OSError if it has not been built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise OSError(f"{path} not found: build it with `python -m paper_2212_01309_b200.build`")
        lib = ctypes.CDLL(path)
        P, V, I64, I32 = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        sigs = {
            "wdd_plan_create": [ctypes.POINTER(I32), ctypes.c_double, ctypes.POINTER(I32), I32,
                                ctypes.POINTER(_Probe), ctypes.c_double, ctypes.POINTER(_Opts), ctypes.POINTER(P)],
            "wdd_ingest": [P, V, ctypes.POINTER(I32), I64, V],
            "wdd_ingest_host": [P, V, ctypes.POINTER(I32), I64, V],
            "wdd_readout": [P, V],
            "wdd_readout_host": [P, V],
            "wdd_readout_spectrum": [P, V, I32],
            "wdd_readout_wait": [P, V],
            "wdd_image_from_spectrum": [P, V, V],
            "wdd_check": [P],
            "wdd_ingest_remote": [P, ctypes.POINTER(I32), I64],
            "wdd_shard_store_handle": [P, ctypes.c_char_p],
            "wdd_set_shard_peers": [P, I32, I32, ctypes.c_char_p],
            "wdd_link_shards": [I32, ctypes.POINTER(P)],
            "wdd_destroy": [P],
            "wdd_get_accumulator": [P, V, ctypes.POINTER(I32), ctypes.POINTER(I64)],
            "wdd_full_wdd": [P, V, V, V],
            "wdd_reset": [P],
            "wdd_nccl_get_unique_id": [ctypes.c_char_p],
            "wdd_set_comm": [P, I32, I32, ctypes.c_char_p],
            "wdd_get_info": [P, ctypes.POINTER(_Info)],
            "wdd_get_tables": [P, V, V, ctypes.POINTER(I32)],
            "wdd_project": [P, V, I64, V, V],
            "wdd_profile_enable": [P, I32],
            "wdd_profile_read": [P, I32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64)],
            "wdd_launch_count": [P, ctypes.POINTER(I64), I32],
            "wdd_sync": [P],
            "wdd_capture_begin": [P, V],
            "wdd_capture_end": [P, ctypes.POINTER(I64)],
            "wdd_graph_launch": [P, I64, V],
        }
        for name, args in sigs.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        lib.wdd_last_error.argtypes = []
        lib.wdd_last_error.restype = ctypes.c_char_p
        _lib = lib
    return _lib


def _check(status: int):
    if status != 0:
        raise WddError(status, load_library().wdd_last_error().decode())


def _ptr(x) -> int:
    if x is None:
        return 0
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    if hasattr(x, "__cuda_array_interface__"):
        return x.__cuda_array_interface__["data"][0]
    return int(x)


def _stream(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _idx(scan_idx) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(scan_idx, dtype=np.int32).reshape(-1))
    return a


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().wdd_nccl_get_unique_id(buf))
    return buf.raw


def link_shards(plans):
    """Link the coefficient stores of plans[r] = shard r of len(plans) in this process
    (wdd_link_shards): each plan's projection then writes the other shards' coefficients directly."""
    arr = (ctypes.c_void_p * len(plans))(*[p._h.value for p in plans])
    _check(load_library().wdd_link_shards(len(plans), arr))


class Plan:
    """A Live-WDD plan (wdd_plan_create ... wdd_destroy)."""

    def __init__(self, scan_shape, step_A: float, det_shape, K: int, wavelength_A: float,
                 semiangle_rad: float, defocus_A: float = 0.0, wiener_eps: float = 1e-3, *,
                 dtype: str = "u16", normalize: bool = False, device: int = 0, sigma_px: float = 0.0,
                 det_px_rad: float = 0.0, combine: int = 0, accumulator: str = "G",
                 ingest_overlap: bool = False, k_shards: int = 0, k_rank: int = 0, ingest_spread: bool = False,
                 readout_async: bool = False):
        lib = load_library()
        scan = (ctypes.c_int32 * 2)(*[int(v) for v in scan_shape])
        det = (ctypes.c_int32 * 2)(*[int(v) for v in det_shape])
        probe = _Probe(float(wavelength_A), float(semiangle_rad), float(defocus_A))
        opts = _Opts()
        opts.det_px_rad = float(det_px_rad)
        opts.sigma_px = float(sigma_px)
        opts.dtype = {"u16": 0, "f32": 1}[dtype]
        opts.normalize = int(bool(normalize))
        opts.device = int(device)
        opts.combine = int(combine)
        opts.accumulator = {"G": 0, "spectrum": 1}[accumulator]
        opts.ingest_overlap = int(bool(ingest_overlap))
        opts.k_shards = int(k_shards)
        opts.k_rank = int(k_rank)
        opts.ingest_spread = int(bool(ingest_spread))
        opts.readout_async = int(bool(readout_async))
        h = ctypes.c_void_p()
        _check(lib.wdd_plan_create(scan, float(step_A), det, int(K), ctypes.byref(probe), float(wiener_eps),
                                   ctypes.byref(opts), ctypes.byref(h)))
        self._h = h
        self._lib = lib
        self.dtype = dtype
        self.readout_async = bool(readout_async)
        self.device = int(device)
        i = self.info()
        self.Sy, self.Sx, self.Q, self.L, self.K, self.n_act = i["Sy"], i["Sx"], i["Q"], i["L"], i["K"], i["n_act"]
        self.k_lo, self.k_count = i["k_lo"], i["k_count"]

    @classmethod
    def from_config(cls, cfg, **kw):
        """Build from any object with the synth.Config attribute names (duck-typed)."""
        return cls((cfg.Sy, cfg.Sx), cfg.step_A, (cfg.Q, cfg.Q), cfg.K, cfg.wavelength_A, cfg.alpha_rad,
                   cfg.defocus_A, cfg.eps, dtype=cfg.dtype, **kw)

    # ---- lifetime
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _check(self._lib.wdd_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- hot path
    def _check_frames(self, frames, n: int, device: bool):
        """Shape / dtype / contiguity of a frame batch against the plan (the C ABI takes a bare
        pointer and trusts n)."""
        shape = tuple(frames.shape)
        if shape != (n, self.Q, self.Q):
            raise ValueError(f"frames shape {shape} != ({n}, {self.Q}, {self.Q}) for {n} scan indices")
        want = "uint16" if self.dtype == "u16" else "float32"
        if want not in str(frames.dtype):
            raise ValueError(f"frames dtype {frames.dtype}, plan expects {want}")
        if hasattr(frames, "is_contiguous"):
            if not frames.is_contiguous():
                raise ValueError("frames must be contiguous")
            if device != frames.is_cuda:
                raise ValueError("frames must be on the " + ("device" if device else "host"))
        elif isinstance(frames, np.ndarray) and not frames.flags["C_CONTIGUOUS"]:
            raise ValueError("frames must be contiguous")

    def ingest(self, frames, scan_idx, stream=None):
        idx = _idx(scan_idx)
        self._check_frames(frames, len(idx), True)
        _check(self._lib.wdd_ingest(self._h, _ptr(frames), idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                    len(idx), _stream(stream)))

    def ingest_host(self, frames, scan_idx, stream=None):
        idx = _idx(scan_idx)
        self._check_frames(frames, len(idx), False)
        _check(self._lib.wdd_ingest_host(self._h, _ptr(frames), idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                         len(idx), _stream(stream)))

    def readout(self, out=None, wait: bool = True):
        """The image (Sy x Sx complex64).  readout_async plans: wait=True orders torch's current
        stream after the readout; wait=False leaves that to a later readout_wait (pipelining)."""
        import torch
        if out is None:
            out = torch.empty((self.Sy, self.Sx), dtype=torch.complex64, device=f"cuda:{self.device}")
        self._check_out(out)
        _check(self._lib.wdd_readout(self._h, _ptr(out)))
        self._maybe_wait(wait)
        return out

    def readout_wait(self, stream=None):
        """Order `stream` (default: torch's current stream) after the latest readout-family call."""
        _check(self._lib.wdd_readout_wait(self._h, _stream(stream)))

    def _maybe_wait(self, wait: bool):
        if wait and self.readout_async and not getattr(self, "_capturing", False):
            self.readout_wait()

    def readout_spectrum(self, out=None, combine: bool = True, wait: bool = True):
        """o_v (Sy x Sx complex64, FFT order, 0 at inactive v): combined over ranks, or this rank's own."""
        import torch
        if out is None:
            out = torch.empty((self.Sy, self.Sx), dtype=torch.complex64, device=f"cuda:{self.device}")
        self._check_out(out)
        _check(self._lib.wdd_readout_spectrum(self._h, _ptr(out), int(bool(combine))))
        self._maybe_wait(wait)
        return out

    def image_from_spectrum(self, spectrum, out=None, wait: bool = True):
        import torch
        self._check_out(spectrum)
        if out is None:
            out = torch.empty((self.Sy, self.Sx), dtype=torch.complex64, device=f"cuda:{self.device}")
        self._check_out(out)
        _check(self._lib.wdd_image_from_spectrum(self._h, _ptr(spectrum), _ptr(out)))
        self._maybe_wait(wait)
        return out

    def check(self):
        """Synchronise and raise WddError(WDD_E_RANGE) if out-of-range float32 frames were ingested."""
        _check(self._lib.wdd_check(self._h))

    def _check_out(self, t):
        if tuple(t.shape) != (self.Sy, self.Sx) or "complex64" not in str(t.dtype) or not t.is_cuda \
                or not t.is_contiguous():
            raise ValueError(f"expected a contiguous ({self.Sy}, {self.Sx}) complex64 device tensor")

    def readout_host(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty((self.Sy, self.Sx), dtype=np.complex64)
        _check(self._lib.wdd_readout_host(self._h, out.ctypes.data))
        return out

    def get_accumulator(self):
        """(G, active v): G is n_act x K complex64 (shard plans: n_act x k_count, coefficients
        k_lo .. k_lo + k_count - 1)."""
        import torch
        G = torch.empty((self.n_act, self.k_count), dtype=torch.complex64, device=f"cuda:{self.device}")
        act = np.empty(self.n_act, dtype=np.int32)
        n = ctypes.c_int64()
        _check(self._lib.wdd_get_accumulator(self._h, _ptr(G), act.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                             ctypes.byref(n)))
        self._maybe_wait(True)
        return G, act

    def active_set(self) -> np.ndarray:
        act = np.empty(self.n_act, dtype=np.int32)
        n = ctypes.c_int64()
        _check(self._lib.wdd_get_accumulator(self._h, None, act.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                             ctypes.byref(n)))
        return act

    def reset(self):
        _check(self._lib.wdd_reset(self._h))

    def set_comm(self, nranks: int, rank: int, uid: bytes):
        _check(self._lib.wdd_set_comm(self._h, int(nranks), int(rank), uid))

    # ---- coefficient-sharded rank groups
    def ingest_remote(self, scan_idx):
        """Positions another rank of the shard group ingests (host bookkeeping only)."""
        idx = _idx(scan_idx)
        _check(self._lib.wdd_ingest_remote(self._h, idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(idx)))

    def shard_store_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _check(self._lib.wdd_shard_store_handle(self._h, buf))
        return buf.raw

    def set_shard_peers(self, nshard: int, rank: int, handles):
        blob = b"".join(bytes(h) if h is not None else bytes(64) for h in handles)
        if len(blob) != 64 * nshard:
            raise ValueError("need one 64-byte handle per shard")
        _check(self._lib.wdd_set_shard_peers(self._h, int(nshard), int(rank), blob))

    # ---- introspection / test hooks
    def info(self) -> dict:
        i = _Info()
        _check(self._lib.wdd_get_info(self._h, ctypes.byref(i)))
        return {k: getattr(i, k) for k, _ in _Info._fields_}

    def tables(self, bank: bool = False):
        basis = np.empty((self.Q, self.L), dtype=np.float64)
        W = np.empty((self.n_act, self.K), dtype=np.complex128) if bank else None
        act = np.empty(self.n_act, dtype=np.int32)
        _check(self._lib.wdd_get_tables(self._h, basis.ctypes.data, None if W is None else W.ctypes.data,
                                        act.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
        return basis, W, act

    def full_wdd(self, frames, out=None, stream=None):
        """Conventional (full) WDD of a whole scan (frames: (S, Q, Q) device tensor in scan order)."""
        import torch
        self._check_frames(frames, self.Sy * self.Sx, True)
        if out is None:
            out = torch.empty((self.Sy, self.Sx), dtype=torch.complex64, device=frames.device)
        _check(self._lib.wdd_full_wdd(self._h, _ptr(frames), _ptr(out), _stream(stream)))
        return out

    def project(self, frames, out=None, stream=None):
        import torch
        n = frames.shape[0]
        self._check_frames(frames, n, True)
        if out is None:
            out = torch.empty((n, self.K), dtype=torch.float32, device=frames.device)
        if tuple(out.shape) != (n, self.K) or out.dtype != torch.float32 or not out.is_cuda or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous ({n}, {self.K}) float32 device tensor")
        _check(self._lib.wdd_project(self._h, _ptr(frames), n, _ptr(out), _stream(stream)))
        return out

    def profile_enable(self, on: bool = True):
        _check(self._lib.wdd_profile_enable(self._h, int(on)))

    def profile_read(self, slot) -> tuple:
        ms = ctypes.c_double()
        cnt = ctypes.c_int64()
        _check(self._lib.wdd_profile_read(self._h, SLOTS.get(slot, slot), ctypes.byref(ms), ctypes.byref(cnt)))
        return ms.value, cnt.value

    def launch_count(self, reset: bool = False) -> int:
        c = ctypes.c_int64()
        _check(self._lib.wdd_launch_count(self._h, ctypes.byref(c), int(reset)))
        return c.value

    # ---- CUDA graphs (capture a fixed sequence, replay its device work)
    def capture_begin(self, stream=None):
        _check(self._lib.wdd_capture_begin(self._h, _stream(stream)))
        self._capturing = True

    def capture_end(self) -> int:
        h = ctypes.c_int64()
        self._capturing = False
        _check(self._lib.wdd_capture_end(self._h, ctypes.byref(h)))
        return h.value

    def graph_launch(self, handle: int, stream=None):
        _check(self._lib.wdd_graph_launch(self._h, int(handle), _stream(stream)))

    def sync(self):
        _check(self._lib.wdd_sync(self._h))
