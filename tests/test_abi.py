"""CPU-side checks of the C-ABI boundary: the library builds for sm_100a, loads, and exports
every symbol include/wdd.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "wdd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wdd_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = _declared()
    for n in ("wdd_plan_create", "wdd_ingest", "wdd_readout", "wdd_destroy"):
        assert n in names


def test_library_builds_loads_and_exports_every_declared_symbol():
    from paper_2212_01309_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_sass_contains_tcgen05_mma():
    import subprocess
    from paper_2212_01309_b200 import build
    out = subprocess.run(["cuobjdump", "-sass", build.build()], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out and "LDTM" in out


def test_error_path_without_gpu():
    # argument validation happens before any device call
    import paper_2212_01309_b200 as w
    import pytest
    with pytest.raises(w.WddError) as e:
        w.Plan((32, 32), 0.2, (32, 32), 63, 0.0197, 0.02)        # K not a square
    assert e.value.name == "WDD_E_ARG"
    with pytest.raises(w.WddError) as e:
        w.Plan((32, 32), 0.2, (48, 48), 64, 0.0197, 0.02)        # unsupported Q
    assert e.value.name == "WDD_E_ARG"
    with pytest.raises(w.WddError) as e:
        w.Plan((32, 32), 0.2, (32, 32), 64, 0.0197, 0.02, wiener_eps=0.0)
    assert e.value.name == "WDD_E_ARG"


def test_gpu_simulator_builds_and_exports():
    # the GPU forward simulator (test-input generator, synth/gpu.py) cross-compiles here
    import ctypes
    from synth import gpu as sim
    lib = ctypes.CDLL(sim.build())
    assert hasattr(lib, "sim_frames")
