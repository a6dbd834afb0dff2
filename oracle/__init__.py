"""Float64 CPU oracle for Live WDD (arXiv 2212.01309) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import anything from this package.  The product path (paper_2212_01309_b200/ and
its CUDA library) never imports, links or executes it, and shares no code, table or
constant generator with it.

Contents (see oracle/wdd.py for per-function citations of PAPER.md):
  * R-oracle: Algorithm 2 (`Algo:ModifiedWDD`) step by step, Wiener step
    deferred to readout (exact by linearity), with the Hermite-Gauss basis of
    P:168-174 / P:348-364 and the Wiener bank of `Algo:PreCompute`.
  * F-oracle: conventional full WDD, `eq:deconv_mat` + `eq:extract`
     as drawn in `Fig:schematic_WDD`.

Pins (tests/test_oracle_*.py) tie every function to something other than itself.
"Parity unpinned": the reduced (HG-basis) reconstruction as a whole has no closed form;
it is pinned piecewise (basis, projection, accumulation, bank, DFT-basis substitution
identity with the F-oracle, phase recovery) -- see DESIGN.md §3.
"""
from .wdd import *  # noqa: F401,F403
