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

Pins (tests/test_oracle_*.py) tie every function to something other than itself; no
function is unpinned.  `reduced_wdd` is basis-agnostic code (Psi is an argument): with the
DFT basis it equals the F-oracle to 3e-16 (an end-to-end pin of projection, accumulation,
bank, readout and image), and the HG basis it uses by default is pinned on its own (Gram,
parity, DFT eigen-property, Hermite recurrence).  What has no closed form is the numerical
VALUE of an HG-basis reconstruction (Eq. hermite_conv is not an identity); it is checked by
phase recovery of a known object and by convergence to full WDD -- see DESIGN.md §2.
"""
from .wdd import *  # noqa: F401,F403
