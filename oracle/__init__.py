"""CPU oracle for one PRGD iteration (arXiv 2501.13385, Alg. 2) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path (the CUDA library
paper_2501_13385_b200/ and its C-ABI include/prgd.h) never imports, links or
executes anything here, and this package never imports the product.

Plain, slow, obviously-correct fp64 NumPy/LAPACK, following the paper's
definitions in the paper's order; see prgd.py for the per-function citations.
Parity pins (tests/test_oracle_*.py) tie it to brute-force materialisation,
closed forms and the paper's invariants.
"""
from .prgd import *  # noqa: F401,F403
