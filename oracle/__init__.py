"""CPU oracle for Algorithm 2 of arXiv 2502.07155 (Kircheis & Potts).

TEST INFRASTRUCTURE ONLY.  Plain, slow, float64 numpy, written from PAPER.md
section by section.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it.  The product path
(`paper_2502_07155_b200`) never imports, links or executes anything here, and
this package shares no code with it.
"""
from .bandlimited import *  # noqa: F401,F403
from . import nfft  # noqa: F401  (Algorithm 1 and the §5 comparison)
