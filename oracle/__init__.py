"""ARKV CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, float64 (fp32-emulated where bit-exactness requires it) reference for
the ARKV decode hot path, written from PAPER.md (arXiv 2603.08727) and the readings
listed in DESIGN.md §3.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this package.
The product path (`paper_2603_08727_b200`) never imports it, and it never imports
the product path.
"""
from .arkv_oracle import *  # noqa: F401,F403
