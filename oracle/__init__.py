"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for arXiv 2202.08361's hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2202_08361_b200``) never imports it and shares no code with it.

``oracle/jsvd_oracle.c`` is the oracle proper (plain C, libm, explicit fma,
``-ffp-contract=off``); this module only marshals numpy arrays into it.
"""
from .oracle import *  # noqa: F401,F403
