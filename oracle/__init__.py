"""ORACLE — test infrastructure only.

A plain, slow, fp64 CPU implementation of the bilateral-space solve of the Fast
Bilateral Solver (Barron & Poole, arXiv 1511.03296), written from PAPER.md.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product path
(``paper_1511_03296_b200``) never imports, links or executes anything here, and
this package shares no code with it.
"""
from .fbs_oracle import *  # noqa: F401,F403
