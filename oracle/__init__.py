"""oracle -- plain, slow, obviously-correct fp64 CPU implementation of the AFN
hot path (arXiv 2304.05460), written from PAPER.md.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.  The
product path (``paper_2304_05460_b200``) never imports, calls or links it, and
it shares no code, headers, tables or constants with the CUDA path.

Every function cites the PAPER.md passage it follows (``P:L<line>``).  Where the
paper is silent the reading taken is listed in DESIGN.md "Readings" and in
SURVEY.md 8(c) (``R<n>`` below refers to that list).

Pinned by ``tests/test_oracle_*.py`` (run with ``-m "not gpu"``).  Parity
status of each function is recorded in DESIGN.md; ``alg1``'s refined branch is
pinned by closed forms (separated clusters, two points) but not by the paper's
printed values (they need m > 500, R13).
"""
from .afn_oracle import *  # noqa: F401,F403
