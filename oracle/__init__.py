"""CPU oracle for the unbalanced domain-decomposition solve path.

TEST INFRASTRUCTURE ONLY.  This package is a numpy restatement of the
reference algorithm (arxiv 2410.08859 reference package ``domdec``; every
function cites the reference file:line it restates).  It exists to check the
CUDA library and to serve as the timed CPU baseline in ``bench.py``
(``cpu_baseline`` / ``--impl reference``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` may import it, and only as the
checker / baseline: the product package ``paper_2410_08859_b200`` never
imports it and fails loudly when its CUDA library is missing.

Parity pinning: the restatement is checked against golden vectors generated
by running the reference itself (``scripts/make_golden.py`` -> ``tests/golden``),
see ``tests/test_oracle_golden.py``.

Layout: problems are embedded as 2D grids (1D grids become shape (1, n));
boxes are (off0, ext0, off1, ext1).
"""
