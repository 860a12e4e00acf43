"""NeuroShard fp64 CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct reference for what the
CUDA hot path computes.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product package ``paper_2305_01868_b200`` never imports, links or calls
anything here, and this package imports nothing from the product package; the
two share only the seeded random recipes in ``workload/``.

Layout (each function cites the PAPER.md passage it follows):

* ``model``  -- O1 featurise, O2 encoder, O3 head, O4 compute cost of a set,
                O5 comm models, O6 plan cost f(c, t)
* ``search`` -- O7 column split, O8 GreedyGridSearch (Alg. 2), O9 BeamSearch
                (Alg. 1), O10 literal life-long cache, O11 decision log,
                O12 work count
* ``brute``  -- exhaustive enumerators used only as pins in tests

Parity status: every function is pinned by a ``-m "not gpu"`` test
(tests/test_oracle_*.py); DESIGN.md §"Oracle pins" lists which pin covers
which function.  There is no "parity unpinned" function.
"""
from . import model, search, brute  # noqa: F401
