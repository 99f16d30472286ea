"""CPU oracle for the SN-like DLR hot path -- TEST INFRASTRUCTURE ONLY.

This package is a numpy/scipy restatement of the reference ``greytrt``
algorithm (``/root/reference/pkg/src/greytrt``) for the path named in
``BASELINE.json:north_star``: the collocated transport sweep, source
iteration, the Galerkin projections of ``step_collocation`` and the per-cell
Newton linearisation / temperature update.  Every function cites the
reference file:line it restates.

Pinning: the restatement is checked against golden vectors produced by the
real reference (``tests/golden/make_golden.py`` imports ``greytrt`` from
``/root/reference/pkg/src`` and writes ``tests/golden/*.npz``); see
``tests/test_oracle_golden.py``.

Who may import this package: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` -- and only as
the checker or the timed CPU baseline.  The product package
``paper_2601_18705_b200`` never imports it and has no CPU fallback.
"""

from . import port  # noqa: F401
