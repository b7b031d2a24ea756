"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the batched DC loadflow path.

Nothing in the product package imports this directory.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may use it, and only as the checker or as the timed CPU
baseline -- never as the thing measured or shipped.

Contents
--------
``port``    numpy restatement of the reference engine's solve path
            (`/root/reference/pkg/src/batchdc/solver.py`, `factors.py`):
            canonicalisation, materialised BSDF/MODF updates, LODF block,
            metric_first / symmetric injection stage, winner report.  Every
            function cites the reference file:line it follows.
``refact``  numpy restatement of the reference's refactorisation oracle
            (`pkg/src/batchdc/oracle.py:62-228`): explicit topology, fresh
            factorisation per contingency, union-find islanding.

Parity pin: both are checked against golden vectors produced by running the
reference itself in the build container (``tests/golden/make_golden.py``);
see ``tests/test_oracle_golden.py``.  The reference is pure Python/NumPy, so
there is no ``oracle/_ref`` build: the port is the CPU baseline
(``cpu_baseline.kind = "port"``).
"""
