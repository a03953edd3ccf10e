"""CPU oracle for the Leja / FD-JVP / MHD-RHS hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in NumPy, the algorithm of the reference implementation
(arxiv/paper_2108_13622, Python package ``xmhd`` under ``pkg/src/xmhd``) for the
path named in BASELINE.json ``north_star``.  Every function cites the reference
file:line it follows.  The restatement reproduces the reference's exact IEEE
operation sequence (NumPy ufuncs evaluate one operation at a time: no FMA
contraction, true division, Python's left-to-right association), so it is
bitwise equal to the reference on the same inputs.

Pinning: ``tests/test_oracle_golden.py`` checks this oracle against golden
vectors produced by running the reference itself (``tests/golden/make_golden.py``
imports ``xmhd`` from ``/root/reference/pkg/src`` in the build container and
stores the outputs under ``tests/golden/``).  Parity is therefore PINNED.

Usage rule: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker or the timed CPU baseline.  The product package
``paper_2108_13622_b200`` never imports it.
"""
