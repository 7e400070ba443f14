"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference search path.

This package is the parity checker for the B200 implementation in
``paper_2506_08276_b200``. Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it, and
only as the checker or the timed CPU baseline — never as a product code path.

Every function cites the reference file:line it restates; the reference is
``slimvec`` 0.1.0 (pure Python/numpy), mounted read-only at
``/root/reference/pkg/src/slimvec``.

Pinning: the restatement is checked (``tests/test_oracle_golden.py``) against
golden vectors produced by the unmodified reference in the build container
(``tests/golden/make_golden.py``) — traversal traces, result lists, counters,
ADC tables and distances — and against the reference's own known-answer tests
(path-graph trace ``test_search.py:103-114``, distance KATs
``test_vectors.py:28-38``).
"""
