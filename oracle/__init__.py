"""TEST INFRASTRUCTURE ONLY -- the CPU oracle of the TNC hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and
only as the checker or the timed CPU baseline.  The product package
``paper_2504_09186_b200`` never imports it (enforced by
``tests/test_boundary.py``).
"""
