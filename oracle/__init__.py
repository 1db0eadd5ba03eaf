"""TEST INFRASTRUCTURE ONLY — the float64 CPU oracle for the otk hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import, call, link or execute anything under ``oracle/``. The product package
(``paper_2601_07376_b200``) never imports it, and the oracle never imports the product package:
the two share no code (only the seeded generators in ``synth/`` feed both).
"""
