"""CPU oracle for the HAPOD hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import anything from this package, and only as the
checker (or as the timed CPU baseline).  The product package
``paper_1607_05210_b200`` never imports it and has no CPU fallback.
"""
