"""TEST INFRASTRUCTURE ONLY -- never imported by the product path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker.
"""
