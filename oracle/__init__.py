"""TEST INFRASTRUCTURE ONLY -- the CPU parity oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.  The product
(``paper_1103_0066_b200``) never imports it.
"""
