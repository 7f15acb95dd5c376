"""Seeded synthetic workloads (kernels + input heaps) shared by tests and bench.

Holds none of the method's arithmetic: it only encodes kernels (asm.py),
lists the paper-shaped kernels (kernels.py) and draws counter-based random
input arrays (inputs.py).  Neither oracle/ nor paper_1308_3203_b200/ imports
it; tests/ and bench.py feed both sides from it.
"""
