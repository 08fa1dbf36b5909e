"""CPU oracle for AD-PSGD (arXiv 1710.06952).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package.  The product path never does.
"""
