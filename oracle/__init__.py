"""CPU oracle of the HAS data plane -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package, and only as the checker / CPU
baseline.  The product package never imports it.
"""
