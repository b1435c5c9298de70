"""CPU oracle for the in situ hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference) may import this package, and only as the checker or the timed CPU
baseline; the product (paper_2312_09888_b200) never does.
"""
