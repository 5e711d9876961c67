"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package, and only as the checker or the timed CPU
baseline.  paper_2310_18813_b200 (the product) never imports it.
"""
