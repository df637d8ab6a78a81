"""TEST INFRASTRUCTURE: parity checkers for the executor (see oracle/oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package; the product (paper_2111_12243_b200) never does.
"""
