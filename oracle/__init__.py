"""CPU oracle of the reference hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu-baseline leg may
import this package.  The product package never does.
"""
