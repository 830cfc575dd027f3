"""CPU oracle for the Flash hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker or as the
reported CPU baseline.  The product package never imports it.
"""
