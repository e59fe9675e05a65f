"""CPU oracle for the conv hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker or the CPU
baseline being timed — never as part of the product path (which has no CPU
fallback).  See oracle/conv_ref.py for the restated algorithm and its
reference citations, and tests/golden/ for the fixtures that pin it.
"""
