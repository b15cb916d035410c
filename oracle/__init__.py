"""ORACLE — test infrastructure only.

Plain, slow, obviously-correct CPU implementations of what the hot path
computes (float64 decode attention, the cost-model interpolation and Eq1-Eq6,
the paged allocator contract).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import, call, link or
execute anything under oracle/.  The product package never does, and it shares
no code with this directory.
"""
