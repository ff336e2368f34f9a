"""CPU oracle for the placement path and the workload kernels.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs as the checker or the timed
CPU baseline.  The product package never imports it.
"""
