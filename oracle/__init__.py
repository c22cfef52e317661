"""CPU oracle — TEST INFRASTRUCTURE, not product code.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package.  It shares no code with the CUDA
path in paper_1901_02330_b200/.  See oracle/solver.py for the per-function
paper citations and DESIGN.md for the readings it follows.
"""
