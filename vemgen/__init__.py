"""Seeded input generator: the host-side mixed-VEM assembler.

BASELINE.json north_star names a "host-side CPU assembler that builds M, B and
the right-hand sides from a seeded mesh, k and K, and also serves as input
generator".  Both the oracle and the CUDA path consume its output (CSR M, B, the
RHS and the DOF layout); it holds none of the solver arithmetic of the hot path
(SpMV, preconditioners, GMRES).  Its correctness is pinned independently by
tests/test_vemgen.py.
"""
