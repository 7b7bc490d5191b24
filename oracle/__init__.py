"""CPU oracle for the DG Euler residual path -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference (`/root/reference/pkg/src/hodg`, the numba
solver of arXiv 2209.01877) used as the checker for the CUDA product:
C kernels (hodg_oracle.c, rcm_oracle.c) plus numpy setup.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import it; the product package never does.

Parity pinning: in 2D it regenerates the reference's golden files
fixtures/residuals_dp.csv and residuals_mp.csv byte for byte and the RCM
spy fixtures exactly (tests/test_oracle_golden.py).  The 3D tetrahedral
path has no reference counterpart; it is the same code with the z terms,
checked by the reference's property tests restated in 3D.
"""
