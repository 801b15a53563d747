"""CPU oracle for the B200 adaptive-GEMM library -- TEST INFRASTRUCTURE ONLY.

Restates the reference's algorithms (/root/reference/pkg/src/adaptgemm/) on
the CPU so the B200 product can be checked and timed against them:

* gemm_oracle.c / gemm.py -- the three numba GEMM loop nests (reference,
  direct, tiled+pack) in C with float64 accumulation in the reference's
  summation order, bit-identical to the reference (pinned by
  tests/golden/gemm_golden.npz, generated from the reference itself by
  tests/golden/make_golden.py);
* cart.py -- CART best_split/train/predict in plain Python (exact ints),
  pinned by the reference's trees in tests/golden/.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product package
`paper_1806_07060_b200` never imports, links or executes it; there is no
CPU fallback in the product path.
"""
