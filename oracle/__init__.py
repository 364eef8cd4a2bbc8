"""CPU ORACLE for the ParaDiag waveform-relaxation hot path of arXiv 2007.13125
(Wu & Zhou, "Parallel-in-time high-order BDF schemes ...").

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything under
`oracle/`.  The product path (`paper_2007_13125_b200/`) never imports it and shares
no code with it: no kernels, headers, helpers, tables or constant generators.
The only shared module is `paper_2007_13125_b200/inputs.py` (seeded problem data,
no method arithmetic).

Plain, slow, obviously-correct NumPy/SciPy/mpmath code in fp64 (tables in exact
rationals / mpmath / 80-bit long double, then rounded).  Each function cites the
PAPER.md lines (P:<line>) it follows.  Readings of garbled or ambiguous passages are
listed in DESIGN.md §"Readings of the paper" and in SURVEY.md §8(c).

Modules
  bdf        BDFk weights (exact), Table 1 corrections (exact), CQ weights, eigenvalues d_p
  spatial    FD Laplacian, DST-I, shifted spatial solves (DST eigen-solve / banded LU);
             space="fem": P1 finite elements, A = M^-1 K (1D mesh, 2D uniform triangulation;
             PAPER.md:1374-1376)
  problem    static right-hand side  f̄_n + tau^-a (sum_{j<n} w_j) v
  sequential O1: corrected sequential BDFk / CQ-BDFk stepping (the WR fixed point)
  wr         O2: Algorithm 1/2 literally (explicit wrap loops, naive DFT matrices)
  dense      O3: dense all-at-once Kronecker system (tiny sizes)
  modal      O4: per-sine-mode scalar WR (data in the span of few modes, e.g. C4)
  theory     exact per-mode WR contraction factor (pin for the paper's gamma(kappa))
  nonlinear  O5: semilinear scheme (Newton per step) and Algorithm 3 (Newton + WR inner solves)

Parity status of each function is recorded in DESIGN.md §"Oracle pins"; every
function listed above is pinned by a `-m "not gpu"` test in tests/test_oracle_*.py.
"""
