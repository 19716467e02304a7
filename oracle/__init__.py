"""CPU oracle for the TT-GBF hot path -- TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference algorithm
(`ttpmf.filters.tt_fft_pmf_step`, Algorithm 3 of arXiv 2501.07942) used as
the *checker* for the CUDA product path.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline / `--impl reference`
legs may import it.  The product package `paper_2501_07942_b200` never
imports it and has no CPU fallback.

Pinning: every routine here is checked against golden vectors produced by
the real reference package (`tests/golden/make_golden.py`, run in the build
container where `/root/reference` exists) by `tests/test_oracle_golden.py`.

Modules
-------
* :mod:`oracle.ttcore`  -- TT primitives (round, Hadamard, sums, dots, point
  evaluation, interpolation, FFT convolution).
* :mod:`oracle.npgen`   -- restated numpy ``Generator`` draws (PCG64 +
  Lemire bounded ints + Floyd/tail-shuffle ``choice``), used to pin the
  device RNG.
* :mod:`oracle.cross`   -- greedy restricted cross with the reference's
  memoised evaluator semantics.
* :mod:`oracle.pmf`     -- grids, measurement models and the filter step.
"""
