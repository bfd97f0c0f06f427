"""CPU oracle for the recycled hypergradient solve -- TEST INFRASTRUCTURE ONLY.

This package is the *checker*, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The product package
``paper_2412_08264_b200`` never imports it and has no CPU fallback.

What it restates (numpy/scipy, fp64), each function citing the reference
``/root/reference/pkg/src/krecycle/<file>:<line>`` it follows:

* ``cpu_imaging``  -- operators: the reference FoE-inpainting operator
  (operators.py) and the BASELINE configs' deblurring operators
  (Gaussian blur + smoothed TV / learned filters with phi_eps), both
  behind the reference's SymmetricOperator / MixedJacobianOperator
  protocol; the seeded problem generators (experiments.py:139-177 pattern).
* ``cpu_krylov``   -- MINRES / RMINRES (Alg. 3) / CG with the reference's
  flop model and stop semantics (krylov.py).
* ``cpu_recycle``  -- candidate basis, Ritz / harmonic Ritz / RGen (GSVD)
  selection, prepare_recycle, next_recycle (recycling.py) and the stop
  rules (stopping.py).
* ``cpu_bilevel``  -- L-BFGS lower solve, Armijo upper linesearch, gradient
  descent, SequenceSolver, hypergradient, record/replay (bilevel.py,
  experiments.py), generalised to a batch of samples.

Parity pin: the oracle is checked against (1) the reference's golden CSVs
``pkg/plots/sample_data/{replay,sweep}.csv`` (integer columns exact, floats
<= 1e-9 relative) and (2) fixtures produced by importing the reference in
the build container (``tests/golden/make_golden.py``).  The deblurring /
TV / phi_eps operators do not exist in the reference: their contract tests
(adjointness, symmetry, finite differences, dense materialisation) carry
over, their values are "parity unpinned" against the reference.
"""
