"""CPU oracle for the decoupled-MoE expert step (arXiv 2504.19925).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2504_19925_b200``) never imports it and
shares no code with it; both sides take inputs from ``synth/`` only.

Plain, slow, obviously correct NumPy (float64 for the planner, IEEE float32 per
op for the reduce and Adam, exactly as the paper's / DESIGN.md's op order).
Every function cites the passage it follows:

  plan.py      Alg. 1 (apx:algo_scheduler) + MINMAX reading A1
               + the static baseline (row f2, reading B2)
  dispatch.py  step 2 replica load-balancing + A8;
               capacity/drops and the policy drop study (row f2, B1/B3)
  reduce.py    intra+inter-rank all-reduce order and normalisation
               (sec:comm_allreduce) + A10, A11
  adam.py      optimizer step 5 + A15 op order
  numerics.py  bf16 round-to-nearest-even (A17)
  place.py     step 8 new-placement materialisation
  step.py      one iteration over G simulated ranks + the App. E byte count
               (apx:nonoffload)
  tokens.py    the token all-to-all along the routing (row f3; C1-C3)

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): SPEC worked examples, exact
apportionment characterisations, brute-force exhaustive search, stable argsort,
closed forms for Adam, torch.optim.Adam within 1e-6, torch's bf16 rounding,
the App. E closed-form volume, the step composition (A7), token round trips and the
adjoint identity, the policy drop ordering; a mutation sweep checks that
plausible one-line mistakes fail a pin.  No function here is "parity unpinned".
"""
