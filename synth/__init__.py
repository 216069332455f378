"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the paper's method (no planning, no
dispatch ranks, no reduction, no Adam, no bf16 rounding).  It only produces
inputs:

* ``configs``  -- the BASELINE.json workloads as concrete shapes (SURVEY.md §8(d).1,
  readings A13/A14 in DESIGN.md).
* ``traces``   -- routing traces (top-k expert ids + gate payloads) shaped like the
  paper's popularity dynamics ("16x swing within 3 iterations").
* ``hashgen``  -- a counter-based generator (splitmix64) for synthetic slot gradients
  and initial master weights.  The CUDA side implements the same counter hash
  independently (``csrc/synth.cu``); values are produced by direct bit
  construction, so no floating-point rounding is involved on either side.
"""
