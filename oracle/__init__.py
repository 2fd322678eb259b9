"""Plain, slow, fp64 CPU ORACLE for MMInference's sparse pre-fill hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` leg may import or execute this
package.  The product path (`paper_2504_16083_b200/`) never imports it, and
this package never imports the product path; the two share only the seeded
input generators in `synth/` (which hold none of the method's arithmetic).

What it computes:
  O1 modality bookkeeping            -> oracle.modality   (Alg.2, Alg.3)
  O2 last_q slab estimate A-hat      -> oracle.estimate   (Alg.1)
  O3 index selection (VS, Grid)      -> oracle.estimate   (Alg.1)
  O4 element-exact masks             -> oracle.masks      (tab:search_space)
  O5 masked attention fp64 + LSE     -> oracle.attention  (Alg.5 P:920-983 semantics)
  O6 per-row fingerprints            -> oracle.attention
  end to end per head                -> oracle.pipeline

Parity pins: see tests/test_oracle_*.py.  "parity unpinned" parts: the
estimator's *rule* (readings C5-C7, C15 of SURVEY.md §8c) is not fixed by the
paper; it is pinned only by brute-force re-enumeration of this oracle's own
definitions plus planted-structure recovery (tests/test_oracle_estimate.py).
"""
