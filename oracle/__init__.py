"""CPU oracle for the Zeppelin per-layer hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU baseline.  The product path (``paper_2509_21841_b200``) never
imports it and has no CPU fallback.

Pinning:
* plans / schedules / remap matrices: the reference implementation itself
  (live in this container, tests/test_planner_parity.py) and committed
  fixtures generated from it (tests/golden/planner_golden.json);
* mask semantics: per ring round, the oracle's unmasked (q,k) count equals the
  reference schedule's ``compute_pairs`` (attention_engine.py:229-244);
* softmax arithmetic: the reference has none ("No actual attention math",
  SPEC.md:279) — the numerics are pinned against torch's independent
  scaled_dot_product_attention in float64 (tests/test_oracle.py).  Attention
  parity is therefore anchored on the reference's mask/pair counts plus an
  independent fp64 implementation, not on reference output vectors.
"""
