"""CPU oracle for the prefix-shared attention hot path — TEST INFRASTRUCTURE ONLY.

Nothing in the product path (``paper_2412_03594_b200``) imports this package.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may use it, and only as the checker or as the timed
reference arm — never as the thing measured for the GPU arm or shipped.

Contents
--------
``segmented``  float64 NumPy restatement of ``pkg/src/prefixbatch/attention.py``
               (the reference's semantic oracle), function by function, with
               file:line citations, plus the multi-head/GQA adapter that calls
               it once per (group, kv-head).
``plan``       pure-Python restatement of the work-item planner implemented in
               C++ inside ``libpsa.so`` (``psa_plan``); the int32 tables the two
               produce must be byte-identical. ``plan.group_costs`` /
               ``plan.shard_groups`` restate the group→rank LPT partition
               (``psa_group_costs`` / ``psa_shard_groups``).

Parity pinning: ``segmented`` is checked against golden vectors produced by
importing the reference itself (``tests/golden/make_golden.py``, run in the
build container where ``/root/reference`` exists) and against every
known-answer test of ``pkg/tests/test_attention.py`` and acceptance criterion 6
(``pkg/tests/test_acceptance.py:178-225``), restated in
``tests/test_oracle.py``.
"""
