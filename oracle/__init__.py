"""CPU oracle for the fused-DAG hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and
only as the checker or the timed CPU baseline — never as part of the product
path (``paper_2410_21120_b200`` does not import it and fails loudly when its
CUDA library is missing).

Contents
  executor_ref  numpy restatement of the reference executor
                (/root/reference/pkg/src/dagfuse/executor.py:56-184):
                ``run_faithful`` keeps the reference fold order (bitwise equal
                to the reference on its nine kinds); ``run_fast`` computes the
                same functions with BLAS over a batch (reference-equal up to
                fp32 reassociation) for real-size models.
  liveness_ref  independent interval-overlap recount of the reference peak
                (/root/reference/pkg/tests/test_repo.py:42-59).
  calibrate     data-calibrated init statistics for the zoo models.

Pinning: tests/golden/make_golden.py imports the reference package from
/root/reference (read-only, in the build container) and records its outputs;
tests/test_oracle.py checks this restatement against those fixtures bitwise.
Extension kinds (depthwise/grouped conv, padded pools, avgpool, hardswish,
hardsigmoid, SiLU, sigmoid, channel_scale) have no reference code: they are
pinned by known-answer tests and by torchvision CPU fp32 cross-checks
(tests/test_zoo_torchvision.py).
"""
