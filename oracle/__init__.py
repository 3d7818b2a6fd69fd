"""CPU oracle for the PipeOptim hot path — TEST INFRASTRUCTURE ONLY.

A restatement of the reference simulator's algorithm (arXiv 2312.00839's
`pipesim`, /root/reference/pkg/src/pipesim) in numpy float64, following the
reference file:line by file:line:

  optim_ref.py     OptimizerConfig / OptimizerState / predict_weights /
                   version_difference                    (optim.py:17-167)
  schedule_ref.py  1F1B timeline, validation, gaps, bubbles, makespan
                                                         (schedule.py, runtime.py:300-315)
  rng_ref.py       Philox RngStream keyed by SHA-256     (linalg.py:141-167)
  data_ref.py      tiny-classification / synthetic-regression / two-spirals
                   datasets and BatchStream               (data.py)
  runtime_ref.py   dense-MLP stages, losses, the strategy-aware executor for
                   the 1F1B path (async_raw, optimizer_prediction, spectrain)
                                                         (stages.py, linalg.py,
                                                          runtime.py:66-496)
  c/optim_oracle.c the optimizer/predictor rules in C (fp64, OpenMP) — the
                   multi-core CPU baseline for bench.py; checked against
                   optim_ref.py

Pinning: every function here is checked (tests/test_oracle.py) against the
reference's own golden vectors (FROZEN_* trajectories in
pkg/tests/test_optim.py:42-53, the schedule/record known answers in
pkg/tests/test_schedule.py and test_runtime.py) and against fixtures generated
by importing the reference itself in the build container
(tests/golden/make_golden.py -> tests/golden/*.json|npz).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package, and only as the checker or the timed CPU
baseline — never on the product path.
"""
