#!/bin/bash
# NOTE: compute-sanitizer is closed on the B200 pool this repo was developed on
# (runs under it left GPUs needing a reset); kept for other machines.
# compute-sanitizer over the device path at small sizes (one B200):
# memcheck (out-of-bounds / misaligned / leaks), racecheck (shared-memory
# hazards), synccheck (barrier misuse), initcheck (uninitialised global reads)
# on smoke() and on the parity tests that exercise the atomic-heavy kernels
# (Alg. 2 counters, splats, field bin counters, multi-rank exchange).
O=gpurun_out/sanitizer
mkdir -p $O
export WFPG_SANITIZE=1
T="tests/test_queries.py::test_atomic_splat_matches_ordered_splat tests/test_render_parity.py::test_pass_pipeline_equals_sequential_passes tests/test_multigpu_gpu.py::test_banded_ranks_reproduce_the_one_gpu_passes"
for tool in memcheck racecheck synccheck initcheck; do
  compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 \
      python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$tool.log 2>&1
  echo "smoke $tool rc=$?"
done
compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 99 \
    python -m pytest -q -x $T -m gpu > $O/tests_memcheck.log 2>&1
echo "tests memcheck rc=$?"
compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 99 \
    python -m pytest -q -x tests/test_render_parity.py -k "partition and 256" -m gpu \
    > $O/tests_racecheck.log 2>&1
echo "tests racecheck rc=$?"
