# round 2 (late): drop-in gather_f32 without a per-call pinned arena (the reference acceptance
# gate's criterion 1 had crossed its 60 s limit) — the drop-in suites first, then the full GPU suite
set -x
timeout 1200 python -m pytest tests/test_dropin.py -m gpu -x -q -rA > gpurun_out/pytest34_dropin.log 2>&1; tail -3 gpurun_out/pytest34_dropin.log
./oracle/_ref/dropin_acceptance tests/golden/demo > gpurun_out/acceptance34.txt 2>&1 || true
cat gpurun_out/acceptance34.txt | tail -12
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest34.log 2>&1; tail -1 gpurun_out/pytest34.log
