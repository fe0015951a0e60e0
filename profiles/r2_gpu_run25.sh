# round 2: lazy staging-ring uploads flushed by one copy kernel per forward — acceptance gate, tests, C1/C4
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -k "dropin or serving or executor or parity or paged or encode or peer" 2>&1 | tail -5 > gpurun_out/gpu_subset25.log
timeout 900 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c1_flush.json 2> gpurun_out/c1_flush.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c4_flush.json 2> gpurun_out/c4_flush.err
cat gpurun_out/gpu_subset25.log
