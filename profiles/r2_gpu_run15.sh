# round 2: dead-warp skip in the attention softmax (short suffixes) — tests, C4, C2 attention share
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "paged or parity or serving or executor or encode or slab or fold" 2>&1 | tail -3 > gpurun_out/gpu_subset15.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c4_dead.json 2> gpurun_out/c4_dead.err
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c2_dead.json 2> gpurun_out/c2_dead.err
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_dead.json 2> gpurun_out/c5_dead.err
cat gpurun_out/gpu_subset15.log
