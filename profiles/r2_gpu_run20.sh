# round 2: K rotation with packed f32x2 math (fewer issue slots beside the softmax) — tests, C4/C2/C5
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "paged or parity or serving" 2>&1 | tail -5 > gpurun_out/gpu_subset20.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c4_rot2.json 2> gpurun_out/c4_rot2.err
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c2_rot2.json 2> gpurun_out/c2_rot2.err
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_rot2.json 2> gpurun_out/c5_rot2.err
cat gpurun_out/gpu_subset20.log
