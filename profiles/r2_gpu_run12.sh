# round 2: layer-ordered demand loads (prefill starts after the first 4 layers' K/V land) — tests, C4/C5 A/B
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "executor or parity or paged or serving or peer or bench" 2>&1 | tail -3 > gpurun_out/gpu_subset12.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0"
timeout 900 $B > gpurun_out/c4_layered.json 2> gpurun_out/c4_layered.err
TKV_LAYERED_LOADS=0 timeout 900 $B > gpurun_out/c4_whole.json 2> gpurun_out/c4_whole.err
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_layered.json 2> gpurun_out/c5_layered.err
TKV_LAYERED_LOADS=0 timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_whole.json 2> gpurun_out/c5_whole.err
cat gpurun_out/gpu_subset12.log
