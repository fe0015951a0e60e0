# round 2, session 4: batched encode tests, C4 bench with encode + 8x rerank lines, C4 attention probe
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "encode or precompute" 2>&1 | tail -5 > gpurun_out/enc_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
bash profiles/r2_attn_c4_probe.sh
ncu -i gpurun_out/r2_attn_c4.ncu-rep --page raw --csv > gpurun_out/r2_attn_c4_raw.csv 2>/dev/null
ncu -i gpurun_out/r2_attn_c4.ncu-rep --page source --csv > gpurun_out/r2_attn_c4_source.csv 2>/dev/null
cat gpurun_out/enc_tests.log
