# round 2 (late): attention items dealt to the persistent CTAs in snake order with a cost model
# (default) vs plain heaviest-first round robin (TKV_ATTN_STRIDE_ORDER=1), C4 and C5; then the GPU suite
set -x
B="python bench.py --steps 3 --warmup 3 --nocache-queries 0 --no-cpu-baseline"
timeout 900 $B --config c4 > gpurun_out/ab33_c4_snake.json 2> gpurun_out/ab33_c4_snake.err
TKV_ATTN_STRIDE_ORDER=1 timeout 900 $B --config c4 > gpurun_out/ab33_c4_stride.json 2> gpurun_out/ab33_c4_stride.err
timeout 1200 $B --config c5 --steps 2 > gpurun_out/ab33_c5_snake.json 2> gpurun_out/ab33_c5_snake.err
TKV_ATTN_STRIDE_ORDER=1 timeout 1200 $B --config c5 --steps 2 > gpurun_out/ab33_c5_stride.json 2> gpurun_out/ab33_c5_stride.err
timeout 900 $B --config c2 > gpurun_out/ab33_c2_snake.json 2> gpurun_out/ab33_c2_snake.err
TKV_ATTN_STRIDE_ORDER=1 timeout 900 $B --config c2 > gpurun_out/ab33_c2_stride.json 2> gpurun_out/ab33_c2_stride.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest33.log 2>&1; tail -1 gpurun_out/pytest33.log
