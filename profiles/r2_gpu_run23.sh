# round 2: metadata uploads by an SM copy kernel from the mapped ring (no DMA queueing behind page copies)
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "serving or executor or parity or paged or encode" 2>&1 | tail -5 > gpurun_out/gpu_subset23.log
rm -f gpurun_out/timing.txt; TKV_DUMP_TIMING=gpurun_out/timing.txt timeout 1000 python scratch/w0_dump.py > gpurun_out/w0_dump2.txt 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c4_smup.json 2> gpurun_out/c4_smup.err
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_smup.json 2> gpurun_out/c5_smup.err
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c2_smup.json 2> gpurun_out/c2_smup.err
cat gpurun_out/gpu_subset23.log
