# round 2: TMA single-row swizzle probe; folded RMSNorm (tests + C4 A/B)
set -x
./scratch/tma_probe > gpurun_out/tma_probe.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "fold or parity or paged" 2>&1 | tail -5 > gpurun_out/gpu_subset6.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0"
timeout 900 $B > gpurun_out/c4_fold.json 2> gpurun_out/c4_fold.err
TKV_NORM_FOLD=0 timeout 900 $B > gpurun_out/c4_nofold.json 2> gpurun_out/c4_nofold.err
cat gpurun_out/tma_probe.txt gpurun_out/gpu_subset6.log
