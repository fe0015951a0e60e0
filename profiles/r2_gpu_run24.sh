# round 2: GEMM variants at the C4/C5 window sizes (M ~ 9.7k / ~12k rows): single-CTA (default) vs 2-SM UMMA vs B-multicast pairs
set -x
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0"
TKV_GEMM=2sm timeout 900 $B > gpurun_out/c4_2sm.json 2> gpurun_out/c4_2sm.err
TKV_GEMM=pair timeout 900 $B > gpurun_out/c4_pair.json 2> gpurun_out/c4_pair.err
timeout 900 $B > gpurun_out/c4_single.json 2> gpurun_out/c4_single.err
TKV_GEMM=2sm timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_2sm.json 2> gpurun_out/c5_2sm.err
