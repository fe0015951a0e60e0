# round 2: attention ring split K3/V2 (default) vs K2/V3 (V loads were late in the C2/C4 timelines)
set -x
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0"
TKV_LIB=paper_2601_08743_b200/lib/k2v3/libtkv.so timeout 900 $B > gpurun_out/c4_k2v3.json 2> gpurun_out/c4_k2v3.err
timeout 900 $B > gpurun_out/c4_k3v2.json 2> gpurun_out/c4_k3v2.err
TKV_LIB=paper_2601_08743_b200/lib/k2v3/libtkv.so timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c2_k2v3.json 2> gpurun_out/c2_k2v3.err
TKV_LIB=paper_2601_08743_b200/lib/k2v3/libtkv.so timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_k2v3.json 2> gpurun_out/c5_k2v3.err
