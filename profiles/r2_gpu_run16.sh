# round 2: host lead (windows the executor's host loop runs ahead: copies of window w start when w-lead ends)
set -x
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0"
timeout 900 $B > gpurun_out/c4_lead2.json 2> gpurun_out/c4_lead2.err
TKV_HOST_LEAD=3 timeout 900 $B > gpurun_out/c4_lead3.json 2> gpurun_out/c4_lead3.err
TKV_HOST_LEAD=4 timeout 900 $B > gpurun_out/c4_lead4.json 2> gpurun_out/c4_lead4.err
TKV_HOST_LEAD=3 timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_lead3.json 2> gpurun_out/c5_lead3.err
TKV_HOST_LEAD=3 timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c2_lead3.json 2> gpurun_out/c2_lead3.err
