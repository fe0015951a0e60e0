# round 2: e2e vs timed gap (kernel-event timing on / host lead), attention timeline with both streams, ncu of one C4 attention launch
set -x
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0"
TKV_E2E_TIMED=1 timeout 900 $B > gpurun_out/c4_e2e_timed.json 2> gpurun_out/c4_e2e_timed.err
TKV_HOST_LEAD=1 timeout 900 $B > gpurun_out/c4_lead1.json 2> gpurun_out/c4_lead1.err
TKV_ATTN_TRACE=gpurun_out/attn_c4_trace.bin timeout 900 python bench.py --config c4 --queries 200 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > /dev/null 2>&1
python profiles/attn_trace.py gpurun_out/attn_c4_trace.bin > gpurun_out/attn_c4_trace.txt 2>&1
C="python bench.py --config c4 --queries 200 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c4_launches.csv $C > /dev/null 2>&1
N=$(grep -c "attn_tc5" gpurun_out/r2_c4_launches.csv)
SKIP=$(( N * 8 / 10 ))
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attn_tc5 --launch-skip $SKIP --launch-count 1 -o gpurun_out/r2_attn_c4_paged $C > /dev/null 2>&1
ncu -i gpurun_out/r2_attn_c4_paged.ncu-rep --page raw --csv > gpurun_out/r2_attn_c4_paged_raw.csv 2>/dev/null
ncu -i gpurun_out/r2_attn_c4_paged.ncu-rep --page source --csv > gpurun_out/r2_attn_c4_paged_source.csv 2>/dev/null
ls -la gpurun_out/
