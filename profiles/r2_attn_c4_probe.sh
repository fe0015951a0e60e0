# C4 serving attention: CTA-0 timeline (TKV_ATTN_TRACE) and one --set full ncu capture with source
set -u
B="python bench.py --config c4 --queries 200 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline"
TKV_ATTN_TRACE=gpurun_out/attn_c4_trace.bin timeout 900 $B > gpurun_out/attn_c4_trace_bench.json 2>&1
python profiles/attn_trace.py gpurun_out/attn_c4_trace.bin > gpurun_out/attn_c4_trace.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_tc5 --csv --log-file gpurun_out/attn_c4_launches.csv $B > /dev/null 2>&1
N=$(grep -c "gpu__time_duration" gpurun_out/attn_c4_launches.csv)
SKIP=$(( N * 8 / 10 ))
echo "launches $N skip $SKIP"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attn_tc5 --launch-skip $SKIP --launch-count 1 -o gpurun_out/r2_attn_c4 $B > /dev/null 2>&1
ls -la gpurun_out/r2_attn_c4.ncu-rep
