# round 2 (late): rotation probe without the math (LDS/STS kept), and one --set full ncu capture
# (with source) of a C4 serving attention launch for per-instruction stall attribution
set -x
B="python bench.py --config c4 --queries 200 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline"
TKV_LIB=paper_2601_08743_b200/lib/nomath/libtkv.so timeout 900 $B > gpurun_out/attn_nomath.json 2> gpurun_out/attn_nomath.err
timeout 900 $B > gpurun_out/attn_base2.json 2> gpurun_out/attn_base2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_tc5 --csv --log-file gpurun_out/attn_c4_launches.csv $B > /dev/null 2>&1
N=$(grep -c "gpu__time_duration" gpurun_out/attn_c4_launches.csv)
SKIP=$(( N * 8 / 10 ))
echo "launches $N skip $SKIP"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attn_tc5 --launch-skip $SKIP --launch-count 1 -o gpurun_out/r2_attn_c4_src $B > gpurun_out/ncu_src.log 2>&1
ls -la gpurun_out/r2_attn_c4_src.ncu-rep
