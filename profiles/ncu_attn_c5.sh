# ncu of ONE serving-path attention launch of the C5 bench: list every attn_tc5 launch (duration
# only), pick one at 80% of the run (the serving / e2e phase, past the corpus precompute), then a
# --set full capture of that launch
set -u
B="python bench.py --config c5 --capacity 64 --queries 1250 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_tc5 --csv --log-file gpurun_out/attn_c5_launches.csv $B > /dev/null 2>&1
N=$(grep -c "gpu__time_duration" gpurun_out/attn_c5_launches.csv)
SKIP=$(( N * 8 / 10 ))
echo "launches $N skip $SKIP"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attn_tc5 --launch-skip $SKIP --launch-count 1 -o gpurun_out/r1_attn_c5_serving $B > /dev/null 2>&1
ls -la gpurun_out/r1_attn_c5_serving.ncu-rep
