# round 2 (final build): ncu launch list of one default C4 serving step
set -x
O=gpurun_out
TKV_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/final37_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --nocache-queries 0 > /dev/null 2>&1
python profiles/ncu_summary.py launches $O/final37_launches.csv > $O/final37_launches.txt 2>&1
cat $O/final37_launches.txt
