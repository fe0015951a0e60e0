# argmax kernel rewrite: tests that compare served first tokens, then the C2 step launch list
set -u
timeout 900 python -m pytest tests/test_gpu.py tests/test_dropin.py -q -m gpu -k "executor or argmax or serving_path or reference_precision or acceptance or bit_identical" 2>&1 | tail -1
TKV_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/argmax_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --nocache-queries 0 > /dev/null 2>&1
python profiles/ncu_summary.py launches gpurun_out/argmax_launches.csv
