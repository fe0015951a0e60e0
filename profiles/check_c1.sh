# c1 regression check + the reference acceptance gate through the drop-in API
set -u
timeout 900 python -m pytest tests/test_dropin.py -x -q -m gpu 2>&1 | tail -1
for i in 1 2; do timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/c1_$i.json 2>/dev/null; python -c "import json,sys;d=json.load(open(sys.argv[1]));print(d['value'],d['p50_ttft_ms'],d['p99_ttft_ms'],d['e2e']['value'],d['e2e']['last_step_ms'])" gpurun_out/c1_$i.json; done
TKV_HOST_PROFILE=1 timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/c1_prof.json 2> gpurun_out/c1_prof.err; tail -30 gpurun_out/c1_prof.err
