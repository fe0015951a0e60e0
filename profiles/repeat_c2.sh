# run-to-run spread of the default C2 bench line on one box
set -u
for i in 1 2 3; do timeout 900 python bench.py --no-cpu-baseline > gpurun_out/rep_c2_$i.json 2>/dev/null; python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],round(d['value'],1),round(d['e2e']['value'],1),round(d['ms_per_step'],1),d['p50_ttft_ms'],d['clocks']['sm_mhz'],d['clocks']['reasons'])" gpurun_out/rep_c2_$i.json run$i; done
