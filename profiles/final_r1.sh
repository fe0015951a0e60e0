# End-of-round evidence run on one B200: full GPU suite, smoke, every bench configuration, the
# reference CPU arm, and the ncu launch list of one C2 serving step.
set -u
O=gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/final_c2.json 2> $O/final_c2.err; tail -c 300 $O/final_c2.err
timeout 900 python bench.py --impl reference > $O/final_ref.json 2> $O/final_ref.err
timeout 900 python bench.py --config c1 --no-cpu-baseline > $O/final_c1.json 2> /dev/null
timeout 900 python bench.py --config c3 --queries 500 --capacity 256 --steps 2 --warmup 3 --nocache-queries 100 --no-cpu-baseline > $O/final_c3.json 2> /dev/null
timeout 900 python bench.py --config c3 --queries 500 --capacity 32 --steps 2 --warmup 3 --nocache-queries 50 --no-cpu-baseline > $O/final_c4.json 2> /dev/null
timeout 1500 python bench.py --config c5 --queries 1250 --capacity 64 --steps 2 --warmup 3 --nocache-queries 100 --no-cpu-baseline > $O/final_c5.json 2> /dev/null
timeout 900 python bench.py --policy fifo --steps 3 --warmup 3 --no-cpu-baseline > $O/final_fifo.json 2> /dev/null
TKV_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/final_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --nocache-queries 0 > /dev/null 2>&1
python profiles/ncu_summary.py launches $O/final_launches.csv > $O/final_launches.txt 2>&1
for c in c2 c1 c3 c4 c5 fifo; do python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],round(d['value'],1),d['p50_ttft_ms'],d['e2e']['value'],d.get('attention_ms_per_step'),d['gather']['ms_per_step'] if d.get('gather') else None,round(d['ms_per_step'],1),d['nocache'].get('p50_ttft_reduction'),d['clocks']['reasons'])" $O/final_$c.json $c; done
tail -c 400 $O/final_ref.json
cat $O/final_launches.txt
