# End-of-round-2 evidence run (re-run after the single-stream attention items) on one B200: full GPU suite (+ the Llama-width parity report), smoke,
# the default C4 line and the other configurations, the reference CPU arm, the 2-rank path on one
# GPU, the launch list of one C4 serving step and a --set full capture of its GEMMs (roofline traffic).
set -u
O=gpurun_out
TKV_PARITY_REPORT=$O/parity_llama2l.json timeout 2000 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1500 python bench.py --steps 5 --warmup 3 > $O/final_c4.json 2> $O/final_c4.err; tail -c 300 $O/final_c4.err
timeout 900 python bench.py --impl reference > $O/final_ref.json 2> $O/final_ref.err
timeout 900 python bench.py --config c1 > $O/final_c1.json 2> /dev/null
timeout 900 python bench.py --config c1 --dtype bf16 --no-cpu-baseline > $O/final_c1_bf16.json 2> /dev/null
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 > $O/final_c2.json 2> /dev/null
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > $O/final_c3.json 2> /dev/null
timeout 1800 python bench.py --config c5 --steps 2 --warmup 3 --nocache-queries 50 --no-cpu-baseline > $O/final_c5.json 2> /dev/null
timeout 900 python bench.py --config c2 --policy fifo --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > $O/final_c2_fifo.json 2> /dev/null
TKV_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 3 --queries 250 --pool-pages 6000 --shard interleave --no-cpu-baseline --nocache-queries 0 > $O/final_2rank_onegpu.json 2> $O/final_2rank_onegpu.err
TKV_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/final_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --nocache-queries 0 > /dev/null 2>&1
python profiles/ncu_summary.py launches $O/final_launches.csv > $O/final_launches.txt 2>&1
C="python bench.py --config c4 --queries 200 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_tc_persistent --csv --log-file $O/gemm_launches.csv $C > /dev/null 2>&1
N=$(grep -c "gpu__time_duration" $O/gemm_launches.csv)
SKIP=$(( N * 8 / 10 ))
timeout 1500 ncu --set full --clock-control none -k regex:gemm_tc_persistent --launch-skip $SKIP --launch-count 4 -o $O/r2_gemm_c4 $C > /dev/null 2>&1
ncu -i $O/r2_gemm_c4.ncu-rep --page raw --csv > $O/r2_gemm_c4_raw.csv 2>/dev/null
for c in c4 c1 c1_bf16 c2 c3 c5 c2_fifo 2rank_onegpu; do python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[2],round(d['value'],1),d['p50_ttft_ms'],d['e2e']['value'],d.get('attention_ms_per_step'),round(d['ms_per_step'],1),d['nocache'].get('p50_ttft_reduction'),d['clocks']['reasons'])" $O/final_$c.json $c; done
tail -c 400 $O/final_ref.json
cat $O/final_launches.txt
