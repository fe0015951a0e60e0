# round 2 (final build): the remaining configuration lines, the reference arm and the 2-rank path
set -u
O=gpurun_out
timeout 900 python bench.py --impl reference > $O/f38_ref.json 2> $O/f38_ref.err
timeout 900 python bench.py --config c1 > $O/f38_c1.json 2> /dev/null
timeout 900 python bench.py --config c1 --dtype bf16 --no-cpu-baseline > $O/f38_c1_bf16.json 2> /dev/null
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > $O/f38_c3.json 2> /dev/null
timeout 1800 python bench.py --config c5 --steps 2 --warmup 3 --nocache-queries 50 --no-cpu-baseline > $O/f38_c5.json 2> /dev/null
timeout 900 python bench.py --config c2 --policy fifo --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > $O/f38_c2_fifo.json 2> /dev/null
TKV_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 3 --queries 250 --pool-pages 6000 --shard interleave --no-cpu-baseline --nocache-queries 0 > $O/f38_2rank_onegpu.json 2> $O/f38_2rank_onegpu.err
ls -la $O/f38_*
