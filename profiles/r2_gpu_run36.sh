# round 2 (final build): full GPU suite, smoke, default C4 line, C2 line
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest36.log 2>&1; tail -1 gpurun_out/pytest36.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke36.log 2>&1; tail -1 gpurun_out/smoke36.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/final36_c4.json 2> gpurun_out/final36_c4.err
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 > gpurun_out/final36_c2.json 2> /dev/null
