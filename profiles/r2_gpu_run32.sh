# round 2 (late): the committed default build — full GPU suite, smoke, default C4 line
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest32.log 2>&1; tail -1 gpurun_out/pytest32.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke32.log 2>&1; tail -1 gpurun_out/smoke32.log
timeout 1500 python bench.py > gpurun_out/bench32_c4.json 2> gpurun_out/bench32_c4.err
tail -c 300 gpurun_out/bench32_c4.json
