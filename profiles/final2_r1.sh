# final GPU suite + smoke, and a --set full capture of one K-only head-major gather launch (C5)
set -u
timeout 1600 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_final.log 2>&1; tail -1 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gather_rope_tma --launch-skip 3000 --launch-count 1 -o gpurun_out/r1_gather_konly python bench.py --config c5 --capacity 64 --queries 1250 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/r1_gather_konly.ncu-rep
