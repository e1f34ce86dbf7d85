#!/bin/bash
# One GPU round: build, smoke, gpu tests, bench, ncu launch list + full capture of the top kernels.
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log | cut -c1-400
if [ "${NCU:-1}" = "1" ]; then
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on \
     -k regex:"k_step|k_forward|k_backward|k_bin_rows|k_prim" -s 30 -c 8 \
     -o gpurun_out/prof_full -f python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
  ls -la gpurun_out/*.ncu-rep 2>/dev/null
fi
tail -2 gpurun_out/smoke.log
