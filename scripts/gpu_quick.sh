#!/bin/bash
# Quick GPU iteration: build, GPU parity tests, bench variants (no CPU baseline), launch list.
set -u
mkdir -p gpurun_out
timeout 180 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log; grep -q "smoke ok\|OK" gpurun_out/smoke.log || { echo SMOKE FAILED; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-"-"}; do
  if [ "$v" = "-" ]; then env_v=""; else env_v="$v"; fi
  echo "== variant $v"
  env $env_v timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_q.log 2>&1
  tail -1 gpurun_out/bench_q.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms'], d['e2e']['value'])" || tail -5 gpurun_out/bench_q.log
done
if [ "${NCU:-0}" = "1" ]; then
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on \
     -k regex:"${NCU_K:-k_step|k_bin_rows|k_prim}" -s 30 -c 6 \
     -o gpurun_out/prof_full -f python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
  ls -la gpurun_out/*.ncu-rep 2>/dev/null
fi
