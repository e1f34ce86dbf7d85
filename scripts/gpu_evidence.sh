#!/bin/bash
# Round evidence on one GPU: default bench line, ncu launch list of the same
# command, ncu --set full captures (c3 fused step, c3 two-kernel path, c5 step),
# kernel timeline, racecheck with the full hazard list.
set -u
mkdir -p gpurun_out/ev
timeout 900 python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/ev/bench.json | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/ev/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-autograd \
   > gpurun_out/ev/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"k_step|k_bin_rows|k_prim" -s 30 -c 6 \
   -o gpurun_out/ev/prof_c3 -f python bench.py --steps 3 --warmup 3 --no-cpu --no-autograd \
   > gpurun_out/ev/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
PF_TWO_KERNEL=1 timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"k_forward|k_backward" -s 20 -c 4 \
   -o gpurun_out/ev/prof_c3_2k -f python bench.py --steps 3 --warmup 3 --no-cpu --no-autograd \
   > gpurun_out/ev/ncu_c3_2k.log 2>&1; echo "ncu c3 two-kernel rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"k_step|k_bin_rows|k_row|k_prim" -s 40 -c 8 \
   -o gpurun_out/ev/prof_c5 -f python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-autograd \
   > gpurun_out/ev/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
timeout 300 python scripts/timeline.py c3 > gpurun_out/ev/timeline_c3.txt 2>&1; echo "timeline rc=$?"
NV_COMPUTE_SANITIZER_MAX_RACECHECK_HAZARDS=100000 timeout 900 compute-sanitizer --tool racecheck \
   python scripts/sanitize_step.py c3 2 > gpurun_out/ev/c3_racecheck_full.log 2>&1; echo "racecheck rc=$?"
ls -la gpurun_out/ev
