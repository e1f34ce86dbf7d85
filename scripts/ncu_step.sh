#!/bin/bash
# ncu --set full of one k_step launch (steady state), report into gpurun_out/prof_step.ncu-rep
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_step}" -s ${NCU_S:-10} -c 1 \
   -o gpurun_out/prof_step -f python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_step.log 2>&1
tail -2 gpurun_out/ncu_step.log
