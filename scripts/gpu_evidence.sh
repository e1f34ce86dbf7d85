#!/bin/bash
# Round evidence on one GPU: default bench line, ncu launch list of the same
# command, ncu --set full captures (c3 fused step, c3 two-kernel path, c5 step),
# kernel timelines, band scaling, (no sanitizer: closed on this pool).
set -u
O=gpurun_out/ev7
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -1 $O/bench.json | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-autograd \
   > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"k_step|k_prim" -s 20 -c 4 \
   -o $O/prof_c3 -f python bench.py --steps 3 --warmup 3 --no-cpu --no-autograd \
   > $O/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
PF_TWO_KERNEL=1 timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"k_forward|k_backward|k_bin_rows" -s 30 -c 6 \
   -o $O/prof_c3_2k -f python bench.py --steps 3 --warmup 3 --no-cpu --no-autograd \
   > $O/ncu_c3_2k.log 2>&1; echo "ncu c3 two-kernel rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"k_step|k_prim" -s 20 -c 4 \
   -o $O/prof_c5 -f python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-autograd \
   > $O/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
for a in "c3" "c5" "c5 band=8:3" "c3 hostio"; do
  echo "== $a"; timeout 300 python scripts/timeline.py $a 2>&1 | tail -8
done > $O/timelines.txt
timeout 900 python scripts/band_scaling.py c5 1 2 4 8 > $O/band_scaling.txt 2>&1; echo "band rc=$?"
cp gpurun_out/band_scaling_c5.json $O/ 2>/dev/null
# (compute-sanitizer is closed on this pool: the r02f logs under profiles/ are the last runs)
# summaries on the box (the reports are too large to bring back together)
for r in prof_c3 prof_c3_2k prof_c5; do
  python scripts/ncu_extract.py $O/$r.ncu-rep $O/${r}_kernels.json > /dev/null 2>&1
  ncu -i $O/$r.ncu-rep --page source --print-source cuda,sass --csv -k regex:"k_step|k_forward" \
     --launch-count 1 > $O/${r}_src.csv 2>/dev/null
  python scripts/ncu_lines.py $O/${r}_src.csv 40 > $O/${r}_lines.txt 2>&1
  rm -f $O/${r}_src.csv
done
ncu -i $O/prof_c3.ncu-rep --page raw --csv > $O/prof_c3_raw.csv 2>/dev/null
rm -f $O/prof_c3_2k.ncu-rep $O/prof_c5.ncu-rep
ls -la $O
