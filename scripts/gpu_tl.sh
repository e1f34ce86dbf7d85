set -u
mkdir -p gpurun_out/tl
for a in "c5" "c5 band=8:0" "c5 band=8:3" "c5 band=8:7" "c3"; do
  echo "== $a"; timeout 300 python scripts/timeline.py $a 2>&1 | tail -16
done > gpurun_out/tl/timeline.txt
cat gpurun_out/tl/timeline.txt
