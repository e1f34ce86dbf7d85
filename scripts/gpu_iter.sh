# quick iteration on one GPU: slot tests, timelines, default bench line
set -u
mkdir -p gpurun_out/it
timeout 900 python -m pytest tests/test_gpu_slots.py -x -q > gpurun_out/it/slots.log 2>&1; echo "slots rc=$?"; tail -25 gpurun_out/it/slots.log
for a in "c3" "c5" "c5 band=8:3"; do
  echo "== $a"; timeout 300 python scripts/timeline.py $a 2>&1 | tail -12
done
timeout 600 python bench.py --no-cpu --no-autograd > gpurun_out/it/bench.json 2> gpurun_out/it/bench.err; echo "bench rc=$?"; tail -1 gpurun_out/it/bench.json | cut -c1-700
