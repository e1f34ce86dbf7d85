set -u
mkdir -p gpurun_out/s1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s1/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s1/pytest.log
timeout 600 python bench.py > gpurun_out/s1/bench.json 2> gpurun_out/s1/bench.err; echo "bench rc=$?"; tail -1 gpurun_out/s1/bench.json | cut -c1-400
timeout 600 python scripts/band_scaling.py c5 1 8 > gpurun_out/s1/band.txt 2>&1; echo "band rc=$?"; cat gpurun_out/s1/band.txt | tail -4
