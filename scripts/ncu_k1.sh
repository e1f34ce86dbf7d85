set -u
mkdir -p gpurun_out/k1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_prim" -s 3 -c 2 \
  -o gpurun_out/k1/band -f python scripts/run_band.py c5 8 3 6 > gpurun_out/k1/band.log 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_prim" -s 3 -c 2 \
  -o gpurun_out/k1/c3 -f python scripts/run_band.py c3 1 0 6 > gpurun_out/k1/c3.log 2>&1; echo "rc=$?"
