# ncu A/B of the fused step: slot mode (default) vs CSR mode (PF_CSR_STEP=1), c3
set -u
mkdir -p gpurun_out/ab
for mode in slot csr; do
  if [ $mode = csr ]; then export PF_CSR_STEP=1; else unset PF_CSR_STEP; fi
  timeout 900 ncu --set full --clock-control none --import-source on \
     -k regex:"k_step|k_prim" -s 20 -c 4 \
     -o gpurun_out/ab/prof_$mode -f python bench.py --steps 3 --warmup 3 --no-cpu --no-autograd \
     > gpurun_out/ab/ncu_$mode.log 2>&1; echo "ncu $mode rc=$?"
  python scripts/ncu_extract.py gpurun_out/ab/prof_$mode.ncu-rep gpurun_out/ab/k_$mode.json > /dev/null 2>&1
done
unset PF_CSR_STEP
