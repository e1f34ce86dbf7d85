mkdir -p gpurun_out/sanitize
cd scripts/sanitize_repro
for v in 0 1; do for gg in 1 3; do
  for tool in racecheck synccheck; do
    compute-sanitizer --tool $tool ./ring_${v}_g$gg > ../../gpurun_out/sanitize/ring${v}_g${gg}_${tool}.log 2>&1
    echo "ring setmaxnreg=$v groups=$gg $tool: $(grep -E 'SUMMARY|ring:' ../../gpurun_out/sanitize/ring${v}_g${gg}_${tool}.log | tr '\n' ' ')"
  done
done; done
