mkdir -p gpurun_out/sanitize
for case in c3 c5band; do
PF_NO_PDL=1 timeout 900 compute-sanitizer --tool synccheck --print-limit 200 python scripts/sanitize_step.py $case 1 > gpurun_out/sanitize/${case}_synccheck_nopdl.log 2>&1
echo "$case synccheck nopdl rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/sanitize/${case}_synccheck_nopdl.log | tail -1)"
done
