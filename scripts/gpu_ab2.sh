set -u
b() { timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-autograd 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,2), d['stage_ms'], round(d['e2e']['value']), round(d['run_loop']['value']))"; }
for mode in slot csr slot csr; do
  if [ $mode = csr ]; then export PF_CSR_STEP=1; else unset PF_CSR_STEP; fi
  echo "== $mode bench: $(b)"
done
for mode in slot csr; do
  if [ $mode = csr ]; then export PF_CSR_STEP=1; else unset PF_CSR_STEP; fi
  echo "== $mode timeline"; timeout 300 python scripts/timeline.py c3 2>&1 | tail -9
  echo "== $mode step_prof"; timeout 300 python scripts/step_prof.py c3 2>&1 | tail -16
done
