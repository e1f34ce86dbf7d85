set -u
timeout 600 python -m pytest tests/test_gpu_slots.py -x -q 2>&1 | tail -3
b() { timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-autograd "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,2), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()}, round(d['e2e']['value']), round(d['run_loop']['value']), d['clocks']['sm_mhz'])"; }
echo "== old c3: $(cd _ab_old && b)"
echo "== new c3: $(b)"
echo "== csr c3: $(PF_CSR_STEP=1 b)"
for a in "c3" "c5" "c5 band=8:3"; do echo "== tl $a"; timeout 300 python scripts/timeline.py $a 2>&1 | tail -6 | head -3; done
timeout 600 python scripts/band_scaling.py c5 1 8 2>&1 | tail -3
