set -u
L=paper_2602_22625_b200/_lib_alt/t256x2.so
timeout 900 env PF_LIB=$L python -m pytest tests/test_gpu_slots.py -x -q 2>&1 | tail -2
for cfg in c5 c3; do
echo "== $cfg slot"; PF_LIB=$L timeout 300 python scripts/step_prof.py $cfg 2>&1 | head -4
done
b() { timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-autograd "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,2), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()}, round(d['e2e']['value']), round(d['run_loop']['value']), d['clocks']['sm_mhz'])"; }
echo "== slot c3: $(PF_LIB=$L b)"
echo "== old c3: $(cd _ab_old && b)"
echo "== slot c5 timeline"; PF_LIB=$L timeout 300 python scripts/timeline.py c5 2>&1 | tail -6 | head -3
echo "== slot c5 band"; PF_LIB=$L timeout 300 python scripts/timeline.py c5 band=8:3 2>&1 | tail -6 | head -3
