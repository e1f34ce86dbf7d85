set -u
L=paper_2602_22625_b200/_lib_alt/t256x2.so
timeout 600 env PF_LIB=$L python -m pytest tests/test_gpu_slots.py -x -q 2>&1 | tail -3
b() { timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-autograd "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,2), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()}, round(d['e2e']['value']), round(d['run_loop']['value']), d['clocks']['sm_mhz'])"; }
echo "== old c3: $(cd _ab_old && b)"
for v in t256x2 t256x3 t128; do echo "== slot $v c3: $(PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so b)"; done
for cfg in c5 c3; do echo "== $cfg step_prof"; PF_LIB=$L timeout 300 python scripts/step_prof.py $cfg 2>&1 | head -3; done
for a in "c3" "c5" "c5 band=8:3"; do echo "== tl $a"; PF_LIB=$L timeout 300 python scripts/timeline.py $a 2>&1 | tail -6 | head -3; done
