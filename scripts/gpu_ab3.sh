set -u
b() { timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-autograd 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,2), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()}, round(d['e2e']['value']), round(d['run_loop']['value']), d['clocks']['sm_mhz'])"; }
echo "== old: $(cd _ab_old && b)"
echo "== slot t128: $(PF_LIB=paper_2602_22625_b200/_lib_alt/t128.so b)"
echo "== slot t256: $(PF_LIB=paper_2602_22625_b200/_lib_alt/t256.so b)"
echo "== csr t256: $(PF_CSR_STEP=1 PF_LIB=paper_2602_22625_b200/_lib_alt/t256.so b)"
echo "== old: $(cd _ab_old && b)"
echo "== old timeline"; (cd _ab_old && timeout 300 python scripts/timeline.py c3 2>&1 | tail -9)
echo "== slot t256 timeline"; PF_LIB=paper_2602_22625_b200/_lib_alt/t256.so timeout 300 python scripts/timeline.py c3 2>&1 | tail -9
echo "== old step_prof"; (cd _ab_old && timeout 300 python scripts/step_prof.py c3 2>&1 | tail -16 | head -6)
