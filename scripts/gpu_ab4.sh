set -u
b() { timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-autograd "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,2), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()}, round(d['e2e']['value']), round(d['run_loop']['value']), d['clocks']['sm_mhz'])"; }
echo "== old: $(cd _ab_old && b)"
for v in t128 t256x2 t256x4; do
  echo "== slot $v: $(PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so b)"
done
echo "== csr t256x2: $(PF_CSR_STEP=1 PF_LIB=paper_2602_22625_b200/_lib_alt/t256x2.so b)"
for v in t128 t256x2; do
  echo "== slot $v timeline c3"; PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python scripts/timeline.py c3 2>&1 | tail -6
  echo "== slot $v timeline c5"; PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python scripts/timeline.py c5 2>&1 | tail -6
  echo "== slot $v timeline c5 band"; PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python scripts/timeline.py c5 band=8:3 2>&1 | tail -6
done
echo "== old c5"; (cd _ab_old && timeout 300 python scripts/timeline.py c5 2>&1 | tail -13)
