# bench + timelines of library variants built by scripts/ab_build.sh: bash scripts/ab_variants.sh v1 v2 ...
set -u
b() { timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-autograd "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,2), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()}, round(d['e2e']['value']), round(d['run_loop']['value']), d['clocks']['sm_mhz'])"; }
for v in "$@"; do
  L=paper_2602_22625_b200/_lib_alt/$v.so
  echo "== $v c3: $(PF_LIB=$L b)"
  echo "== $v c5: $(PF_LIB=$L b --config c5 --steps 50)"
  echo "== $v c2: $(PF_LIB=$L b --config c2)"
done
