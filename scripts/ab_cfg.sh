# bench A/B of library variants on one config, alternating, 2 rounds:
# bash scripts/ab_cfg.sh <config> v1 v2 ...
set -u
c=$1; shift
for r in 1 2; do for v in "$@"; do
  echo "== $v $c: $(PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu --no-autograd 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), round(d['run_loop']['value']))")"
done; done
