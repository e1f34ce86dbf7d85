# c3 bench A/B of library variants, alternating, 3 rounds: bash scripts/ab_c3.sh v1 v2 ...
set -u
for r in 1 2 3; do
  for v in "$@"; do
    echo "== $v: $(PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-autograd 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), round(d['run_loop']['value']))")"
  done
done
