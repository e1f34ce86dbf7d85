bash scripts/ab_env.sh "X=1" "PF_CSLEEP=100" "PF_CSLEEP=50 PF_PSLEEP=100" "PF_PSLEEP=200" "PF_CSLEEP=400"
for v in base dm1 dm4 ks4 ks6; do
  echo "== $v: $(PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-autograd 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['stage_ms']['step']*1e3,2), round(d['e2e']['value']))") c2: $(PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python bench.py --config c2 --steps 300 --warmup 10 --no-cpu --no-autograd 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']))")"
done
