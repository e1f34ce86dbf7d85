for r in 1 2; do for v in b4 b8; do
  echo "== $v c5: $(PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python bench.py --config c5 --steps 60 --warmup 5 --no-cpu --no-autograd 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), round(d['run_loop']['value']))")"
done; done
for v in b4 b8; do PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python scripts/timeline.py c5 2>&1 | grep "lists"; done
bash scripts/ab_c3.sh b4 b8
