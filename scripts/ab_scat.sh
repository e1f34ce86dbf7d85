# A/B of the K1 slot-scatter batch (PF_SCAT_BATCH) on c3 and on a c5 band of an 8-way split
set -u
for r in 1 2; do for v in s4 s8 s2; do
  echo "== $v c3: $(PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python bench.py --config c3 --steps 100 --warmup 5 --no-cpu --no-autograd 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), round(d['run_loop']['value']))")"
  echo "== $v c5 band8: $(PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python scripts/band_scaling.py c5 1 8 2>&1 | grep 'N=8 uniform')"
done; done
