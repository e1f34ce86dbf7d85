# fp32 bilinear path A/B (PF_F32_LERP), with the fp64 / fp32 shared atlas
set -u
b() { timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-autograd "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), round(d['run_loop']['value']))"; }
for r in 1 2; do
  for v in base lerp; do
    echo "== $v atl64: $(PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so b)"
    echo "== $v atl32: $(PF_STEP_ATL32=1 PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so b)"
  done
done
for v in base lerp; do echo "== $v c5: $(PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so b --config c5 --steps 60)"; done
PF_LIB=paper_2602_22625_b200/_lib_alt/lerp.so timeout 900 python -m pytest tests/test_gpu_slots.py tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x 2>&1 | tail -2
PF_STEP_ATL32=1 PF_LIB=paper_2602_22625_b200/_lib_alt/lerp.so timeout 900 python -m pytest tests/test_gpu_slots.py tests/test_gpu_scale.py -q -x -k "fused or slot or edge" 2>&1 | tail -2
