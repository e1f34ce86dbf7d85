set -u
b() { timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['stage_ms']['step'])"; }
echo "nbuf2 atl64"; b
echo "nbuf2 atl32"; PF_STEP_ATL32=1 b
PF_NVCC_DEFS="-DPF_NBUF=3" python -c "from paper_2602_22625_b200 import build; build.build(force=True)"
echo "nbuf3 atl32"; PF_STEP_ATL32=1 b
echo "nbuf3 atl32 prof"; PF_STEP_ATL32=1 timeout 120 python scripts/step_prof.py c3 2>&1 | sed -n 2,5p
