#!/bin/bash
# A/B of launch knobs via env (diagnostics): bash scripts/ab_env.sh "A=1" "B=2 C=3" ...
set -u
b() { timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-autograd 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['stage_ms']['step']*1e3,2), round(d['e2e']['value']))"; }
for v in "$@"; do echo "== $v: $(env $v bash -c "$(declare -f b); b")"; done
