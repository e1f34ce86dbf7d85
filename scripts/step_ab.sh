#!/bin/bash
# A/B sweep of pf_fit_step launch knobs (diagnostics).
for v in "$@"; do
  echo "== $v"
  env $v python scripts/step_prof.py c3 2>&1 | tail -9
done
