# K1 variants: bench c3 twice each, alternating, plus K1 timelines
set -u
for r in 1 2; do bash scripts/ab_variants.sh "$@" 2>&1 | grep c3; done
for v in "$@"; do echo "== $v"; for k in 1 2 3; do PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python scripts/timeline.py c3 2>&1 | grep "k_prim"; done; done
