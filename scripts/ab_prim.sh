# K1 occupancy variants (PF_PRIM_HI) on the c5 full canvas and an 8-way band
set -u
for v in hi5 hi4 hi3; do
  for a in "c5" "c5 band=8:3"; do
    echo "== $v $a"; PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python scripts/timeline.py $a 2>&1 | tail -6
  done
done
