# A/B of K1's lanes per primitive (PF_PRIM_LPP) on the c5 8-way band and full c5
# (build first: bash scripts/ab_build.sh "l0:" "l8:-DPF_PRIM_LPP=8")
set -u
for r in 1 2; do for v in l0 l8; do
  echo "== $v: $(PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python scripts/band_scaling.py c5 1 8 2>&1 | grep -E 'N=(1|8) uniform' | tr '\n' ' ' | cut -c1-260)"
done; done
