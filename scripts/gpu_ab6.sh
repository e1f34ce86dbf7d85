set -u
for v in t256x2 nosort; do
  echo "== slot $v timeline c5"; PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python scripts/timeline.py c5 2>&1 | tail -6 | head -3
  echo "== slot $v step_prof c5"; PF_LIB=paper_2602_22625_b200/_lib_alt/$v.so timeout 300 python scripts/step_prof.py c5 2>&1 | head -7
done
echo "== csr step_prof c5"; PF_CSR_STEP=1 PF_LIB=paper_2602_22625_b200/_lib_alt/t256x2.so timeout 300 python scripts/step_prof.py c5 2>&1 | head -7
echo "== old step_prof c5"; (cd _ab_old && timeout 300 python scripts/step_prof.py c5 2>&1 | head -7)
