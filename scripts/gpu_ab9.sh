set -u
for v in t256x2 nosort; do
L=paper_2602_22625_b200/_lib_alt/$v.so
for cfg in c5 c3; do
echo "== $cfg $v"; PF_LIB=$L timeout 300 python scripts/step_prof.py $cfg 2>&1 | head -3
done
done
echo "== c5 csr"; PF_CSR_STEP=1 PF_LIB=$L timeout 300 python scripts/step_prof.py c5 2>&1 | head -3
