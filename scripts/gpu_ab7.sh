set -u
L=paper_2602_22625_b200/_lib_alt/t256x2.so
for cfg in c5 c3; do
echo "== $cfg slot"; PF_LIB=$L timeout 300 python scripts/step_prof.py $cfg 2>&1 | head -4
echo "== $cfg slot psleep50"; PF_PSLEEP=50 PF_LIB=$L timeout 300 python scripts/step_prof.py $cfg 2>&1 | head -4
echo "== $cfg slot psleep50 csleep50"; PF_CSLEEP=50 PF_PSLEEP=50 PF_LIB=$L timeout 300 python scripts/step_prof.py $cfg 2>&1 | head -4
echo "== $cfg csr"; PF_CSR_STEP=1 PF_LIB=$L timeout 300 python scripts/step_prof.py $cfg 2>&1 | head -4
done
