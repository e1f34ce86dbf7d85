set -u
mkdir -p gpurun_out/ab3
run() { # name dir env...
  local name=$1 dir=$2; shift 2
  (cd $dir && env "$@" timeout 900 ncu --set full --clock-control none --import-source on \
     -k regex:"k_step|k_prim" -s 20 -c 4 -o $GRAFT_REPO_ROOT/gpurun_out/ab3/prof_$name -f \
     python bench.py --steps 3 --warmup 3 --no-cpu --no-autograd > $GRAFT_REPO_ROOT/gpurun_out/ab3/ncu_$name.log 2>&1); echo "ncu $name rc=$?"
}
run old _ab_old X=1
run csr . PF_CSR_STEP=1 PF_LIB=paper_2602_22625_b200/_lib_alt/t256x2.so
run slot . PF_LIB=paper_2602_22625_b200/_lib_alt/t256x2.so
