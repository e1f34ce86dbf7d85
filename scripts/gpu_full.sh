# full GPU suite + smoke
set -u
mkdir -p gpurun_out/full
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/full/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/full/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
