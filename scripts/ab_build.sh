#!/bin/bash
# Build A/B variants of the library into paper_2602_22625_b200/_lib_alt/<name>.so
# (diagnostics): bash scripts/ab_build.sh "base:" "x:-DFOO=1" ...; run them on one box
# with PF_LIB=paper_2602_22625_b200/_lib_alt/<name>.so (scripts/ab_env.sh).
set -e
mkdir -p paper_2602_22625_b200/_lib_alt
for v in "$@"; do
  n=${v%%:*}; d=${v#*:}
  PF_NVCC_DEFS="$d" python -c "from paper_2602_22625_b200 import build; build.build(force=True)"
  cp paper_2602_22625_b200/_lib/libprimfit_b200.so paper_2602_22625_b200/_lib_alt/$n.so
done
python -c "from paper_2602_22625_b200 import build; build.build(force=True)"
