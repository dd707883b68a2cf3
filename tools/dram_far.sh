#!/bin/bash
# DRAM bytes of the apply and off-surface k_nbody launches on cfg 5, per library
cd "${GRAFT_REPO_ROOT:-.}"
for lib in "$@"; do
  cp "$lib" paper_1707_06551_b200/libbie.so
  echo "== $lib"
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:^k_nbody$ -c 2 python tools/profile_step.py --config 5 2>&1 | grep -E "k_nbody|dram__|gpu__time|pipe_fp64"
done
