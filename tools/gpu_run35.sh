#!/bin/bash
# ncu --set full: K far field (cfg 3, R = 7) and the off-surface kernel (cfg 5, 200k targets, R = 7).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 300 python tools/profile_extra.py --what K > /dev/null 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_nbody -c 1 \
  -o gpurun_out/r46_K -f python tools/profile_extra.py --what K > gpurun_out/r46_ncuK.log 2>&1
echo "K exit $?"
timeout 600 python tools/profile_step.py --config 5 --targets 200000 > /dev/null 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_nbody -s 1 -c 1 \
  -o gpurun_out/r46_off -f python tools/profile_step.py --config 5 --targets 200000 > gpurun_out/r46_ncuoff.log 2>&1
echo "off exit $?"
