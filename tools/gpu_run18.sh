#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 300 python tools/profile_extra.py --what self > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_self -s 1 -c 1 \
  -o gpurun_out/r19_self5 -f python tools/profile_extra.py --what self > gpurun_out/r19_ncu.log 2>&1
echo "ncu exit $?"; tail -2 gpurun_out/r19_ncu.log
