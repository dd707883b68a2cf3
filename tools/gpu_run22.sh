#!/bin/bash
# ncu --set full of the far-field kernel on the cfg 5 apply (roofline.traffic source).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 600 python tools/profile_step.py --config 5 --no-off > gpurun_out/r25_plain.log 2>&1; echo "plain exit $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_nbody -c 1 \
  -o gpurun_out/r25_nbody_cfg5 -f python tools/profile_step.py --config 5 --no-off > gpurun_out/r25_ncu.log 2>&1
echo "ncu exit $?"; tail -2 gpurun_out/r25_ncu.log
