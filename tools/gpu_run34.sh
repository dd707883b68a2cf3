#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
RESTART=200 MAX_ITER=300 timeout 2400 python tools/porous_bench.py 4 > gpurun_out/r45_porous4.jsonl 2> gpurun_out/r45.err; echo "exit $?"; cat gpurun_out/r45_porous4.jsonl; tail -2 gpurun_out/r45.err
