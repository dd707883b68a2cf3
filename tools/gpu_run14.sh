#!/bin/bash
# GMRES restart-length study for BIE 5.4 (NEXT-2).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
for R in 30 50 100 200; do
  RESTART=$R MAX_ITER=400 timeout 600 python tools/porous_bench.py 2 3 >> gpurun_out/r15_restart.jsonl 2>> gpurun_out/r15.err
done
RESTART=300 MAX_ITER=400 timeout 1500 python tools/porous_bench.py 5 >> gpurun_out/r15_restart.jsonl 2>> gpurun_out/r15.err
echo "exit $?"; cat gpurun_out/r15_restart.jsonl; tail -3 gpurun_out/r15.err
