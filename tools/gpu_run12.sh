#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 900 python tools/traction_bench.py 3 5 > gpurun_out/r13_traction_bench.jsonl 2> gpurun_out/r13_tb.err
echo "exit $?"; cat gpurun_out/r13_traction_bench.jsonl; tail -3 gpurun_out/r13_tb.err
