#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 1800 python tools/fig9_bench.py > gpurun_out/r40_fig9.jsonl 2> gpurun_out/r40_fig9.err; echo "exit $?"; cat gpurun_out/r40_fig9.jsonl; tail -2 gpurun_out/r40_fig9.err
