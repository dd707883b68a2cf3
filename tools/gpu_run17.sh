#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 1800 python tools/config_report.py > gpurun_out/r18_configs.jsonl 2> gpurun_out/r18_configs.err
echo "exit $?"; cat gpurun_out/r18_configs.jsonl; tail -3 gpurun_out/r18_configs.err
