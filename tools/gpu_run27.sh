#!/bin/bash
# Evidence refresh: per-config report + ncu launch list of the default bench.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 1800 python tools/config_report.py > gpurun_out/r32_configs.jsonl 2> gpurun_out/r32_configs.err; echo "report exit $?"
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r32_launches.csv python bench.py > gpurun_out/r32_ncu_bench.log 2>&1
echo "ncu exit $?"
