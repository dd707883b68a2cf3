#!/bin/bash
# ncu launch list of the default bench command (shares, cold-cache, serialised).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/r27_bench_plain.json 2>/dev/null; echo "plain exit $?"
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r27_launches.csv python bench.py > gpurun_out/r27_ncu_bench.log 2>&1
echo "ncu exit $?"; wc -l gpurun_out/r27_launches.csv
