#!/bin/bash
# K apply cost with the near correction + completion; ncu of k_near_K (cfg 4).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 900 python tools/k_bench.py 3 4 5 > gpurun_out/r11_kbench.jsonl 2> gpurun_out/r11_kbench.err
echo "kbench exit $?"
cat gpurun_out/r11_kbench.jsonl
timeout 300 python tools/profile_extra.py --what nearK > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_near_K -c 1 \
  -o gpurun_out/r11_nearK -f python tools/profile_extra.py --what nearK > gpurun_out/r11_ncu.log 2>&1
echo "ncu exit $?"
tail -3 gpurun_out/r11_ncu.log
