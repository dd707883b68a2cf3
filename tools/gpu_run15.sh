#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_near.py tests/test_gpu_traction.py -q -m gpu -k "high_order" > gpurun_out/r16.log 2>&1
echo "exit $?"; tail -15 gpurun_out/r16.log
