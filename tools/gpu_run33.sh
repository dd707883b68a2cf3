#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_physics.py -q -m gpu > gpurun_out/r44.log 2>&1; echo "exit $?"; tail -5 gpurun_out/r44.log
