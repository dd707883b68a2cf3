#!/bin/bash
# NEXT-3 completion operator + traction tests on the GPU.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_traction.py -q -m gpu > gpurun_out/r9_traction.log 2>&1
echo "exit $?" >> gpurun_out/r9_traction.log
tail -5 gpurun_out/r9_traction.log
