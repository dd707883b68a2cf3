#!/bin/bash
# NEXT-3 near-corrected K on the GPU.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_traction.py -q -m gpu -x > gpurun_out/r37_traction.log 2>&1
echo "exit $?" >> gpurun_out/r37_traction.log
tail -30 gpurun_out/r37_traction.log
