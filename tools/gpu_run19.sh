#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_near.py tests/test_gpu_porous.py tests/test_gpu_traction.py tests/test_gpu_properties.py -q -m gpu -x > gpurun_out/r48.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/r48.log
timeout 600 python tools/self_bench.py > gpurun_out/r48_self.txt 2>&1; cat gpurun_out/r48_self.txt
