#!/bin/bash
# near / traction / porous GPU tests after the k_near<STAGE, K> refactor
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_near.py tests/test_gpu_traction.py tests/test_gpu_porous.py tests/test_gpu_physics.py -q -m gpu > gpurun_out/r17.log 2>&1
echo "exit $?"; tail -4 gpurun_out/r17.log
timeout 600 python tools/k_bench.py 4 > gpurun_out/r17_k.jsonl 2>&1; cat gpurun_out/r17_k.jsonl
timeout 600 python tools/near_bench.py 4 > gpurun_out/r17_near.jsonl 2>&1; tail -2 gpurun_out/r17_near.jsonl
