#!/bin/bash
# After the per-kernel R change: GPU suite, bench, K and traction throughput.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r30_pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -2 gpurun_out/r30_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r30_bench.json 2> gpurun_out/r30_bench.err
echo "bench exit $?"; python -c "import json;d=json.load(open('gpurun_out/r30_bench.json'));print(d['value'],d['ms_per_step'],d['roofline']['fp64_pipe_frac'],d['kernels']['nbody'],d['kernels']['offsurface'],d['e2e']['value'],d['clocks'])"
timeout 900 python tools/k_bench.py 3 4 5 > gpurun_out/r30_k.jsonl 2>&1; cat gpurun_out/r30_k.jsonl
timeout 900 python tools/traction_bench.py 3 5 > gpurun_out/r30_tr.jsonl 2>&1; cat gpurun_out/r30_tr.jsonl
