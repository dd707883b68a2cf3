#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/r38_bench.json 2> gpurun_out/r38_bench.err
echo "bench exit $?"; python -c "import json;d=json.load(open('gpurun_out/r38_bench.json'));print(d['value'],d['kernels'],d['roofline']['fp64_pipe_frac'])"; tail -2 gpurun_out/r38_bench.err
