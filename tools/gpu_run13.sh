#!/bin/bash
# Full GPU suite + smoke + default bench (round-end style check).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r49_pytest_gpu.log 2>&1
echo "pytest exit $?" | tee -a gpurun_out/r49_pytest_gpu.log
tail -3 gpurun_out/r49_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r49_smoke.log 2>&1
echo "smoke exit $?"; tail -1 gpurun_out/r49_smoke.log
timeout 900 python bench.py > gpurun_out/r49_bench.json 2> gpurun_out/r49_bench.err; echo "bench exit $?"

