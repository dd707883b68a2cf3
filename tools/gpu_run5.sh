set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/config_report.py --configs 1 2 > gpurun_out/configs12.jsonl 2>&1; cat gpurun_out/configs12.jsonl
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
cat gpurun_out/bench_default.json
