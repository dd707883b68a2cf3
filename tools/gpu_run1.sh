set -x
nvidia-smi -L; nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"
timeout 120 ./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1; cat gpurun_out/fp64_peak.json
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -50 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config 3 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "bench3 rc=$?"
cat gpurun_out/bench_cfg3.json; tail -5 gpurun_out/bench_cfg3.err
timeout 600 python bench.py --config 5 --steps 2 --warmup 1 --cpu-seconds 10 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "bench5 rc=$?"
cat gpurun_out/bench_cfg5.json; tail -5 gpurun_out/bench_cfg5.err
