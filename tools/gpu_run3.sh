set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
cat gpurun_out/bench_default.json
timeout 300 python tools/profile_step.py --config 3 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nbody -c 1 \
   -o gpurun_out/prof_nbody_cfg3_r8 python tools/profile_step.py --config 3 > gpurun_out/ncu_nbody.log 2>&1
echo "ncu rc=$?"
