set -x
mkdir -p gpurun_out
timeout 1500 python tools/config_report.py --configs 1 2 3 4 5 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "report rc=$?"
cat gpurun_out/configs.jsonl; tail -3 gpurun_out/configs.err
timeout 300 python tools/profile_step.py --config 5 --no-off > gpurun_out/plain5a.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_nbody -c 1 \
   -o gpurun_out/prof_nbody_cfg5 python tools/profile_step.py --config 5 --no-off > gpurun_out/ncu_nbody5.log 2>&1
echo "ncu rc=$?"
