# ncu: launch list of the default bench command, then a full capture of the top kernels
set -x
mkdir -p gpurun_out
timeout 300 python tools/profile_step.py --config 3 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nbody -c 1 \
   -o gpurun_out/prof_nbody_cfg3 python tools/profile_step.py --config 3 > gpurun_out/ncu_nbody.log 2>&1
echo "ncu nbody rc=$?"
timeout 300 python tools/profile_step.py --config 5 --targets 200000 > gpurun_out/plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_nbody|k_self|k_pack|k_reduce" -c 6 \
   -o gpurun_out/prof_cfg5 python tools/profile_step.py --config 5 --targets 200000 > gpurun_out/ncu_cfg5.log 2>&1
echo "ncu cfg5 rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --cpu-seconds 5 > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --e2e-steps 1 --cpu-seconds 5 > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
ls -la gpurun_out
