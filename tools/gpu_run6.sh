mkdir -p gpurun_out
timeout 300 python tools/self_bench.py 4 > gpurun_out/self4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_self -s 5 -c 1 \
   -o gpurun_out/prof_self_cfg4 python tools/self_bench.py 4 > gpurun_out/ncu_self.log 2>&1
echo "ncu rc=$?"
