mkdir -p gpurun_out
timeout 300 python tools/profile_extra.py --what near > gpurun_out/plain_near.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_near$" -c 1 -o gpurun_out/prof_knear python tools/profile_extra.py --what near > gpurun_out/ncu_knear.log 2>&1; echo knear=$?
