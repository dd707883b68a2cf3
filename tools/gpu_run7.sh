mkdir -p gpurun_out
for w in K near nearoff self; do timeout 300 python tools/profile_extra.py --what $w > gpurun_out/plain_$w.log 2>&1 || echo "plain $w failed"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nbody -c 1 -o gpurun_out/prof_K python tools/profile_extra.py --what K > gpurun_out/ncu_K.log 2>&1; echo K=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_near" -c 2 -o gpurun_out/prof_near python tools/profile_extra.py --what near > gpurun_out/ncu_near.log 2>&1; echo near=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_near_off" -c 1 -o gpurun_out/prof_nearoff python tools/profile_extra.py --what nearoff > gpurun_out/ncu_nearoff.log 2>&1; echo nearoff=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_self" -s 1 -c 1 -o gpurun_out/prof_self5 python tools/profile_extra.py --what self > gpurun_out/ncu_self.log 2>&1; echo self=$?
