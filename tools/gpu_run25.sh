#!/bin/bash
# k_nbody blocking sweep with tools/nbody_tune (2,000 spheres x p = 6 grouping): apply/off then K.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 ./tools/nbody_tune 2000 3 P > gpurun_out/r31_tune_P.txt 2>&1; echo "exit $?"; cat gpurun_out/r31_tune_P.txt

