#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 ./tools/nbody_tune 106 20 S > gpurun_out/r34_small.txt 2>&1; echo "exit $?"; cat gpurun_out/r34_small.txt
