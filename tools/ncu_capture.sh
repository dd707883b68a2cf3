#!/bin/bash
# ncu_capture.sh NAME KERNEL_REGEX SKIP -- CMD...
# One `ncu --set full` capture of the kernel matching KERNEL_REGEX (skipping
# SKIP matching launches) of CMD, after CMD has exited 0 without ncu (the
# profiling recipe's rule).  Writes gpurun_out/NAME.ncu-rep and NAME.log.
# Run on the GPU box (gpurun), one GPU, never a multi-rank command.
set -u
name=$1; regex=$2; skip=$3; shift 4
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 "$@" > "gpurun_out/${name}_plain.log" 2>&1 || { echo "plain run failed: $name"; exit 1; }
timeout 2400 ncu --set full --clock-control none --import-source on -k "regex:${regex}" -s "$skip" -c 1 \
  -f -o "gpurun_out/${name}" "$@" > "gpurun_out/${name}.log" 2>&1
echo "ncu $name exit $?"
