#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 600 python tools/chunk_sweep.py 2 0 27 54 81 > gpurun_out/r36_chunks.jsonl 2>&1; echo "exit $?"; cat gpurun_out/r36_chunks.jsonl
