#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 1500 python tools/sj_convergence.py > gpurun_out/r43_sj.jsonl 2> gpurun_out/r43_sj.err; echo "exit $?"
python -c "
import json
for l in open('gpurun_out/r43_sj.jsonl'):
    d=json.loads(l); print(d['gap'], d['p'], d['iterations'], '%.2e'%d['rel_resid'], '%.3e'%d['rel_err'])
"; tail -3 gpurun_out/r43_sj.err
