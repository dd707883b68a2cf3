#!/bin/bash
# A/B of far-field libraries on one box: abtest/ab.sh CFG MODES_NEW LIB...
cd "${GRAFT_REPO_ROOT:-.}"
cfg=$1; shift
for round in 1 2; do
  for lib in "$@"; do
    cp "$lib" paper_1707_06551_b200/libbie.so
    modes=1; case "$lib" in *new*) modes=1,6;; esac
    FR_MODES=$modes timeout 600 python tools/far_reduction_bench.py $cfg | sed "s|^|{\"lib\": \"$lib\", \"round\": $round} |"
  done
done
