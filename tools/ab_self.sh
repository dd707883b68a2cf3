#!/bin/bash
# A/B of self-term libraries on one box (two interleaved rounds):
#   tools/ab_self.sh "CFGS" LIB...   e.g. tools/ab_self.sh "3 4 5" abtest/libbie_a.so abtest/libbie_b.so
cd "${GRAFT_REPO_ROOT:-.}"
cfgs=$1; shift
for round in 1 2; do
  for lib in "$@"; do
    cp "$lib" paper_1707_06551_b200/libbie.so
    timeout 600 python tools/self_bench.py $cfgs --variants 2 | sed "s|^|{\"lib\": \"$lib\", \"round\": $round} |"
  done
done
