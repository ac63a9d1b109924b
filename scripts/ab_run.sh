#!/bin/bash
# usage: scripts/ab_run.sh "A B" "cfg plan" rounds steps -> gpurun_out/ab.txt
mkdir -p gpurun_out
for r in $(seq 1 ${3:-2}); do
  for v in $1; do
    CE_LIB_OVERRIDE=scripts/build/ab/$v.so timeout 600 python scripts/ab_factor.py $2 ${4:-3} >> gpurun_out/ab.txt 2>/dev/null
  done
done
