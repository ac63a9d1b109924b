#!/bin/bash
# factor-time A/B of environment settings on one box -> gpurun_out/ab_envs.txt
#   scripts/ab_envs.sh "CFG PLAN" STEPS "ENV1=a ENV2=b" "ENV1=c" ...   (use "-" for no overrides)
mkdir -p gpurun_out
cp="$1"; steps="$2"; shift 2
for v in "$@"; do
  [ "$v" = "-" ] && v=""
  echo -n "[$v] " >> gpurun_out/ab_envs.txt
  env $v timeout 900 python scripts/ab_factor.py $cp $steps >> gpurun_out/ab_envs.txt 2>/dev/null
done
