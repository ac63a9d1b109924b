#!/bin/bash
mkdir -p gpurun_out
for cp in "3 reference" "2 reference" "2 merge_all_colored" "3 merge_all_colored"; do
  set -- $cp
  CE_PROFILE=1 timeout 600 python scripts/level_table.py $1 $2 > gpurun_out/levels_cfg$1_$2.jsonl 2> gpurun_out/levels_cfg$1_$2.err
done
