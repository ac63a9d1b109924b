#!/bin/bash
# factor-time A/B of the chain ticket placement (CE_CHAIN_FRAC) on one box -> gpurun_out/ab_chain.txt
#   scripts/ab_chain.sh "1.0 0.5 0.3" "3 reference" [rounds] [steps]
mkdir -p gpurun_out
for r in $(seq 1 ${3:-1}); do
  for v in $1; do
    echo -n "frac=$v " >> gpurun_out/ab_chain.txt
    CE_CHAIN_FRAC=$v timeout 900 python scripts/ab_factor.py $2 ${4:-2} >> gpurun_out/ab_chain.txt 2>/dev/null
  done
done
