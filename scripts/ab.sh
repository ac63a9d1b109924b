#!/bin/bash
# alternate two library builds on the same box: scripts/ab.sh A B [rounds]
for r in $(seq 1 ${3:-2}); do
  for v in $1 $2; do echo -n "$v: "; CE_LIB_OVERRIDE=scripts/build/ab/$v.so ./scripts/sweep_levels.sh; done
done
