#!/bin/bash
# factor-time A/B of library builds on one box: scripts/ab_bench.sh A B [rounds]
for r in $(seq 1 ${3:-2}); do
  for v in $1 $2; do
    echo -n "$v: "
    CE_LIB_OVERRIDE=scripts/build/ab/$v.so python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['factor_ms_steps'], d['pcg_ms_steps'])"
  done
done
