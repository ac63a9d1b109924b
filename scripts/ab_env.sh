#!/bin/bash
# factor-time A/B of one build under two environment settings on one box:
#   scripts/ab_env.sh "VAR=a" "VAR=b" [rounds]
for r in $(seq 1 ${3:-2}); do
  for v in "$1" "$2"; do
    echo -n "$v: "
    env $v python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['factor_ms_steps'], d['pcg_ms_steps'], d['pcg_iterations'])"
  done
done
