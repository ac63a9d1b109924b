#!/bin/bash
# factor-time comparison of several library builds on one box: scripts/ab_multi.sh rounds A B C ...
rounds=$1; shift
for r in $(seq 1 $rounds); do
  for v in "$@"; do
    echo -n "$v: "
    CE_LIB_OVERRIDE=scripts/build/ab/$v.so python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['factor_ms_steps'], d['pcg_ms_steps'])"
  done
done
