#!/bin/bash
# Per-level sweep + apply timings (CE_PROFILE=1) for cfg2 and cfg3 on the reference plan.
mkdir -p gpurun_out
for c in 2 3; do
  CE_PROFILE=1 timeout 600 python bench.py --cfg $c --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-variants --no-extra \
    > gpurun_out/prof_cfg$c.json 2> gpurun_out/prof_cfg$c.err
done
