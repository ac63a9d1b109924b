#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): bench line, ncu launch list, sweep DRAM
# traffic per level, one --set full capture of the level-6 sweep launch.  Outputs in gpurun_out/.
set -x
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
timeout 900 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:sweep_kernel -c 9 --csv --log-file gpurun_out/sweep_traffic.csv python scripts/levels.py 2 > gpurun_out/ncu_traffic.log 2>&1
timeout 1200 $NCU --set full --import-source on --clock-control none -k regex:sweep_kernel --launch-skip 5 -c 1 \
  -o gpurun_out/sweep_L6 python scripts/ncu_sweep.py 1024 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
