#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun): the default bench line (cfg3), its ncu launch
# list, the sweep kernels' DRAM traffic over one cfg3 factorization, one --set full capture of the
# level-8 sweep launch.  Outputs in gpurun_out/; scripts/process_profiles_r2.py files them.
set -x
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv \
  python scripts/ab_factor.py 3 reference 1 > gpurun_out/ncu_launches.log 2>&1
timeout 1200 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:sweep_kernel -c 10 --csv --log-file gpurun_out/sweep_traffic_cfg3.csv python scripts/level_table.py 3 reference \
  > gpurun_out/ncu_traffic.log 2>&1
timeout 1500 $NCU --set full --import-source on --clock-control none -k regex:sweep_kernel --launch-skip 7 -c 1 \
  -o gpurun_out/sweep_cfg3_L8 python scripts/ab_factor.py 3 reference 0 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
