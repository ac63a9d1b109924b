#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_shard.py tests/test_gpu_fullsize_parity.py -q > gpurun_out/pytest_shard.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_shard.log
bash scripts/ab_run.sh "base vec" "3 reference" 2 3
bash scripts/ab_run.sh "base vec" "2 reference" 2 3
