#!/bin/bash
# Sharded-factorization GPU checks + the full-size parity report.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_shard.py tests/test_gpu_fullsize_parity.py -q -x > gpurun_out/pytest_shard.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_shard.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
