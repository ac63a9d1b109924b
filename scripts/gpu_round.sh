#!/bin/bash
# One gpurun pass: GPU tests (parity report into gpurun_out/), the default bench line, smoke.
# usage (from the repo root, under gpurun): bash scripts/gpu_round.sh [pytest -k expr]
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
K=${1:+-k "$1"}
timeout 2400 python -m pytest tests -m gpu -x -q $K > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
