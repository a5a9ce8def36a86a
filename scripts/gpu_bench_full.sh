#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${1:-bf}
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/${TAG}_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_gpu.txt
timeout -s KILL 600 python bench.py > gpurun_out/${TAG}_bench.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_bench.txt
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_ref.txt 2>&1
