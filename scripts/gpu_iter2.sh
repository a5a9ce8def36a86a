#!/bin/bash
# one iteration on the GPU box: tests, bench, GEMM phase stamps, warm ncu launch list (32 layers)
cd "$GRAFT_REPO_ROOT"
TAG=${1:-it}
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/${TAG}_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_gpu.txt
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-baseline > gpurun_out/${TAG}_bench.txt 2>&1
timeout -s KILL 300 python scripts/gemm_phases.py 0,256,8 1,256,8 0,256,4 0,128,8 > gpurun_out/${TAG}_phases.txt 2>&1
bash scripts/gpu_launch32.sh ${TAG}
