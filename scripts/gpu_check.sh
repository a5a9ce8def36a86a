#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r1_smi.txt 2>&1
timeout -s KILL 400 python -m pytest tests/test_gpu_gemm.py -x -q --timeout 120 > gpurun_out/r1_gemm.txt 2>&1
echo "gemm rc=$?" >> gpurun_out/r1_gemm.txt
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r1_gpu.txt 2>&1
echo "gpu rc=$?" >> gpurun_out/r1_gpu.txt
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-baseline > gpurun_out/r1_bench.txt 2>&1
echo "bench rc=$?" >> gpurun_out/r1_bench.txt
tail -5 gpurun_out/r1_gemm.txt gpurun_out/r1_gpu.txt gpurun_out/r1_bench.txt
