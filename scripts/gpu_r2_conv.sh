#!/bin/bash
# f4 conv ResNet: GPU tests (+ the f1 ops tests), strategy comparison
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_ops.py -x -q > gpurun_out/c_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/c_tests.txt
CONV=1 HW=32 DEPTHS=3,3,3 WIDTHS=128,256,512 B=64 timeout -s KILL 600 python scripts/ops_strategies.py > gpurun_out/c_strategies.json 2>&1
