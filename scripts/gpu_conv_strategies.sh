#!/bin/bash
# f4 conv ResNet: tests + five strategies vs depth (Fig. 5 style)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_conv.py -x -q > gpurun_out/c2_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/c2_tests.txt
for dep in 1,1,1 3,3,3 6,6,6 12,12,12; do
  CONV=1 HW=32 DEPTHS=$dep WIDTHS=128,256,512 B=64 timeout -s KILL 600 python scripts/ops_strategies.py > gpurun_out/c2_strat_$dep.json 2>&1
done
