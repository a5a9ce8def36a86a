#!/bin/bash
# LSTM GPU tests + C3 bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/test_gpu_lstm.py -x -q > gpurun_out/l_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/l_tests.txt
timeout -s KILL 900 python bench.py --model lstm --steps 3 > gpurun_out/l_bench.json 2> gpurun_out/l_bench.err
