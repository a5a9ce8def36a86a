#!/bin/bash
# chain: GPU suite + C2 bench line (quick A/B of a chain change)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x > gpurun_out/q_gpu_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/q_gpu_tests.txt
timeout -s KILL 900 python bench.py --no-lstm > gpurun_out/q_bench_c2.json 2> gpurun_out/q_bench_c2.err
